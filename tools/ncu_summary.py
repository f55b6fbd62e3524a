"""Summarise ncu reports/CSVs into profiles/*.md (run here, no GPU needed).

  python tools/ncu_summary.py report  <x.ncu-rep>  > profiles/...md
  python tools/ncu_summary.py launches <launches.csv>
"""
import collections
import csv
import io
import subprocess
import sys


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    rows = ncu_csv([path, "--page", "details"])
    h = rows[0]
    keep = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Theoretical Active Warps per SM",
            "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
            "Executed Instructions", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
    kname = None
    print(f"# ncu summary: `{path}`\n")
    print("| metric | value |\n|---|---|")
    for r in rows[1:]:
        d = dict(zip(h, r))
        kname = kname or d.get("Kernel Name")
        if d["Metric Name"] in keep:
            print(f"| {d['Metric Name']} | {d['Metric Value']} {d['Metric Unit']} |")
    raw = ncu_csv([path, "--page", "raw"])
    names, vals = raw[0], raw[2]
    stalls, pipes, other = [], [], {}
    for n, v in zip(names, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
            stalls.append((x, n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        if n.startswith("sm__inst_executed_pipe_") and n.endswith("avg.pct_of_peak_sustained_active"):
            pipes.append((x, n.replace("sm__inst_executed_pipe_", "").split(".")[0]))
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            other[n] = (x, raw[1][names.index(n)])
    for n, (x, u) in other.items():
        print(f"| {n} | {x} {u} |")
    print(f"\nKernel: `{kname}`\n")
    tot = sum(x for x, _ in stalls) or 1
    print("Warp stall samples: " + ", ".join(f"{n} {x / tot * 100:.1f}%"
                                              for x, n in sorted(stalls, reverse=True)[:8]))
    print("\nPipe utilisation (% of peak, active): " +
          ", ".join(f"{n} {x:.1f}%" for x, n in sorted(pipes, reverse=True)[:8] if x > 0.5))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = ""
    for r in rows[hdr_i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        k = d["Kernel Name"].split("(")[0][:90]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(t for _, t in agg.values()) or 1
    print(f"# ncu launch list: `{path}` (cold-cache, serialised: compare shares)\n")
    print(f"| kernel | launches | total {unit} | avg {unit} | share |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.0f} | {t / n:.1f} | {t / tot * 100:.1f}% |")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])

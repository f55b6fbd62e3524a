"""Opcode mix of an ncu capture (executed warp-instructions per SASS opcode),
from `ncu -i REP --page source --csv --print-source sass`.

  python tools/ncu_opmix.py REP [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, ie, iw = h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
mix, stall = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    src = r[ia].strip()
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    mix[op] += int(float(r[ie] or 0))
    stall[op] += int(float(r[iw] or 0))
tot = sum(mix.values())
ts = sum(stall.values()) or 1
print(f"total executed warp-instructions: {tot}")
print("| opcode | executed | share | stall samples share |\n|---|---|---|---|")
for op, n in mix.most_common(top):
    print(f"| {op} | {n} | {100 * n / tot:.1f} % | {100 * stall[op] / ts:.1f} % |")

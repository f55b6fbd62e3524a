#!/usr/bin/env python3
"""Benchmark driver for the B200-native WMC filter.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cfg1..cfg5] [--all OUT.json]

Default workload: BASELINE.json configs[3] ("cfg4"), the 16384x16384 fp32
image filtered for 200 iterations -- the configuration the metric's 1/2/4/8
GPU scaling is quoted on (row-band sharded across ranks, one process per GPU,
halo rows exchanged over NCCL each launch).  One STEP = the whole 200-iteration
filter of that image.  Inputs are seeded synthetic images of the configured
shape / value distribution; the 1 GiB image exceeds the 126 MB
L2, so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line (metric, value, e2e, roofline, cpu_baseline,
clocks, gpu_launches, ...).  ``--impl reference`` times the reference CPU path
(the fp64 SPEC-faithful restatement in oracle/, all host threads) on a bounded
sample of the same workload and prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "WMC Gpixel-updates/s"
UNIT = "Gpixel-updates/s"
BYTES_PER_UPDATE = 8  # 4 B read of U^t + 4 B write of U^{t+1}
L2_BYTES = 126 * 1024 * 1024


def _ncu_json():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_launch_ms(kernel: str, h: int, w: int, planes: int):
    """ncu gpu__time_duration of one launch at this geometry (cold cache,
    serialised) from the committed capture, else None."""
    return _ncu_json().get(f"{kernel}@{planes}x{h}x{w}:ms")


def ncu_traffic(kernel: str, h: int, w: int, planes: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at
    this geometry, from the committed ncu --set full capture
    (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(f"{kernel}@{planes}x{h}x{w}")
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# ------------------------------------------------------------- helpers -----
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_name(cfg) -> str:
    """The config's name in both arms' JSON lines."""
    return (f"{cfg.name}: {cfg.planes}x{cfg.h}x{cfg.w} {'u8' if cfg.u8 else 'f32'}, "
            f"{cfg.iters or 1} {'iterations' if cfg.iters else 'map evaluation'}, dt={cfg.dt}")


def make_input(cfg, rows=None, threads=0, planes=None):
    """Seeded synthetic input (host numpy); rows = (r0, r1) crop, planes =
    (p0, p1) subset (plane p keeps its own seed, so shards equal the slices
    of the full batch)."""
    import numpy as np

    import paper_1903_07189_b200 as cf
    imgs = []
    p0, p1 = planes if planes is not None else (0, cfg.planes)
    for p in range(p0, p1):
        a = cf.synth_image(cfg.h, cfg.w, cfg.seed(p), cfg.n_rects, cfg.n_discs, cfg.sigma,
                           dtype="u8" if cfg.u8 else "f32", threads=threads)
        imgs.append(a if rows is None else a[rows[0]:rows[1]])
    return np.stack(imgs) if cfg.planes > 1 else imgs[0]


def load_configs():
    """paper_1903_07189_b200/configs.py loaded as a standalone module, so the
    reference arm imports nothing else from the product package."""
    import importlib.util
    path = os.path.join(ROOT, "paper_1903_07189_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("cf_bench_configs", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["cf_bench_configs"] = mod  # dataclasses resolve the module by name
    spec.loader.exec_module(mod)
    return mod.CONFIGS, mod.SUPPLEMENTAL


def bench_config(cfg) -> dict:
    """The workload's `config` object -- identical in both arms' JSON lines
    (implementation details go to "impl_config")."""
    return {"workload": workload_name(cfg), "iters": cfg.iters, "planes": cfg.planes,
            "h": cfg.h, "w": cfg.w, "dt": cfg.dt}


def algorithmic_bytes(cfg, pixels: int, u8_out: bool) -> int:
    """4 B read of U^t + 4 B write of U^{t+1} per pixel-update;
    the u8 path reads 1 B on the first sweep and (u8 out) writes 1 B on the
    last one.  `pixels` = pixels of one full-image pass."""
    if cfg.iters == 0:
        return pixels * BYTES_PER_UPDATE
    if not cfg.u8:
        return pixels * cfg.iters * BYTES_PER_UPDATE
    last_w = 1 if u8_out else 4
    if cfg.iters == 1:
        return pixels * (1 + last_w)
    return pixels * ((1 + 4) + (cfg.iters - 2) * 8 + (4 + last_w))


def cpu_reference(threads: int):
    """The reference CPU path: the fp64 SPEC-faithful mc_flow / wmc_half_laplace
    run on the reference's own executor (oracle/_ref/libcf_ref.so, compiled
    against /root/reference/proj/include/curveflow/parallel.hpp:26-47), or,
    when that build is absent, the oracle's for_rows restatement.
    Returns (flow(img, n), map(img), kind, what)."""
    import oracle
    if oracle.ref_lib() is not None:
        return (lambda img, n, dt: oracle.ref_flow_f64(img, n, dt, threads, inplace=True),
                lambda img: oracle.ref_wmc_map_f64(img, threads), "reference",
                "oracle/_ref/libcf_ref.so: the fp64 SPEC-faithful restatement on the "
                "reference's own curveflow::parallel executor (parallel.hpp:26-47)")
    return (lambda img, n, dt: oracle.flow_f64(img, n, dt, threads, inplace=True),
            lambda img: oracle.wmc_map_f64(img, threads), "port",
            "oracle/wmc_oracle.c: the fp64 SPEC-faithful restatement (for_rows port)")


def cpu_reference_sample(cfg, img64, budget_s=10.0):
    """Time the reference CPU path on a bounded sample of the workload: the
    FULL-SIZE first plane `img64` (fp64, widened from u8 if needed), n of the
    workload's iterations (a map workload: n evaluations), n sized from one
    timed iteration so the sample is ~budget_s of CPU work.
    Returns (Gupd/s, cores, sample description, kind, n, seconds per sample)."""
    threads = os.cpu_count() or 1
    flow, wmap, kind, what = cpu_reference(threads)
    h, w = img64.shape
    work = img64.copy()
    t0 = time.perf_counter()
    if cfg.iters == 0:
        wmap(work)
    else:
        flow(work, 1, cfg.dt)
    one = time.perf_counter() - t0
    n = max(1, min(cfg.iters or 50, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    if cfg.iters == 0:
        for _ in range(n):
            wmap(work)
    else:
        flow(work, n, cfg.dt)
    sec = time.perf_counter() - t0
    rate = h * w * n / sec / 1e9
    sample = (f"{what}; {'wmc_half_laplace' if cfg.iters == 0 else 'mc_flow'} on the full "
              f"{h}x{w} first plane of the {cfg.name} input, {n} "
              f"{'evaluation(s)' if cfg.iters == 0 else 'of its ' + str(cfg.iters) + ' iterations'}"
              f" in {sec:.1f} s, {threads} threads")
    return rate, threads, sample, kind, n, sec


# ------------------------------------------------------------- b200 arm ----
def bench_b200(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_07189_b200 as cf
    from paper_1903_07189_b200 import sharded

    world, rank, local = dist_env()
    # CF_BENCH_DEVICE (testing only): put every rank on one device, to run the
    # N > 1 code path on a single GPU (timings then mean nothing)
    local = int(os.environ.get("CF_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # ranks sharing a device (CF_BENCH_DEVICE, IPC halo only -- it needs no
    # device collective) use gloo for the few host barriers; NCCL otherwise
    backend = "gloo" if args.halo == "ipc" and "CF_BENCH_DEVICE" in os.environ else "nccl"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    L = cf.lib()
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    # ---------------- inputs (host, pinned) and device buffers ----------------
    # sweeps per launch = the C-ABI filter's schedule for this geometry
    K = int(L.cf_wmc_filter_sweeps_per_launch(cfg.w, cfg.h, cfg.planes))
    if world > 1 and cfg.sharding == "rows":
        # row bands: the step is replayed as one CUDA graph, so launch count
        # costs no host time and the filter's K = 2 stays (N = 8 band:
        # 134 us per 2-sweep launch vs 210 per 3-sweep, tools/probe_shard_host.py)
        lay = sharded.BandLayout(cfg.h, cfg.w, rank, world, K)
        rows = (lay.r0, lay.r1)
    elif world > 1 and cfg.sharding == "images":
        per = (cfg.planes + world - 1) // world
        p0, p1 = rank * per, min(cfg.planes, (rank + 1) * per)
        rows = None
    else:
        rows = None
    # each rank generates only its share, on its share of the host cores
    gen_threads = 0 if world == 1 else max(1, (os.cpu_count() or 1) // world)
    host = make_input(cfg, rows=rows, threads=gen_threads,
                      planes=(p0, p1) if world > 1 and cfg.sharding == "images" else None)
    host_t = torch.from_numpy(np.ascontiguousarray(host)).pin_memory()
    # u8 frames in -> u8 frames out (save-time rounding); f32 otherwise
    out_dtype = torch.uint8 if cfg.u8 else torch.float32
    out_host = torch.empty(host_t.shape, dtype=out_dtype).pin_memory()
    dev_in = host_t.to(dev)
    n_px_local = int(np.prod(host.shape))
    P, H, W = (host.shape if host.ndim == 3 else (1,) + host.shape)
    updates_local = n_px_local * max(1, cfg.iters)
    launches_per_step = 0
    widen_launches = 0  # u8 paths: 1 when a separate widening launch precedes the sweeps

    def cur_sp():  # the current stream (a graph's capture stream while capturing)
        return torch.cuda.current_stream(dev).cuda_stream

    ws = None
    prep = None  # per-step input restore of the in-place paths, run before each step's events
    if cfg.iters == 0:  # single map evaluation (cfg1)
        out = torch.empty(dev_in.shape, dtype=torch.float32, device=dev)

        def step():
            rc = L.cf_wmc_map_f32(dev_in.data_ptr(), out.data_ptr(), W, H, W, P, H * W, cur_sp())
            assert rc == 0, rc
        launches_per_step = 1
    elif world > 1 and cfg.sharding == "rows" and args.halo == "ipc":
        # halo exchange fused into the band kernel (CUDA IPC peer stores)
        flow = sharded.IpcBandFlow(lay, dist, f"cf_bench_{os.environ.get('MASTER_PORT', '0')}")
        band_ptr = flow._row_ptr(flow.bufs[0], lay.buf_row0, lay.r0)
        band_bytes = dev_in.numel() * 4
        ipc_result = [0]

        def prep():  # restore U^0 into the band (outside the timed region)
            assert L.cf_copy(band_ptr, dev_in.data_ptr(), band_bytes, sp) == 0

        def step():
            ipc_result[0] = flow.run(cfg.iters, cfg.dt, stream=sp)
        launches_per_step = len(sharded.launch_schedule(cfg.iters, K))
    elif world > 1 and cfg.sharding == "rows":
        buf_a = torch.zeros((lay.rows, cfg.w), dtype=torch.float32, device=dev)
        buf_b = torch.zeros_like(buf_a)
        flag = torch.full((1,), 0x7F7F7F7F, dtype=torch.int32, device=dev)
        band_fn = sharded.cuda_compute(flag)
        n_band_calls = [0]

        def counted(*a):  # kernel launches per step (boundary + interior band calls)
            n_band_calls[0] += 1
            band_fn(*a)
        flow = sharded.ShardedFlow(lay, counted, dist, side_stream=torch.cuda.Stream(dev))

        def prep():  # restore U^0 into the band (outside the timed region)
            buf_a[lay.band_slice()].copy_(dev_in)

        def step():
            return flow.run(buf_a, buf_b, cfg.iters, cfg.dt)
        prep()
        step()
        launches_per_step = n_band_calls[0]
    else:
        work = torch.empty(dev_in.shape, dtype=torch.float32, device=dev)
        nbytes = int(L.cf_wmc_filter_workspace_bytes(W, H, W, P, H * W))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        # first_bad_iter = NULL: no host sync inside the step (capturable);
        # the device flag is checked once after the timed region.
        if cfg.u8:
            out8 = torch.empty(dev_in.shape, dtype=torch.uint8, device=dev)
            nb8 = int(L.cf_wmc_filter_u8_u8_workspace_bytes(W, H, P))
            ws8 = torch.empty(nb8, dtype=torch.uint8, device=dev)
            f32_bytes = (P * H * W * 4 + 255) // 256 * 256  # the filter workspace follows
            flag_ws = ws8[f32_bytes:]

            def step():
                rc = L.cf_wmc_filter_u8_u8(dev_in.data_ptr(), W, H * W, out8.data_ptr(), W,
                                           H * W, W, H, P, cfg.iters, cfg.dt, ws8.data_ptr(),
                                           nb8, None, cur_sp())
                assert rc == 0, rc
        else:
            def prep():  # the filter is in place: restore U^0 (outside the timed region)
                work.copy_(dev_in)

            def step():
                rc = L.cf_wmc_filter_f32(work.data_ptr(), W, H, W, P, H * W, cfg.iters, cfg.dt,
                                         ws.data_ptr(), nbytes, None, cur_sp())
                assert rc == 0, rc
        # u8: + the widening kernel unless the first sweep reads the bytes
        # itself (the re-quantisation is fused into the last sweep)
        widen_launches = (1 - int(L.cf_wmc_filter_u8_fused(dev_in.data_ptr(), W, H * W, W,
                                                             cfg.iters))) if cfg.u8 else 0
        launches_per_step = int(L.cf_wmc_filter_launches(W, H, P, cfg.iters)) + widen_launches

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # L2 rule: a working set that fits in L2 (126 MB) is flushed between timed
    # steps (a 256 MiB memset, outside the per-step events).
    l2_resident = n_px_local * 4 <= L2_BYTES
    flush_buf = (torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
                 if l2_resident else None)

    def timed(fn, steps):
        """Per-step CUDA events on the launching stream; the in-place paths'
        input restore (prep) and the L2 flush run before each step's start
        event.  Returns (median, mean) ms per step, each the max over ranks
        (the median of the repetitions)."""
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        for e0, e1 in evs:
            if prep is not None:
                prep()
            if flush_buf is not None:
                flush_buf.zero_()
            e0.record(stream)
            fn()
            e1.record(stream)
        barrier()
        per = [e0.elapsed_time(e1) for e0, e1 in evs]
        med, mean = statistics.median(per), sum(per) / steps
        if world > 1:
            t = torch.tensor([med, mean], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            med, mean = (float(v) for v in t.tolist())
        return med, mean

    # ---------------- device-resident timing (value) ----------------
    for _ in range(args.warmup):
        if prep is not None:
            prep()
        step()
    torch.cuda.synchronize(dev)
    run_step = step
    # Host enqueue cost of one eager step (no sync inside: the time the
    # Python / ctypes / NCCL-enqueue loop spends per step), for the N > 1
    # readiness numbers.
    host_ms = None
    if world > 1:
        hs = []
        for _ in range(3):
            if prep is not None:
                prep()
            torch.cuda.synchronize(dev)
            h0 = time.perf_counter()
            step()
            hs.append((time.perf_counter() - h0) * 1e3)
            torch.cuda.synchronize(dev)
        host_ms = statistics.median(hs)
    # One CUDA graph per step: no host launch gaps in the timed region.  At
    # N > 1 (row bands over NCCL) the step's kernels, events and NCCL
    # point-to-point ops are captured too (NCCL >= 2.9.6 is capturable); no
    # NCCL op executes during capture, and every rank replays only if every
    # rank captured (else all run eagerly).  The IPC halo path's host-side
    # ordering (shared-memory counters) cannot be captured.
    graph = world == 1 or (cfg.sharding == "rows" and args.halo == "nccl" and backend == "nccl")
    graph_note = None
    if graph:
        g = torch.cuda.CUDAGraph()
        if prep is not None:
            prep()
        ok = True
        try:
            with torch.cuda.graph(g):
                step()
        except Exception as e:  # capture refused: eager steps
            ok = False
            graph_note = f"capture failed ({type(e).__name__}); eager steps"
        if world > 1:
            t = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = bool(t.item())
            if not ok and graph_note is None:
                graph_note = "a peer rank's capture failed; eager steps"
        graph = ok
        if graph:
            if prep is not None:
                prep()
            g.replay()
            torch.cuda.synchronize(dev)
            run_step = g.replay
        else:
            del g
            torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        ms_step, ms_mean = timed(run_step, args.steps)
    if world > 1 and cfg.sharding == "rows" and args.halo != "ipc":
        assert int(flag.item()) == 0x7F7F7F7F, f"non-finite value in band launch {flag.item()}"
    if ws is not None:  # device non-finite flag of the last timed step
        import ctypes
        bad = ctypes.c_int32(0)
        rc = L.cf_wmc_filter_query_nonfinite((flag_ws if cfg.u8 else ws).data_ptr(),
                                             ctypes.byref(bad), sp)
        assert rc == 0, f"non-finite value in the timed run (iteration {bad.value})"
    # Self-check (no oracle here): the timed output must equal, bit for bit,
    # the same filter run as band launches of a different depth -- another
    # steady-loop instantiation and schedule (any schedule gives the same
    # Jacobi iterates).  f32 single-GPU configs; tests cover the rest.
    selfcheck = None
    if world == 1 and cfg.iters > 0 and not cfg.u8:
        k_alt = 3 if K != 3 else 2
        cur = dev_in.reshape(P, H, W).clone()
        nxt = torch.empty_like(cur)
        it = 0
        for kk in sharded.launch_schedule(cfg.iters, k_alt):
            for pl in range(P):
                cf.sweeps_band(cur[pl], 0, nxt[pl], 0, H, 0, H, kk, cfg.dt, it)
            cur, nxt = nxt, cur
            it += kk
        same = bool(torch.equal(cur.view(torch.int32), work.reshape(P, H, W).view(torch.int32)))
        selfcheck = {"reference": f"band launches of {k_alt} sweeps (no oracle)",
                     "bitwise_equal": same}
        assert same, "self-check failed: the timed output differs from an alternative schedule"
        del cur, nxt
    elif world > 1 and cfg.sharding == "rows" and cfg.iters > 0:
        # N > 1: gather the bands to rank 0 and compare with one GPU's filter
        # of the same input (whatever the halo transport, NCCL or IPC)
        if args.halo == "ipc":
            prep()
            step()
            band = torch.empty((lay.r1 - lay.r0, cfg.w), dtype=torch.float32, device=dev)
            src_ptr = flow._row_ptr(flow.bufs[ipc_result[0]], lay.buf_row0, lay.r0)
            assert L.cf_copy(band.data_ptr(), src_ptr, band.numel() * 4, sp) == 0
        else:
            prep()
            band = step()[lay.band_slice()].clone()
        torch.cuda.synchronize(dev)
        maxr = max(r1 - r0 for r0, r1 in sharded.band_bounds(cfg.h, world))
        pad = torch.zeros((maxr, cfg.w), dtype=torch.float32, device=dev)
        pad[:band.shape[0]] = band
        on = dev if backend == "nccl" else "cpu"
        parts = [torch.empty((maxr, cfg.w), dtype=torch.float32, device=on)
                 for _ in range(world)]
        dist.all_gather(parts, pad.to(on))
        if rank == 0:
            full_in = torch.from_numpy(make_input(cfg)).to(dev)
            ref_out = cf.mc_flow(full_in, cf.FlowConfig(dt=cfg.dt, iters=cfg.iters),
                                 inplace=True, check_finite=False)
            got = torch.cat([parts[q][:r1 - r0].to(dev) for q, (r0, r1)
                             in enumerate(sharded.band_bounds(cfg.h, world))])
            same = bool(torch.equal(got.view(torch.int32), ref_out.view(torch.int32)))
            selfcheck = {"reference": "single-GPU filter of the same input on rank 0 "
                                      "(no oracle)", "bitwise_equal": same}
            assert same, "self-check failed: sharded result differs from the single-GPU filter"
            del full_in, ref_out, got
        del parts, pad, band
    updates_job = cfg.updates  # whole job over all ranks (strong scaling for rows)
    if world > 1 and cfg.sharding == "images":
        updates_job = updates_local * world  # per-rank fixed share (weak scaling)
    value = updates_job / (ms_step * 1e-3) / 1e9

    # ---------------- dominant kernel: average launch duration ----------------
    # Measured live over the timed region: the step is a chain of K-sweep
    # launches of one kernel (u8: the first reads the bytes itself, or one
    # widening launch precedes them), so the kernel's average launch duration
    # is the median step time over the step's sweep launches (inter-launch
    # gaps included, so it can only understate).
    sweep_launches = launches_per_step - (widen_launches if world == 1 else 0)
    kern_ms = ms_step / max(1, sweep_launches)
    alg_bytes_step = algorithmic_bytes(cfg, n_px_local, u8_out=cfg.u8)
    peak, peak_src = peaks()

    # ---------------- end-to-end through the public API, host buffers ----------
    # Every step copies its input from pinned host memory and reads its result
    # back.  Copies run on two copy streams, triple-buffered, so step i's D2H
    # and step i+1's H2D overlap step i+1's / i's compute (a streaming user's
    # pipeline); the filter itself is the public mc_flow / mc_flow_u8 /
    # wmc_half_laplace call on the compute stream.
    pipelined = not (world > 1 and cfg.sharding == "rows")
    if pipelined:
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        # triple-buffered: step i+1's H2D goes to a buffer whose D2H (step
        # i-2) finished long ago, so it overlaps step i's compute entirely
        NB = 3
        dbufs = [torch.empty(host_t.shape, dtype=host_t.dtype, device=dev) for _ in range(NB)]
        obufs = [torch.empty(out_host.shape, dtype=out_dtype, device=dev) for _ in range(NB)]
        ws_e2e = int(L.cf_wmc_filter_u8_u8_workspace_bytes(W, H, P) if cfg.u8 else
                     L.cf_wmc_filter_workspace_bytes(W, H, W, P, H * W))
        flag_off = (P * H * W * 4 + 255) // 256 * 256 if cfg.u8 else 0
        wss = [torch.empty(ws_e2e, dtype=torch.uint8, device=dev) for _ in range(NB)]
        ev_out = [torch.cuda.Event() for _ in range(NB)]
        ev_in = [torch.cuda.Event() for _ in range(NB)]
        ev_c = [torch.cuda.Event() for _ in range(NB)]
        for e in ev_out:
            e.record(s_out)
        flag_host = torch.zeros(NB, dtype=torch.int32).pin_memory()
        e2e_i = [0]
        # copies through cf_copy (cudaMemcpyAsync on an explicit stream) and
        # events created once: the host loop stays cheaper than the GPU step
        # even for cfg1's ~10 us map
        sp_in, sp_out = s_in.cuda_stream, s_out.cuda_stream
        in_bytes = host_t.numel() * host_t.element_size()
        out_bytes = out_host.numel() * out_host.element_size()
        fcfg = cf.FlowConfig(dt=cfg.dt, iters=cfg.iters)

        def e2e_step():
            i = e2e_i[0]
            e2e_i[0] += 1
            b = i % NB
            s_in.wait_event(ev_out[b])               # buffer b's previous D2H done
            assert L.cf_copy(dbufs[b].data_ptr(), host_t.data_ptr(), in_bytes, sp_in) == 0
            ev_in[b].record(s_in)
            stream.wait_event(ev_in[b])
            if cfg.iters == 0:
                L.cf_wmc_map_f32(dbufs[b].data_ptr(), obufs[b].data_ptr(), W, H, W, P, H * W, sp)
                res = obufs[b]
            elif cfg.u8:
                res = cf.mc_flow_u8(dbufs[b], fcfg, workspace=wss[b], out=obufs[b],
                                    check_finite=False, out_dtype="u8")
            else:
                res = cf.mc_flow(dbufs[b], fcfg, workspace=wss[b], inplace=True,
                                 check_finite=False)
            if cfg.iters > 0:  # non-finite flag of this step (device check), read async
                assert L.cf_copy(flag_host[b:b + 1].data_ptr(), wss[b].data_ptr() + flag_off, 4,
                                 sp) == 0
            ev_c[b].record(stream)
            s_out.wait_event(ev_c[b])
            assert L.cf_copy(out_host.data_ptr(), res.data_ptr(), out_bytes, sp_out) == 0
            ev_out[b].record(s_out)
    else:
        # row bands: the band runs in place in the flow's own buffers, so the
        # copies go through device staging buffers (2 each way): step i+1's
        # H2D and step i-1's D2H overlap step i's run
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        band_shape = (lay.r1 - lay.r0, cfg.w)
        st_in = [torch.empty(band_shape, dtype=torch.float32, device=dev) for _ in range(2)]
        st_out = [torch.empty(band_shape, dtype=torch.float32, device=dev) for _ in range(2)]
        ev_in_free = [torch.cuda.Event() for _ in range(2)]   # st_in[b] consumed
        ev_out_done = [torch.cuda.Event() for _ in range(2)]  # st_out[b] read back
        for e in ev_in_free + ev_out_done:
            e.record(stream)
        e2e_i = [0]
        host_band = host_t.reshape(band_shape)

        def e2e_step():
            i = e2e_i[0]
            e2e_i[0] += 1
            b = i % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_in_free[b])
                st_in[b].copy_(host_band, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            stream.wait_event(ev_in)
            if args.halo == "ipc":
                assert L.cf_copy(band_ptr, st_in[b].data_ptr(), band_bytes, sp) == 0
                ev_in_free[b].record(stream)
                which = flow.run(cfg.iters, cfg.dt, stream=sp)
                src = flow._row_ptr(flow.bufs[which], lay.buf_row0, lay.r0)
                stream.wait_event(ev_out_done[b])
                assert L.cf_copy(st_out[b].data_ptr(), src, band_bytes, sp) == 0
            else:
                buf_a[lay.band_slice()].copy_(st_in[b])
                ev_in_free[b].record(stream)
                r = flow.run(buf_a, buf_b, cfg.iters, cfg.dt)[lay.band_slice()]
                stream.wait_event(ev_out_done[b])
                st_out[b].copy_(r)
            ev_c = torch.cuda.Event()
            ev_c.record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_c)
                out_host.copy_(st_out[b].reshape(out_host.shape), non_blocking=True)
                ev_out_done[b].record(s_out)

    def e2e_timed(steps):
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            e2e_step()
        stream.wait_stream(s_out)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(stream)
        barrier()
        ms = t0.elapsed_time(t1)
        if world > 1:
            t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps

    # streaming steady state: enough steps for ~3 s of streaming (at least
    # max(8, K), at most 2000) so the pipeline fill (first H2D) and drain
    # (last D2H) are amortised like in a long-running frame pipeline; the
    # per-step estimate comes from timed warm-up steps
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize(dev)
    est_ms = e2e_timed(2)
    e2e_steps = int(min(2000, max(8, args.steps, math.ceil(3000.0 / max(est_ms, 1e-3)))))
    if world > 1:  # every rank runs the same count
        t = torch.tensor([e2e_steps], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        e2e_steps = int(t.item())
    torch.cuda.synchronize(dev)
    ms_e2e = e2e_timed(e2e_steps)
    torch.cuda.synchronize(dev)
    if pipelined and cfg.iters > 0:
        assert all(int(v) in (0x7F7F7F7F,) or int(v) <= 0 for v in flag_host.tolist()), \
            "non-finite value during the e2e run"
    e2e_value = updates_job / (ms_e2e * 1e-3) / 1e9
    h2d = host_t.numel() * host_t.element_size()
    d2h = out_host.numel() * out_host.element_size()

    if world > 1 and cfg.sharding == "rows" and args.halo == "ipc":
        flow.close()  # collective: neighbours stop writing before unmapping
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    res = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak" if cfg.sharding == "images" else "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded generator, DESIGN.md §6)",
        "config": bench_config(cfg),
        "impl_config": {
            "sweeps_per_launch": 1 if cfg.iters == 0 else K,
            "parallelism": (f"rowband{world}-{args.halo}" if cfg.sharding == "rows" and world > 1 else
                            f"images{world}" if world > 1 else "single"),
            "l2": ("inputs larger than L2 (126 MB)" if not l2_resident else
                   "working set fits in L2: 256 MiB flush between timed steps"),
            "timing": ("one CUDA graph per step; CUDA events per step on the launching stream; "
                       "median of the steps" + (", max over ranks" if world > 1 else "") if graph else
                       "CUDA events per step on the launching stream; median of the steps, "
                       "max over ranks") + ("; the in-place filter's input restore runs "
                                            "before each step's start event" if prep else ""),
            "ms_per_step_mean": round(ms_mean, 4),
            **({"host_enqueue_ms_per_step_eager": round(host_ms, 3),
                "host_enqueue_ms_per_launch_eager": round(host_ms / max(1, launches_per_step), 4),
                "gpu_ms_per_launch": round(ms_step / max(1, launches_per_step), 4)}
               if host_ms is not None else {}),
            **({"graph": graph_note} if graph_note else {}),
        },
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4), "steps": e2e_steps,
                "pipeline": ("H2D/D2H from pinned host memory every step on two copy streams, "
                             "triple-buffered against the compute stream; steady state over "
                             "~3 s of streaming" if pipelined else
                             "H2D/D2H of each rank's band on two copy streams through "
                             "double-buffered device staging")},
        "gpu_launches": launches_per_step * args.steps,
        "selfcheck": selfcheck,
        "clocks": clk.summary(),
    }
    achieved = alg_bytes_step / (ms_step * 1e-3) / 1e9
    kname = (f"wmc_sweeps_kernel<K={K}>" if cfg.iters else "wmc_map_kernel")
    res["roofline"] = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": ncu_traffic(kname, H, W, P),
        "kernel": kname + ((" (first launch reads u8)" if not widen_launches else
                            " (+1 u8 widening launch)") if cfg.u8 and cfg.iters else ""),
        "kernel_ms": round(kern_ms, 4), "launches_per_step": sweep_launches,
        "algorithmic_bytes_per_step": alg_bytes_step,
        "ncu_launch_ms": ncu_launch_ms(kname, H, W, P),
        "peak_source": peak_src,
        "note": "achieved = algorithmic bytes of the step (8 B per pixel-update, SURVEY.md "
                "§8d) / the median step time of the timed region; kernel_ms = that step "
                "time / the sweep launches of the step; traffic = physical DRAM bytes per "
                "launch from the committed ncu --set full capture, ncu_launch_ms its "
                "cold-cache duration",
    }
    assert kern_ms * sweep_launches <= ms_step * 1.0001
    if world == 1 and not args.no_cpu_baseline:
        import numpy as np
        plane0 = host[0] if host.ndim == 3 else host
        img64 = plane0.astype(np.float64) / 255.0 if cfg.u8 else plane0.astype(np.float64)
        rate, cores, sample, kind, _, _ = cpu_reference_sample(cfg, img64)
        res["cpu_baseline"] = {"value": round(rate, 4), "unit": UNIT, "cores": cores,
                               "kind": kind, "sample": sample}
    if world > 1:
        dist.destroy_process_group()
    return res



# ------------------------------------------------------- fp64 b200 arm ----
def bench_b200_f64(args, cfg):
    """--precision fp64 (N = 1): the SPEC-faithful fp64 path (DESIGN.md §3.6,
    bit-identical to the reference CPU path) on the same workload: fp64
    images (u8 input widened on device as q / 255.0), one CUDA graph per
    step, median step; e2e through the public API with host buffers."""
    import numpy as np
    import torch

    import paper_1903_07189_b200 as cf
    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("--precision fp64 is a single-GPU line")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = cf.lib()
    stream = torch.cuda.current_stream(dev)
    host = make_input(cfg)
    if not cfg.u8:
        host = host.astype(np.float64)
    host_t = torch.from_numpy(np.ascontiguousarray(host)).pin_memory()
    dev_in = host_t.to(dev)
    P, H, W = (host.shape if host.ndim == 3 else (1,) + host.shape)
    n_px = P * H * W
    out = torch.empty((P, H, W), dtype=torch.float64, device=dev)
    nb = int(L.cf_wmc_filter_f64_workspace_bytes(W, H, W, P, H * W))
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
    cur = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
    prep = None
    if cfg.iters == 0:
        def step():
            assert L.cf_wmc_map_f64(dev_in.data_ptr(), out.data_ptr(), W, H, W, P, H * W,
                                    cur()) == 0
        launches = 1
    elif cfg.u8:
        def step():
            assert L.cf_wmc_filter_u8_f64(dev_in.data_ptr(), W, H * W, out.data_ptr(), W, H, W, P,
                                          H * W, cfg.iters, cfg.dt, ws.data_ptr(), nb, None,
                                          cur()) == 0
        launches = cfg.iters + 1
    else:
        def prep():
            out.copy_(dev_in.reshape(out.shape))

        def step():
            assert L.cf_wmc_filter_f64(out.data_ptr(), W, H, W, P, H * W, cfg.iters, cfg.dt,
                                       ws.data_ptr(), nb, None, cur()) == 0
        launches = cfg.iters
    l2_resident = n_px * 8 <= L2_BYTES
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if l2_resident else None
    for _ in range(args.warmup):
        if prep:
            prep()
        step()
    g = torch.cuda.CUDAGraph()
    if prep:
        prep()
    with torch.cuda.graph(g):
        step()
    torch.cuda.synchronize(dev)
    per = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if prep:
                prep()
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            per.append(e0.elapsed_time(e1))
    ms = statistics.median(per)
    if cfg.iters:
        import ctypes
        bad = ctypes.c_int32(0)
        assert L.cf_wmc_filter_f64_query_nonfinite(ws.data_ptr(), ctypes.byref(bad),
                                                   stream.cuda_stream) == 0, bad.value
    updates = n_px * max(1, cfg.iters)
    value = updates / (ms * 1e-3) / 1e9
    # e2e: host input -> device -> public call -> host output, serial steps
    out_host = torch.empty((P, H, W), dtype=torch.float64).pin_memory()
    fcfg = cf.FlowConfig(dt=cfg.dt, iters=cfg.iters)

    def e2e_step():
        d_in = host_t.to(dev, non_blocking=True)
        if cfg.iters == 0:
            r = cf.wmc_half_laplace(d_in, precision="fp64")
        elif cfg.u8:
            r = cf.mc_flow_u8(d_in, fcfg, out=out, workspace=ws, out_dtype="f64",
                              check_finite=False)
        else:
            r = cf.mc_flow(d_in, fcfg, inplace=True, workspace=ws, check_finite=False)
        out_host.copy_(r.reshape(out_host.shape), non_blocking=True)
    e2e_step()
    torch.cuda.synchronize(dev)
    n_e2e = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n_e2e):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_e2e = e0.elapsed_time(e1) / n_e2e
    alg = (n_px * 16 * max(1, cfg.iters) if not cfg.u8 else
           n_px * ((1 + 8) + (cfg.iters - 1) * 16))
    peak, peak_src = peaks()
    achieved = alg / (ms * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak" if cfg.sharding == "images" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, DESIGN.md §6)",
        "config": bench_config(cfg),
        "impl_config": {"precision": "fp64 SPEC-faithful (bit-identical to the reference CPU "
                                     "path, DESIGN.md §3.6)",
                        "timing": "one CUDA graph per step, CUDA events, median of the steps",
                        "l2": ("working set fits in L2: 256 MiB flush between timed steps"
                               if l2_resident else "inputs larger than L2")},
        "e2e": {"value": round(updates / (ms_e2e * 1e-3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": host_t.numel() * host_t.element_size(),
                "d2h_bytes_per_step": out_host.numel() * 8, "ms_per_step": round(ms_e2e, 4),
                "pipeline": "serial H2D, call, D2H per step (pinned host buffers)"},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": "wmc_f64_kernel", "kernel_ms": round(ms / launches, 4),
                     "peak_source": peak_src,
                     "note": "16 B per fp64 pixel-update (8 B read + 8 B write); the kernel is "
                             "FP64-pipe bound, not HBM bound (DESIGN.md §3.6)"},
    }

# -------------------------------------------------------- reference arm ----
def bench_reference(args, cfg):
    """The reference arm: the reference's CPU path (fp64 SPEC-faithful mc_flow
    on the reference's own parallel::for_rows executor, oracle/_ref) on all
    host threads, on the same workload -- the full-size first plane of the
    config's seeded input, generated on the CPU by oracle/synth_ref.c (no
    product library is loaded on this arm).  One step = n of the workload's
    iterations on that image, n sized so the whole run stays within a few
    minutes."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    import numpy as np

    import oracle
    threads = os.cpu_count() or 1
    flow, wmap, kind, what = cpu_reference(threads)
    plane0 = oracle.synth(cfg.w, cfg.h, cfg.seed(0), cfg.n_rects, cfg.n_discs, cfg.sigma,
                          u8=cfg.u8, threads=threads)
    img = plane0.astype(np.float64) / 255.0 if cfg.u8 else plane0.astype(np.float64)
    del plane0

    def run(n):
        if cfg.iters == 0:
            for _ in range(n):
                wmap(img)
        else:
            flow(img, n, cfg.dt)
    t0 = time.perf_counter()
    run(1)
    one = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)  # whole run ~2.5 min of CPU work
    n_it = max(1, min(cfg.iters or 50, int(budget / max(one, 1e-6))))
    for _ in range(args.warmup):
        run(n_it)
    per = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run(n_it)
        per.append(time.perf_counter() - t0)
    sec = statistics.median(per)
    rate = cfg.h * cfg.w * n_it / sec / 1e9
    desc = (f"{what}; {'wmc_half_laplace' if cfg.iters == 0 else 'mc_flow'} on the full "
            f"{cfg.h}x{cfg.w} first plane of the {cfg.name} input (oracle/synth_ref.c), "
            f"{n_it} {'evaluation(s)' if cfg.iters == 0 else 'of its ' + str(cfg.iters) + ' iterations'}"
            f" per step, median of {args.steps} steps, {threads} threads")
    return {
        "impl": "reference", "metric": METRIC, "value": round(rate, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak" if cfg.sharding == "images" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, DESIGN.md §6)",
        "config": bench_config(cfg),
        "impl_config": {"parallelism": f"cpu{threads}",
                        "sample": f"{n_it} iteration(s) of the full first plane per step"},
        "cpu_baseline": {"value": round(rate, 4), "unit": UNIT, "cores": threads,
                         "kind": kind, "sample": desc},
        "e2e": {"value": round(rate, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--all", default=None, help="run every config (+ the supplemental 16384^2 "
                    "map) at N=1, write JSON lines")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="fp64: the SPEC-faithful fp64 path, bit-identical to the reference "
                         "CPU path (single GPU)")
    ap.add_argument("--halo", default="nccl", choices=["nccl", "ipc"],
                    help="row-band halo exchange at N > 1: NCCL send/recv overlapped with the "
                         "band interior (default) or fused into the band kernel's stores over "
                         "CUDA IPC peer memory")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    CONFIGS, SUPPLEMENTAL = load_configs()
    if args.all:
        with open(args.all, "w") as f:
            for name, c in list(CONFIGS.items()) + list(SUPPLEMENTAL.items()):
                r = bench_b200(args, c)
                if r:
                    f.write(json.dumps(r) + "\n")
                    f.flush()
                    print(json.dumps(r), flush=True)
        return
    cfg = {**CONFIGS, **SUPPLEMENTAL}[args.workload]
    if args.impl == "reference":
        res = bench_reference(args, cfg)
    elif args.precision == "fp64":
        res = bench_b200_f64(args, cfg)
    else:
        res = bench_b200(args, cfg)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

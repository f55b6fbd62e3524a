"""Row-band sharded WMC flow across ranks (BASELINE cfg 4: one huge image).

One process per GPU.  The image's rows are split like the reference's
``curveflow::parallel::for_rows`` (contiguous ceil-div blocks,
proj/include/curveflow/parallel.hpp:36-44); each rank owns one band and keeps
``k`` halo rows above and below it.  Each launch of ``kk <= k`` fused sweeps
needs the ``kk`` boundary rows of the current iterate from the neighbours
(point-to-point over NCCL / NVLink; gloo in the CPU tests); each rank
advances its band with the row-band kernel (C-ABI
``cf_wmc_sweeps_band_f32``), computing the rows its neighbours need first so
the exchange overlaps the band interior (ShardedFlow, overlap=True).  Jacobi semantics make the result
bit-identical to the single-GPU filter for any band count.

The compute step is injected, so the exchange protocol is the same code in
the GPU bench (CUDA kernel) and in the CPU tests (oracle compute over gloo).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Tuple


def band_bounds(h: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous ceil-div row blocks (parallel.hpp:36-44); one per rank."""
    if world < 1 or h < world:
        raise ValueError(f"cannot split {h} rows over {world} ranks")
    chunk = (h + world - 1) // world
    bands = []
    for p in range(world):
        r0, r1 = min(h, p * chunk), min(h, (p + 1) * chunk)
        if r0 >= r1:
            raise ValueError(f"rank {p} would own no rows (h={h}, world={world})")
        bands.append((r0, r1))
    return bands


def launch_schedule(iters: int, k: int) -> List[int]:
    """Sweeps per launch: chunks of k, remainder last."""
    ks, left = [], iters
    while left > 0:
        ks.append(min(k, left))
        left -= ks[-1]
    return ks


# compute(src, src_row0, dst, dst_row0, h, y0, y1, sweeps, dt, iter_base)
ComputeFn = Callable[..., None]


@dataclass
class BandLayout:
    h: int
    w: int
    rank: int
    world: int
    k: int

    def __post_init__(self):
        self.r0, self.r1 = band_bounds(self.h, self.world)[self.rank]
        if self.r1 - self.r0 < self.k and self.world > 1:
            raise ValueError("band height must be >= sweeps per launch")
        self.top = self.k if self.rank > 0 else 0
        self.bot = self.k if self.rank < self.world - 1 else 0
        self.rows = self.top + (self.r1 - self.r0) + self.bot
        self.buf_row0 = self.r0 - self.top  # global row of buffer row 0

    def band_slice(self):
        return slice(self.top, self.top + self.r1 - self.r0)


class ShardedFlow:
    """Sharded mc_flow over a band buffer pair (torch tensors, any device).

    overlap=True (default): each launch first computes the rows the
    neighbours will need for the NEXT launch (the band's top / bottom kk'
    rows), starts the halo exchange of those rows, and computes the band
    interior meanwhile -- on `side_stream` when given (CUDA), so the
    point-to-point transfer hides behind the interior sweep.  The rows each
    call produces are disjoint and all read the same iterate, so the result is
    bit-identical to overlap=False (exchange, then one band launch).
    """

    def __init__(self, layout: BandLayout, compute: ComputeFn, dist, group=None,
                 overlap: bool = True, side_stream=None):
        self.L = layout
        self.compute = compute
        self.dist = dist
        self.group = group
        self.overlap = overlap
        self.side = side_stream

    def _ops(self, buf, kk: int):
        L, dist = self.L, self.dist
        ops = []
        b0, b1 = L.top, L.top + (L.r1 - L.r0)
        if L.rank > 0:
            ops.append(dist.P2POp(dist.isend, buf[b0:b0 + kk], L.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[b0 - kk:b0], L.rank - 1, self.group))
        if L.rank < L.world - 1:
            ops.append(dist.P2POp(dist.isend, buf[b1 - kk:b1], L.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[b1:b1 + kk], L.rank + 1, self.group))
        return ops

    def exchange(self, buf, kk: int) -> None:
        """Fill the kk halo rows nearest the band from the neighbours' bands."""
        ops = self._ops(buf, kk)
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def _band(self, cur, nxt, y0: int, y1: int, kk: int, dt: float, it: int) -> None:
        if y1 > y0:
            L = self.L
            self.compute(cur, L.buf_row0, nxt, L.buf_row0, L.h, y0, y1, kk, dt, it)

    def run(self, buf_a, buf_b, iters: int, dt: float):
        """buf_a holds U^0 in its band rows; returns the buffer holding U^iters."""
        L = self.L
        cur, nxt = buf_a, buf_b
        sched = launch_schedule(iters, L.k)
        if not sched:
            return cur
        self.exchange(cur, sched[0])
        it = 0
        for i, kk in enumerate(sched):
            nk = sched[i + 1] if i + 1 < len(sched) else 0
            # src covers [max(0, r0-kk), min(h, r1+kk)); dst rows [r0, r1)
            if not self.overlap or nk == 0 or L.world == 1:
                self._band(cur, nxt, L.r0, L.r1, kk, dt, it)
                if nk:
                    self.exchange(nxt, nk)
            else:
                top = nk if L.rank > 0 else 0
                bot = nk if L.rank < L.world - 1 else 0
                # rows the neighbours need next (clipped to the band)
                t1 = min(L.r0 + top, L.r1)
                b0 = max(L.r1 - bot, t1)
                ready = self._mark()              # cur (with its halo) is final here
                self._band(cur, nxt, L.r0, t1, kk, dt, it)
                self._band(cur, nxt, b0, L.r1, kk, dt, it)
                reqs = self.dist.batch_isend_irecv(self._ops(nxt, nk))
                self._interior(cur, nxt, t1, b0, kk, dt, it, ready)
                for req in reqs:
                    req.wait()
                self._join()
            it += kk
            cur, nxt = nxt, cur
        return cur

    def _mark(self):
        if self.side is None:
            return None
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.side.device))
        return ev

    def _interior(self, cur, nxt, y0: int, y1: int, kk: int, dt: float, it: int,
                  ready=None) -> None:
        if self.side is None:
            self._band(cur, nxt, y0, y1, kk, dt, it)
            return
        import torch
        self.side.wait_event(ready)   # not the boundary kernels: their rows are disjoint
        with torch.cuda.stream(self.side):
            self._band(cur, nxt, y0, y1, kk, dt, it)

    def _join(self) -> None:
        if self.side is not None:
            import torch
            torch.cuda.current_stream(self.side.device).wait_stream(self.side)


def cuda_compute(flag=None) -> ComputeFn:
    """Row-band kernel through the C-ABI (cf_wmc_sweeps_band_f32), on the
    caller's current stream; a lean ctypes call (the sharded loop issues a
    few of these per launch, so host cost per call matters at N = 8)."""
    import torch

    from ._lib import check, lib
    fn_c = lib().cf_wmc_sweeps_band_f32
    flag_ptr = flag.data_ptr() if flag is not None else None

    def fn(src, src_row0, dst, dst_row0, h, y0, y1, sweeps, dt, iter_base):
        W = src.shape[1]
        check(fn_c(src.data_ptr(), src_row0, src.shape[0], dst.data_ptr(), dst_row0, W, h, W, y0,
                   y1, sweeps, float(dt), iter_base, flag_ptr,
                   torch.cuda.current_stream().cuda_stream), "sweeps_band")
    return fn


def plan(h: int, w: int, parts: int, k: int):
    """cf_shard_plan for the single-process sharded filter (C-ABI)."""
    import ctypes as C

    from ._lib import CfShardPlan, check, lib
    pl = CfShardPlan()
    check(lib().cf_shard_plan_init(h, w, parts, k, C.addressof(pl)), "cf_shard_plan_init")
    return pl


def filter_sharded(img, iters: int, dt: float = 1.0, parts: int = 2, devices=None, k=None,
                   check_finite: bool = True):
    """mc_flow of one image split into `parts` row bands on `devices` (one
    process; cf_wmc_filter_sharded_f32: halos over cudaMemcpyPeerAsync).
    img: (H, W) float32 torch tensor or numpy array; returns a tensor on the
    first device (numpy for numpy input)."""
    import ctypes as C

    import numpy as np
    import torch

    from ._lib import CF_ENONFINITE, check, lib
    from .curveflow import FlowError
    host = isinstance(img, np.ndarray)
    x = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)) if host else img
    H, W = x.shape
    devices = list(devices) if devices is not None else [torch.cuda.current_device()] * parts
    if len(devices) != parts:
        raise ValueError("one device per part")
    k = int(k) if k is not None else int(lib().cf_wmc_filter_sweeps_per_launch(W, H, 1))
    pl = plan(H, W, parts, k)
    bufs_a, bufs_b, flags, streams = [], [], [], []
    for p in range(parts):
        dev = torch.device("cuda", devices[p])
        a = torch.zeros((pl.rows[p], W), dtype=torch.float32, device=dev)
        a[pl.top[p]:pl.top[p] + pl.row1[p] - pl.row0[p]] = x[pl.row0[p]:pl.row1[p]].to(dev)
        bufs_a.append(a)
        bufs_b.append(torch.empty_like(a))
        flags.append(torch.empty(1, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.current_stream(dev))
    arr = lambda xs: (C.c_void_p * parts)(*[t.data_ptr() for t in xs])  # noqa: E731
    pa, pb, pf = arr(bufs_a), arr(bufs_b), arr(flags)
    pd = (C.c_int32 * parts)(*devices)
    ps = (C.c_void_p * parts)(*[s.cuda_stream for s in streams])
    bad = C.c_int32(0)
    rc = lib().cf_wmc_filter_sharded_f32(C.addressof(pl), C.addressof(pa), C.addressof(pb),
                                         C.addressof(pf), C.addressof(pd), C.addressof(ps),
                                         int(iters), float(dt),
                                         C.byref(bad) if check_finite else None)
    if rc == CF_ENONFINITE:
        raise FlowError(bad.value)
    check(rc, "filter_sharded")
    out = torch.empty((H, W), dtype=torch.float32, device=torch.device("cuda", devices[0]))
    for p in range(parts):
        band = bufs_a[p][pl.top[p]:pl.top[p] + pl.row1[p] - pl.row0[p]]
        out[pl.row0[p]:pl.row1[p]] = band.to(out.device)
    return out.cpu().numpy() if host else out



class IpcBandFlow:
    """Row-band flow across processes with the halo exchange FUSED into the
    band kernel: each rank's launch stores the boundary rows
    its neighbours need next straight into their buffers (CUDA IPC peer
    memory; NVLink between GPUs) via cf_wmc_sweeps_band_peer_f32.  No
    collective runs per launch: ordering is interprocess CUDA events plus a
    launch counter per rank in POSIX shared memory (a rank waits on a
    neighbour's event only after the counter shows it was recorded), and
    `dist` is used once, to exchange the IPC handles.  No kernel waits on
    another, so ranks may share one GPU (the tests do).

    Launch i of rank p reads bufs[i % 2] (its band + halos) and writes
    bufs[(i+1) % 2]; it waits first for both neighbours' launch i-1 (they
    wrote its halos, and it is about to overwrite theirs in the buffer their
    launch i-1 read)."""

    RING = 4  # events per rank; neighbours lag by at most 2 sequence numbers
    WAIT_S = 300.0  # a neighbour silent this long has died: raise instead of hanging

    def __init__(self, layout: BandLayout, dist, shm_name: str, group=None):
        import ctypes as C

        import numpy as np
        from multiprocessing import shared_memory

        from ._lib import check, lib
        self.L, self.C, self.np = layout, C, np
        L, self._lib = layout, lib()
        self._check = check
        self.w = L.w
        self.row_bytes = L.w * 4
        self.bufs, self.events = [], []
        for _ in range(2):
            p = C.c_void_p()
            check(self._lib.cf_device_alloc(L.rows * self.row_bytes, C.byref(p)), "alloc")
            self.bufs.append(p.value)
        flag = C.c_void_p()
        check(self._lib.cf_device_alloc(256, C.byref(flag)), "alloc flag")
        self.flag = flag.value
        for _ in range(self.RING):
            e = C.c_void_p()
            check(self._lib.cf_ipc_event_create(C.byref(e)), "ipc event")
            self.events.append(e.value)

        def handle(fn, obj):
            buf = C.create_string_buffer(64)
            check(fn(obj, buf), "ipc handle")
            return buf.raw
        mine = {"rank": L.rank, "r0": L.r0, "r1": L.r1, "buf_row0": L.buf_row0,
                "mem": [handle(self._lib.cf_ipc_mem_handle, b) for b in self.bufs],
                "ev": [handle(self._lib.cf_ipc_event_handle, e) for e in self.events]}
        everyone = [None] * L.world
        dist.all_gather_object(everyone, mine, group=group)
        self.nbr = {}
        for side, q in (("up", L.rank - 1), ("dn", L.rank + 1)):
            if 0 <= q < L.world:
                o = everyone[q]
                mem = []
                for hb in o["mem"]:
                    p = C.c_void_p()
                    check(self._lib.cf_ipc_open_mem(hb, C.byref(p)), "ipc open mem")
                    mem.append(p.value)
                ev = []
                for hb in o["ev"]:
                    e = C.c_void_p()
                    check(self._lib.cf_ipc_open_event(hb, C.byref(e)), "ipc open event")
                    ev.append(e.value)
                self.nbr[side] = {"rank": q, "buf_row0": o["buf_row0"], "mem": mem, "ev": ev}
        if L.rank == 0:
            self.shm = shared_memory.SharedMemory(name=shm_name, create=True, size=8 * L.world)
        dist.barrier(group=group)
        if L.rank != 0:
            self.shm = shared_memory.SharedMemory(name=shm_name)
        self.count = np.ndarray((L.world,), dtype=np.int64, buffer=self.shm.buf)
        self.count[L.rank] = -1
        dist.barrier(group=group)
        self.dist, self.group = dist, group
        self.seq = 0  # launches are numbered across runs (counters only grow)
        self.stream = None  # the stream of the last run (read / close order after it)

    def _row_ptr(self, base: int, buf_row0: int, y: int) -> int:
        return base + (y - buf_row0) * self.row_bytes

    def load(self, band) -> None:
        """Place the owned rows (host float32, (r1 - r0) x w) into bufs[0]."""
        arr = self.np.ascontiguousarray(band, dtype=self.np.float32)
        L = self.L
        # the previous run's launches (on its own stream) still read bufs[0]
        self._check(self._lib.cf_stream_synchronize(self.stream), "sync")
        self._check(self._lib.cf_copy(self._row_ptr(self.bufs[0], L.buf_row0, L.r0),
                                      arr.ctypes.data, arr.nbytes, None), "load")
        self._check(self._lib.cf_stream_synchronize(None), "sync")

    def _wait(self, i: int, stream) -> None:
        import time
        for side in ("up", "dn"):
            if side in self.nbr:
                q = self.nbr[side]
                deadline = None
                while self.count[q["rank"]] < i:
                    now = time.monotonic()
                    if deadline is None:
                        deadline = now + self.WAIT_S
                    elif now > deadline:
                        raise RuntimeError(f"IpcBandFlow: rank {q['rank']} did not publish "
                                           f"launch {i} within {self.WAIT_S:.0f} s")
                    time.sleep(0)
                self._check(self._lib.cf_stream_wait_event(stream, q["ev"][i % self.RING]),
                            "wait event")

    def _publish(self, i: int, stream) -> None:
        self._check(self._lib.cf_event_record(self.events[i % self.RING], stream), "record")
        self.count[self.L.rank] = i

    def run(self, iters: int, dt: float, stream=None) -> int:
        """Advance iters Jacobi sweeps from bufs[0]; returns the index of the
        result buffer.  Runs may follow each other without a barrier: each
        run first waits for the neighbours' last launch of the previous one
        (their halo reads end before this run's initial fill overwrites them)."""
        L, lib = self.L, self._lib
        sched = launch_schedule(iters, L.k)
        self.stream = stream
        if not sched:
            return 0
        # the band kernels atomicMin the first bad iteration into the flag
        self._check(lib.cf_device_memset(self.flag, 0x7F, 4, stream), "flag reset")
        base = self.seq
        if base > 0:
            self._wait(base, stream)
        kk0 = sched[0]
        # initial halo fill: our boundary rows into the neighbours' bufs[0]
        for side, rows in (("up", (L.r0, L.r0 + kk0)), ("dn", (L.r1 - kk0, L.r1))):
            if side in self.nbr:
                q = self.nbr[side]
                self._check(lib.cf_copy(self._row_ptr(q["mem"][0], q["buf_row0"], rows[0]),
                                        self._row_ptr(self.bufs[0], L.buf_row0, rows[0]),
                                        (rows[1] - rows[0]) * self.row_bytes, stream), "halo")
        self._publish(base + 1, stream)
        it = 0
        for i, kk in enumerate(sched):
            self._wait(base + 1 + i, stream)
            nk = sched[i + 1] if i + 1 < len(sched) else 0
            src, dst = self.bufs[i % 2], self.bufs[(i + 1) % 2]
            up, dn = self.nbr.get("up"), self.nbr.get("dn")
            rc = lib.cf_wmc_sweeps_band_peer_f32(
                src, L.buf_row0, L.rows, dst, L.buf_row0, L.w, L.h, L.w, L.r0, L.r1, kk,
                float(dt), it, self.flag,
                up["mem"][(i + 1) % 2] if up and nk else None,
                up["buf_row0"] if up else 0, L.r0 + nk,
                dn["mem"][(i + 1) % 2] if dn and nk else None,
                dn["buf_row0"] if dn else 0, L.r1 - nk, stream)
            self._check(rc, "band launch")
            self._publish(base + 2 + i, stream)
            it += kk
        self.seq = base + 1 + len(sched)
        return len(sched) % 2

    def first_bad_iteration(self) -> int:
        """Collective: the first iteration (1-based) whose iterate held a
        non-finite value on ANY rank's band, 0 if none.
        Synchronises the run stream."""
        import torch
        bad = self.C.c_int32(0)
        rc = self._lib.cf_wmc_filter_query_nonfinite(self.flag, self.C.byref(bad), self.stream)
        if rc not in (0, 3):
            self._check(rc, "query flag")
        v = torch.tensor([bad.value if bad.value > 0 else 2**31 - 1], dtype=torch.int64)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN, group=self.group)
        return 0 if int(v.item()) == 2**31 - 1 else int(v.item())

    def check_finite(self) -> None:
        """Collective: raise FlowError naming the first bad iteration."""
        from .curveflow import FlowError
        bad = self.first_bad_iteration()
        if bad:
            raise FlowError(bad)

    def read(self, which: int):
        """The owned rows of bufs[which] (host float32)."""
        L = self.L
        out = self.np.empty((L.r1 - L.r0, L.w), dtype=self.np.float32)
        self._check(self._lib.cf_stream_synchronize(self.stream), "sync")
        self._check(self._lib.cf_stream_synchronize(None), "sync")
        self._check(self._lib.cf_copy(out.ctypes.data,
                                      self._row_ptr(self.bufs[which], L.buf_row0, L.r0),
                                      out.nbytes, None), "read")
        self._check(self._lib.cf_stream_synchronize(None), "sync")
        return out

    def close(self) -> None:
        """Collective: every rank must call it (neighbours stop writing first)."""
        self._check(self._lib.cf_stream_synchronize(self.stream), "sync")
        self._check(self._lib.cf_stream_synchronize(None), "sync")
        self.dist.barrier(group=self.group)
        for q in self.nbr.values():
            for p in q["mem"]:
                self._lib.cf_ipc_close_mem(p)
            for e in q["ev"]:
                self._lib.cf_event_destroy(e)
        for e in self.events:
            self._lib.cf_event_destroy(e)
        for b in self.bufs:
            self._lib.cf_device_free(b)
        self._lib.cf_device_free(self.flag)
        self.shm.close()
        self.dist.barrier(group=self.group)
        if self.L.rank == 0:
            self.shm.unlink()

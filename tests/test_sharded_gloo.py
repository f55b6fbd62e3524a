"""N>1 row-band sharding on CPU: world_size 2 and 3 over gloo, with the oracle
as the per-band compute (test-only); result must equal the single-process
oracle flow bit-for-bit (SPEC.md:82 determinism across decompositions)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1903_07189_b200.sharded import BandLayout, ShardedFlow, band_bounds, launch_schedule


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_compute(src, src_row0, dst, dst_row0, h, y0, y1, sweeps, dt, iter_base):
    # rows [max(0,y0-sweeps), min(h,y1+sweeps)) of the current iterate
    a0, a1 = max(0, y0 - sweeps), min(h, y1 + sweeps)
    sub = src[a0 - src_row0:a1 - src_row0].numpy()
    out, bad = oracle.flow_f32(sub, sweeps, dt)
    assert bad == 0
    dst[y0 - dst_row0:y1 - dst_row0] = torch.from_numpy(out[y0 - a0:y1 - a0].copy())


def _worker(rank, world, port, img, iters, k, q, overlap=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, w = img.shape
        L = BandLayout(h, w, rank, world, k)
        a = torch.zeros((L.rows, w), dtype=torch.float32)
        b = torch.zeros_like(a)
        a[L.band_slice()] = torch.from_numpy(img[L.r0:L.r1])
        out = ShardedFlow(L, oracle_compute, dist, overlap=overlap).run(a, b, iters, 1.0)
        q.put((rank, L.r0, L.r1, out[L.band_slice()].numpy().copy()))
    finally:
        dist.destroy_process_group()


def run_sharded(img, world, iters, k, overlap=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, iters, k, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = np.empty_like(img)
    for _, r0, r1, band in parts:
        out[r0:r1] = band
    return out


def test_band_bounds_match_for_rows():
    # parallel.hpp:36 chunk = ceil(h / workers)
    assert band_bounds(10, 4) == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert band_bounds(16384, 8)[3] == (6144, 8192)
    with pytest.raises(ValueError):
        band_bounds(3, 4)


def test_launch_schedule():
    assert launch_schedule(7, 2) == [2, 2, 2, 1]
    assert sum(launch_schedule(200, 4)) == 200


@pytest.mark.parametrize("world,k,iters,overlap", [(2, 2, 7, True), (3, 3, 8, True),
                                                   (2, 4, 4, True), (2, 2, 7, False),
                                                   (3, 3, 8, False)])
def test_sharded_equals_single(world, k, iters, overlap):
    import paper_1903_07189_b200 as cf
    img = cf.synth_image(41, 37, seed=5, n_rects=3, n_discs=3, sigma=0.1)
    ref, _ = oracle.flow_f32(img, iters, 1.0)
    got = run_sharded(img, world, iters, k, overlap)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_sharded_thin_bands_overlap():
    """Bands thinner than two halos (12 rows over 3 ranks, k = 3): the
    boundary computations cover the whole band, the interior is empty."""
    import paper_1903_07189_b200 as cf
    img = cf.synth_image(12, 29, seed=9, n_rects=2, n_discs=2, sigma=0.1)
    ref, _ = oracle.flow_f32(img, 10, 1.0)
    got = run_sharded(img, 3, 10, 3, True)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


class _RecordingDist:
    """Single-process stand-in for torch.distributed: records P2P ops."""

    def __init__(self):
        self.batches = []
        self.isend, self.irecv = "send", "recv"

    def P2POp(self, op, t, peer, group=None):
        return (op, t.shape[0], peer)

    def batch_isend_irecv(self, ops):
        self.batches.append(ops)
        return []


def test_overlap_schedule_covers_band_once():
    """Every launch computes each band row exactly once, the rows sent to the
    neighbours are computed before the exchange, halos are nk rows."""
    calls = []

    def rec(src, src_row0, dst, dst_row0, h, y0, y1, sweeps, dt, it):
        calls.append((it, y0, y1, sweeps))
    L = BandLayout(100, 8, 1, 3, 3)          # middle rank: rows [34, 68)
    d = _RecordingDist()
    a = torch.zeros((L.rows, 8))
    ShardedFlow(L, rec, d).run(a, torch.zeros_like(a), 10, 1.0)
    sched = launch_schedule(10, 3)
    its = [sum(sched[:i]) for i in range(len(sched))]
    for i, it in enumerate(its):
        rows = sorted((y0, y1) for (c_it, y0, y1, _) in calls if c_it == it)
        covered = [y for y0, y1 in rows for y in range(y0, y1)]
        assert covered == list(range(L.r0, L.r1)), (it, rows)
    # one initial exchange + one per launch but the last; halo widths follow the schedule
    assert len(d.batches) == len(sched)
    assert [b[0][1] for b in d.batches] == sched

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


def _worker(rank, world, port, img, iters, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, w = img.shape
        L = BandLayout(h, w, rank, world, k)
        a = torch.zeros((L.rows, w), dtype=torch.float32)
        b = torch.zeros_like(a)
        a[L.band_slice()] = torch.from_numpy(img[L.r0:L.r1])
        out = ShardedFlow(L, oracle_compute, dist).run(a, b, iters, 1.0)
        q.put((rank, L.r0, L.r1, out[L.band_slice()].numpy().copy()))
    finally:
        dist.destroy_process_group()


def run_sharded(img, world, iters, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, iters, k, q))
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


@pytest.mark.parametrize("world,k,iters", [(2, 2, 7), (3, 3, 8), (2, 4, 4)])
def test_sharded_equals_single(world, k, iters):
    import paper_1903_07189_b200 as cf
    img = cf.synth_image(41, 37, seed=5, n_rects=3, n_discs=3, sigma=0.1)
    ref, _ = oracle.flow_f32(img, iters, 1.0)
    got = run_sharded(img, world, iters, k)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))

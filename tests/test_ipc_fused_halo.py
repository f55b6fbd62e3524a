"""Fused-halo row bands across PROCESSES (sharded.IpcBandFlow):
each band kernel stores its boundary rows straight into the neighbours'
buffers through CUDA IPC peer memory, ordered by interprocess events and a
shared-memory launch counter.  Ranks share this one GPU (no kernel waits on
another: all ordering is host-enqueued event waits).  Bit-identical to the
single-process filter."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, h, w, iters, k, shm, q, nan_at=None, side_stream=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1903_07189_b200 as cf
        from paper_1903_07189_b200 import sharded
        img = cf.synth_image(h, w, seed=17, n_rects=12, n_discs=12, sigma=0.1)
        if nan_at is not None:
            img[nan_at] = np.nan
        lay = sharded.BandLayout(h, w, rank, world, k)
        flow = sharded.IpcBandFlow(lay, dist, shm)
        # a non-default (non-blocking) stream: read() / close() must order
        # after it, not after the legacy stream
        strm = torch.cuda.Stream() if side_stream else None
        sp = strm.cuda_stream if strm is not None else None
        flow.load(img[lay.r0:lay.r1])
        which = flow.run(iters, 1.0, stream=sp)
        if nan_at is not None:
            bad = flow.first_bad_iteration()
            try:
                flow.check_finite()
                raised = 0
            except cf.FlowError as e:
                raised = e.iteration
            flow.close()
            q.put((rank, lay.r0, lay.r1, ("bad", bad, raised)))
            return
        # a second run back to back (no barrier), from the same input: the
        # launch numbering and the run-boundary wait keep the halos ordered
        flow.load(img[lay.r0:lay.r1])
        which = flow.run(iters, 1.0, stream=sp)
        assert flow.first_bad_iteration() == 0
        band = flow.read(which)
        flow.close()
        q.put((rank, lay.r0, lay.r1, band))
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((rank, -1, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h,w,iters,k", [(2, 150, 300, 7, 2), (3, 240, 517, 10, 3),
                                               (2, 1200, 4096, 9, 2), (4, 96, 200, 5, 2)])
def test_ipc_fused_halo_equals_single(world, h, w, iters, k):
    import paper_1903_07189_b200 as cf
    img = cf.synth_image(h, w, seed=17, n_rects=12, n_discs=12, sigma=0.1)
    ref, _ = oracle.flow_f32(img, iters, 1.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = f"cf_test_{os.getpid()}_{port}"
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, iters, k, shm, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errors = [b for (_, r0, _, b) in parts if r0 < 0]
    assert not errors, errors
    out = np.empty_like(img)
    for _, r0, r1, band in parts:
        out[r0:r1] = band
    bad = np.argwhere(out.view(np.uint32) != ref.view(np.uint32))
    assert len(bad) == 0, f"{len(bad)} mismatches, first {bad[:3].tolist()}"


def _run(world, h, w, iters, k, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = f"cf_test_{os.getpid()}_{port}"
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, iters, k, shm, q), kwargs=kw)
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errors = [b for (_, r0, _, b) in parts if r0 < 0]
    assert not errors, errors
    return parts


def test_ipc_fused_halo_side_stream():
    import paper_1903_07189_b200 as cf
    h, w, iters = 130, 260, 6
    img = cf.synth_image(h, w, seed=17, n_rects=12, n_discs=12, sigma=0.1)
    ref, _ = oracle.flow_f32(img, iters, 1.0)
    out = np.empty_like(img)
    for _, r0, r1, band in _run(2, h, w, iters, 2, side_stream=True):
        out[r0:r1] = band
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("row", [5, 70, 124])  # in rank 0's band, rank 1's, near the bottom
def test_ipc_fused_halo_nonfinite(row):
    """A NaN in one band: every rank reports the oracle's first bad iteration
    (the flag is reset per run, read back and min-reduced over the ranks)."""
    import paper_1903_07189_b200 as cf
    h, w, iters = 130, 200, 7
    img = cf.synth_image(h, w, seed=17, n_rects=12, n_discs=12, sigma=0.1)
    img[row, 33] = np.nan
    _, ref_bad = oracle.flow_f32(img, iters, 1.0)
    assert ref_bad == 1
    for _, _, _, res in _run(2, h, w, iters, 2, nan_at=(row, 33)):
        assert res == ("bad", ref_bad, ref_bad), res

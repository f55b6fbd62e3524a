"""Host (CPU) cost per launch of the sharded flow loop vs its GPU time (dev tool).

Rank 1 of a simulated world of 8 on cfg4's shape (2048-row band), P2P as
no-ops: the GPU work is the real band kernels; wall time vs device time shows
whether the Python launch loop can keep the GPU fed at N = 8."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_07189_b200 as cf
from paper_1903_07189_b200 import sharded


class NoDist:
    isend, irecv = "send", "recv"

    def P2POp(self, op, t, peer, group=None):
        return (op, t, peer)

    def batch_isend_irecv(self, ops):
        return []


H = W = 16384
for world in (2, 4, 8):
    for k in (2, 3):
        lay = sharded.BandLayout(H, W, 1, world, k)
        a = torch.rand((lay.rows, W), device="cuda")
        b = torch.empty_like(a)
        flow = sharded.ShardedFlow(lay, sharded.cuda_compute(), NoDist(),
                                   side_stream=torch.cuda.Stream())
        flow.run(a, b, 20, 1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        flow.run(a, b, 200, 1.0)
        t_host = time.perf_counter() - t0          # host loop done (GPU may still run)
        e1.record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t0
        n = len(sharded.launch_schedule(200, k))
        print(f"world={world} k={k}: launches={n} host {t_host / n * 1e6:.0f} us/launch, "
              f"gpu {e0.elapsed_time(e1) / n * 1e3:.0f} us/launch, wall {t_wall * 1e3:.1f} ms",
              flush=True)

# The same step captured as one CUDA graph (what bench.py does at N > 1):
# band kernels, the side-stream interior launches and their events replay
# without the Python loop (P2P stubbed here: NCCL needs one GPU per rank).
for world in (8,):
    for k in (2, 3):
        lay = sharded.BandLayout(H, W, 1, world, k)
        a = torch.rand((lay.rows, W), device="cuda")
        b = torch.empty_like(a)
        flow = sharded.ShardedFlow(lay, sharded.cuda_compute(), NoDist(),
                                   side_stream=torch.cuda.Stream())
        flow.run(a, b, 20, 1.0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            flow.run(a, b, 200, 1.0)
        g.replay()
        torch.cuda.synchronize()
        n = len(sharded.launch_schedule(200, k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        g.replay()
        t_host = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        print(f"graph world={world} k={k}: launches={n} host {t_host / n * 1e6:.2f} us/launch, "
              f"gpu {e0.elapsed_time(e1) / n * 1e3:.0f} us/launch", flush=True)

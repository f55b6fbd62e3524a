"""Solver-mode throughput (dev tool): solve_l2_area / solve_l1_area vs the
plain filter on 8192^2, 40 iterations, device-resident (pixel-updates/s)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_1903_07189_b200 as cf

n, it = 8192, 40
f = torch.rand((n, n), device="cuda")
u = torch.empty_like(f); d = torch.empty_like(f)
L = cf.lib()
s = torch.cuda.current_stream().cuda_stream
ws2 = torch.empty(int(L.cf_wmc_filter_workspace_bytes(n, n, n, 1, n * n)), dtype=torch.uint8, device="cuda")
ws1 = torch.empty(int(L.cf_wmc_solve_l1_area_workspace_bytes(n, n, n, 1, n * n)), dtype=torch.uint8, device="cuda")
runs = {
    "flow": lambda: L.cf_wmc_filter_f32(u.data_ptr(), n, n, n, 1, n * n, it, 1.0, ws2.data_ptr(), ws2.numel(), None, s),
    "l2_area": lambda: L.cf_wmc_solve_l2_area_f32(f.data_ptr(), u.data_ptr(), n, n, n, 1, n * n, it, 0.15, 2.0, 1, ws2.data_ptr(), ws2.numel(), None, s),
    "l1_area": lambda: L.cf_wmc_solve_l1_area_f32(f.data_ptr(), u.data_ptr(), d.data_ptr(), n, n, n, 1, n * n, it, 0.15, 2.0, 0.3, 1, ws1.data_ptr(), ws1.numel(), None, s),
}
for name, fn in runs.items():
    u.copy_(f)
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"{name}: {n * n * it / (ms * 1e-3) / 1e9:.1f} G updates/s ({ms:.2f} ms)", flush=True)

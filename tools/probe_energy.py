"""Time cf_wmc_energy_f64 (map + fixed-order reduction) against the map alone
on the 16384^2 supplemental image: CUDA events, median of 9."""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import SUPPLEMENTAL  # noqa: E402

c = SUPPLEMENTAL["cfg1_16k"]
x = torch.from_numpy(cf.synth_image(c.h, c.w, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
y = torch.empty_like(x)
L = cf.lib()
W, H = c.w, c.h
nb = int(L.cf_wmc_reduce_workspace_bytes(W, H, 1))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
out = torch.empty(1, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def t(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


ms_map = t(lambda: L.cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), W, H, W, 1, W * H, s))
res = {}
for q in (1.0, 2.0):
    res[q] = t(lambda: L.cf_wmc_energy_f64(x.data_ptr(), W, H, W, 1, W * H, q, out.data_ptr(),
                                           ws.data_ptr(), nb, s))
nbins = 512
counts = torch.empty(nbins, dtype=torch.int64, device="cuda")
ms_hist = t(lambda: L.cf_wmc_histogram(x.data_ptr(), W, H, W, 1, W * H, 255.0, -256.0, 1.0, nbins,
                                       counts.data_ptr(), ws.data_ptr(), nb, s))
ms_fid = t(lambda: L.cf_wmc_fidelity_f64(x.data_ptr(), y.data_ptr(), W, H, W, 1, W * H, 2.0,
                                         out.data_ptr(), ws.data_ptr(), nb, s))
print(json.dumps({"fidelity_q2_ms": round(ms_fid, 4)}))
print(json.dumps({"map_ms": round(ms_map, 4), "energy_q1_ms": round(res[1.0], 4),
                  "energy_q2_ms": round(res[2.0], 4), "histogram_ms": round(ms_hist, 4)}))

"""Time the C-ABI filter (cf_wmc_filter_f32) of the in-tree library and of
each tools/variants/lib_*.so (tools/build_variants.sh) on a BASELINE config
(default cfg4: 16384^2, here 20 iterations = 10 K=2 launches per call, graph
replayed), and check each variant's output bit-for-bit against the in-tree
library's."""
import ctypes as C
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = CONFIGS[name]
imgs = [cf.synth_image(c.h, c.w, c.seed(p), c.n_rects, c.n_discs, c.sigma) for p in range(c.planes)]
x0 = torch.from_numpy(np.stack(imgs) if c.planes > 1 else imgs[0]).cuda()
P = c.planes
s = torch.cuda.current_stream().cuda_stream
libs = [os.path.join(ROOT, "paper_1903_07189_b200", "libcurveflow_b200.so")] + sorted(
    glob.glob(os.path.join(ROOT, "tools", "variants", "lib_*.so")))
ref = None
for path in libs:
    L = C.CDLL(path)
    L.cf_wmc_filter_workspace_bytes.restype = C.c_size_t
    L.cf_wmc_filter_workspace_bytes.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                                C.c_int64]
    f = L.cf_wmc_filter_f32
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64, C.c_int32,
                  C.c_float, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    nb = L.cf_wmc_filter_workspace_bytes(c.w, c.h, c.w, P, c.h * c.w)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    x = x0.clone()
    run = lambda: f(x.data_ptr(), c.w, c.h, c.w, P, c.h * c.w, iters, c.dt, ws.data_ptr(), nb,  # noqa
                    None, s)
    if run() != 0:
        print(json.dumps({"lib": os.path.basename(path), "error": True}), flush=True)
        continue
    out = x.clone()
    for _ in range(3):
        run()
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    if ref is None:
        ref = out
    same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
    upd = c.w * c.h * P * iters
    print(json.dumps({"config": name, "lib": os.path.basename(path), "ms": round(ms, 4),
                      "Gupd_s": round(upd / ms / 1e6, 1),
                      "frac": round(upd * 8 / ms / 1e6 / 6452.2, 4), "bitexact": same}), flush=True)

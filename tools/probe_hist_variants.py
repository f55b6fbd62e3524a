"""cf_wmc_histogram timing of the in-tree library and tools/variants builds."""
import ctypes as C, glob, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch  # noqa: E402
import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import SUPPLEMENTAL  # noqa: E402
c = SUPPLEMENTAL["cfg1_16k"]
x = torch.from_numpy(cf.synth_image(c.h, c.w, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
W, H = c.w, c.h
s = torch.cuda.current_stream().cuda_stream
ref = None
for path in [os.path.join(ROOT, "paper_1903_07189_b200", "libcurveflow_b200.so")] + sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "lib_*.so"))):
    L = C.CDLL(path)
    L.cf_wmc_reduce_workspace_bytes.restype = C.c_size_t
    L.cf_wmc_reduce_workspace_bytes.argtypes = [C.c_int32] * 3
    f = L.cf_wmc_histogram
    f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64, C.c_float, C.c_float, C.c_float, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    nb = L.cf_wmc_reduce_workspace_bytes(W, H, 1)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    cnt = torch.empty(512, dtype=torch.int64, device="cuda")
    run = lambda: f(x.data_ptr(), W, H, W, 1, W * H, 255.0, -256.0, 1.0, 512, cnt.data_ptr(), ws.data_ptr(), nb, s)  # noqa
    for _ in range(3): run()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    h = cnt.cpu().numpy()
    ref = h if ref is None else ref
    print(json.dumps({"lib": os.path.basename(path), "hist_ms": round(statistics.median(ts), 4), "same": bool(np.array_equal(h, ref))}))

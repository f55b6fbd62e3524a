import ctypes as C, glob, os, sys, statistics, json
sys.path.insert(0, '.')
import torch
import paper_1903_07189_b200 as cf
from paper_1903_07189_b200.configs import SUPPLEMENTAL
c = SUPPLEMENTAL["cfg1_16k"]
x = torch.from_numpy(cf.synth_image(c.h, c.w, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
W, H = c.w, c.h
s = torch.cuda.current_stream().cuda_stream
for path in ["paper_1903_07189_b200/libcurveflow_b200.so"] + sorted(glob.glob("tools/variants/lib_*.so")):
    L = C.CDLL(path)
    L.cf_wmc_reduce_workspace_bytes.restype = C.c_size_t
    L.cf_wmc_reduce_workspace_bytes.argtypes = [C.c_int32]*3
    f = L.cf_wmc_energy_f64
    f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    nb = L.cf_wmc_reduce_workspace_bytes(W, H, 1)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda"); out = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(3): f(x.data_ptr(), W, H, W, 1, W*H, 1.0, out.data_ptr(), ws.data_ptr(), nb, s)
    ts=[]
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(x.data_ptr(), W, H, W, 1, W*H, 1.0, out.data_ptr(), ws.data_ptr(), nb, s); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(json.dumps({"lib": os.path.basename(path), "energy_ms": round(statistics.median(ts),4), "value": out.item()}))

"""Time the K=1..4 sweep kernels and the map of each tools/variants/*.so (dev tool)."""
import ctypes as C, glob, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
H = W = 16384
x = torch.rand((H, W), device="cuda"); y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=8, warm=2):
    for _ in range(warm): fn()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3
out = {}
for path in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "variants", "*.so"))):
    L = C.CDLL(path)
    L.cf_wmc_sweeps_band_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_int32, C.c_void_p, C.c_void_p]
    L.cf_wmc_map_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64, C.c_void_p]
    r = {}
    t = timeit(lambda: L.cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), W, H, W, 1, H * W, s))
    r["map"] = round(H * W / t / 1e9, 1)
    for k in (1, 2, 3, 4):
        t = timeit(lambda: L.cf_wmc_sweeps_band_f32(x.data_ptr(), 0, H, y.data_ptr(), 0, W, H, W, 0, H, k, 1.0, 0, None, s))
        r[f"K{k}"] = round(H * W * k / t / 1e9, 1)
    out[os.path.basename(path)] = r
    print(os.path.basename(path), r, flush=True)

"""K=2 vs K=3 sweep-kernel rate across image geometries (dev tool).

Times a filter call of 2K iterations (= two K-sweep launches) per geometry
for K in (2, 3) through tools/variants/full_L2.so (K=2 schedule) and the
in-tree library (K=3 schedule for large images)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_07189_b200 as cf

libs = {"K3": cf.lib(), "K2": C.CDLL(os.path.join(os.path.dirname(__file__), "variants", "full_L2.so"))}
for L in libs.values():
    L.cf_wmc_filter_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64,
                                    C.c_int32, C.c_float, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    L.cf_wmc_filter_workspace_bytes.restype = C.c_size_t
    L.cf_wmc_filter_workspace_bytes.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64]
geoms = [(16384, 16384, 1), (8192, 8192, 4), (4096, 4096, 16), (2048, 2048, 64), (1920, 1080, 128),
         (16384, 2048, 8), (2048, 16384, 8), (3840, 2160, 32), (1024, 1024, 256), (32768, 8192, 1)]
s = torch.cuda.current_stream().cuda_stream
for (w, h, p) in geoms:
    x = torch.rand((p, h, w), device="cuda")
    row = {}
    for name, L in libs.items():
        k = 2 if name == "K2" else 3
        nb = L.cf_wmc_filter_workspace_bytes(w, h, w, p, h * w)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        f = lambda: L.cf_wmc_filter_f32(x.data_ptr(), w, h, w, p, h * w, 2 * k, 1.0, ws.data_ptr(), nb, None, s)
        for _ in range(2):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(5):
            f()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 5 * 1e-3
        row[name] = round(w * h * p * 2 * k / t / 1e9, 1)
    print(f"{w}x{h}x{p}", row, flush=True)

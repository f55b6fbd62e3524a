import sys, os; sys.path.insert(0, os.getcwd())
import ctypes as C, torch
from paper_1903_07189_b200._lib import lib
L = lib()
P, h, w = 256, 1080, 1920
q = torch.randint(0, 256, (P, h, w), dtype=torch.uint8, device="cuda")
o8 = torch.empty_like(q)
x = torch.empty((P, h, w), device="cuda")
s = torch.cuda.current_stream().cuda_stream
nbf = int(L.cf_wmc_filter_workspace_bytes(w, h, w, P, h * w)); wsf = torch.empty(nbf, dtype=torch.uint8, device="cuda")
nb8 = int(L.cf_wmc_filter_u8_u8_workspace_bytes(w, h, P)); ws8 = torch.empty(nb8, dtype=torch.uint8, device="cuda")
def t(f, n=5):
    for _ in range(2): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
widen = t(lambda: L.cf_wmc_filter_u8_f32(q.data_ptr(), w, h * w, x.data_ptr(), w, h, w, P, h * w, 0, 1.0, None, 0, None, s))
u8u8 = t(lambda: L.cf_wmc_filter_u8_u8(q.data_ptr(), w, h * w, o8.data_ptr(), w, h * w, w, h, P, 20, 1.0, ws8.data_ptr(), nb8, None, s))
u8f32 = t(lambda: L.cf_wmc_filter_u8_f32(q.data_ptr(), w, h * w, x.data_ptr(), w, h, w, P, h * w, 20, 1.0, wsf.data_ptr(), nbf, None, s))
f32 = t(lambda: L.cf_wmc_filter_f32(x.data_ptr(), w, h, w, P, h * w, 20, 1.0, wsf.data_ptr(), nbf, None, s))
print(f"widen {widen:.3f} ms ({P*h*w*5/widen/1e6:.0f} GB/s); u8->u8 x20 {u8u8:.3f}; u8->f32 x20 {u8f32:.3f}; f32 x20 {f32:.3f} ms")

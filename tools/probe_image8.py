"""A/B of the fused interleaved 8-bit path (cf_wmc_filter_image8 on a
3840x2160 RGB image, 50 iterations): run with CF_U8_FUSE=0 (deinterleave /
interleave passes) and without (first / last sweep launch read and write the
bytes)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07189_b200._lib import lib

L = lib()
h, w, ch, iters = 2160, 3840, 3, int(os.environ.get("ITERS", 50))
g = torch.Generator(device="cuda").manual_seed(3)
img = torch.randint(0, 256, (h, w * ch), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty_like(img)
nb = int(L.cf_wmc_filter_image8_workspace_bytes(w, h, ch))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run():
    assert L.cf_wmc_filter_image8(img.data_ptr(), w * ch, out.data_ptr(), w * ch, w, h, ch, iters,
                                  1.0, ws.data_ptr(), nb, None, s) == 0
for _ in range(3):
    run()
ts = []
for _ in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
print(json.dumps({"fuse": os.environ.get("CF_U8_FUSE", "1"),
                  "fused_path": int(L.cf_wmc_filter_image8_fused(img.data_ptr(), w * ch, w, ch,
                                                                 iters)),
                  "iters": iters, "ms": round(ms, 3),
                  "Gupd_s": round(h * w * ch * iters / ms / 1e6, 1),
                  "checksum": int(out.to(torch.int64).sum())}))

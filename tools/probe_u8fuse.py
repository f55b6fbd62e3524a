"""A/B of the fused u8 ingest (cfg5: 256 x 1080p u8 frames, 20 iterations,
u8 -> u8).  Run twice: CF_U8_FUSE=0 (separate widening pass) and default."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07189_b200._lib import lib

L = lib()
if os.environ.get("CF_PROBE_LIB"):   # a dev variant (tools/build_variants.sh)
    import ctypes as C
    V = C.CDLL(os.environ["CF_PROBE_LIB"])
    for name in ("cf_wmc_filter_u8_u8", "cf_wmc_filter_u8_u8_workspace_bytes"):
        getattr(V, name).argtypes = getattr(L, name).argtypes
        getattr(V, name).restype = getattr(L, name).restype
    L = V
P, h, w, iters = int(os.environ.get("P", 256)), 1080, 1920, 20
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randint(0, 256, (P, h, w), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty_like(q)
nb = int(L.cf_wmc_filter_u8_u8_workspace_bytes(w, h, P))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run():
    assert L.cf_wmc_filter_u8_u8(q.data_ptr(), w, h * w, out.data_ptr(), w, h * w, w, h, P, iters,
                                 1.0, ws.data_ptr(), nb, None, s) == 0
for _ in range(3):
    run()
ts = []
for _ in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
print(json.dumps({"lib": os.path.basename(os.environ.get("CF_PROBE_LIB", "in-tree")),
                  "fuse": os.environ.get("CF_U8_FUSE", "1"), "ms": round(ms, 3),
                  "Gupd_s": round(P * h * w * iters / ms / 1e6, 1),
                  "checksum": int(out.to(torch.int64).sum())}))

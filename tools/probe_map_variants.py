"""Time cf_wmc_map_f32 of each tools/variants/lib_*.so (dev builds, see
tools/build_variants.sh) on the supplemental 16384^2 image and check every
variant's output bit-for-bit against the in-tree library's."""
import ctypes as C
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import SUPPLEMENTAL  # noqa: E402

from paper_1903_07189_b200.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1_16k"
if "x" in name:  # HxWxP: seeded uniform planes of that geometry
    H, W, P = (int(v) for v in name.split("x"))
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand((P, H, W), device="cuda", generator=g)
else:
    c = SUPPLEMENTAL.get(name) or CONFIGS[name]
    H, W, P = c.h, c.w, 1
    x = torch.from_numpy(cf.synth_image(c.h, c.w, c.seed(0), c.n_rects, c.n_discs,
                                        c.sigma)).cuda()
ref = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
assert cf.lib().cf_wmc_map_f32(x.data_ptr(), ref.data_ptr(), W, H, W, P, W * H, s) == 0
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
libs = [os.path.join(ROOT, "paper_1903_07189_b200", "libcurveflow_b200.so")] + sorted(
    glob.glob(os.path.join(ROOT, "tools", "variants", "lib_*.so")))
for path in libs:
    L = C.CDLL(path)
    f = L.cf_wmc_map_f32
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                  C.c_int64, C.c_void_p]
    y = torch.empty_like(x)
    rc = f(x.data_ptr(), y.data_ptr(), W, H, W, P, W * H, s)
    if rc != 0:
        print(json.dumps({"lib": os.path.basename(path), "error": rc}), flush=True)
        continue
    for _ in range(2):
        assert f(x.data_ptr(), y.data_ptr(), W, H, W, P, W * H, s) == 0
    ts = []
    for _ in range(15):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f(x.data_ptr(), y.data_ptr(), W, H, W, P, W * H, s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    same = bool(torch.equal(y.view(torch.int32), ref.view(torch.int32)))
    print(json.dumps({"config": name, "lib": os.path.basename(path), "ms": round(ms, 4),
                      "frac": round(W * H * P * 8 / ms / 1e6 / 6452.2, 4), "bitexact": same}),
          flush=True)

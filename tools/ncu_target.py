"""Small fixed workloads for ncu captures (tools/gpu_session*.sh):

  python tools/ncu_target.py map [n]      # n maps of the supplemental 16384^2 image
  python tools/ncu_target.py flowK [n]    # n K-sweep band launches on 16384^2
  python tools/ncu_target.py cfg2|cfg3|cfg4|cfg5
        # the C-ABI filter of that BASELINE config's input with 4 iterations
        # (2 K=2 launches; cfg5: the u8 -> u8 path, widening + 2 launches)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import CONFIGS, SUPPLEMENTAL  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "map"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
H = W = 16384
s = torch.cuda.current_stream().cuda_stream
if what in CONFIGS:
    c = CONFIGS[what]
    imgs = [cf.synth_image(c.h, c.w, c.seed(p), c.n_rects, c.n_discs, c.sigma,
                           dtype="u8" if c.u8 else "f32") for p in range(c.planes)]
    x = torch.from_numpy(np.stack(imgs) if c.planes > 1 else imgs[0]).cuda()
    cfg = cf.FlowConfig(dt=c.dt, iters=4)
    for _ in range(2):
        if c.u8:
            cf.mc_flow_u8(x, cfg, out_dtype="u8", check_finite=False)
        else:
            cf.mc_flow(x, cfg, check_finite=False)
elif what == "map":  # the supplemental map config's synthetic image (cfg1 generator)
    c = SUPPLEMENTAL["cfg1_16k"]
    x = torch.from_numpy(cf.synth_image(H, W, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
    y = torch.empty_like(x)
    for _ in range(n):
        cf.lib().cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), W, H, W, 1, H * W, s)
else:
    x = torch.rand((H, W), device="cuda")
    y = torch.empty_like(x)
    for _ in range(n):
        k = int(what[-1])
        cf.sweeps_band(x, 0, y, 0, H, 0, H, k, 1.0, 0)
torch.cuda.synchronize()
print("ok", what)

"""Small fixed workload for ncu captures: `python tools/ncu_target.py map|flowK [n]`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_07189_b200 as cf

what = sys.argv[1] if len(sys.argv) > 1 else "map"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
H = W = 16384
if what == "map":  # the supplemental map config's synthetic image (cfg1 generator)
    from paper_1903_07189_b200.configs import SUPPLEMENTAL
    c = SUPPLEMENTAL["cfg1_16k"]
    x = torch.from_numpy(cf.synth_image(H, W, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
else:
    x = torch.rand((H, W), device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(n):
    if what == "map":
        cf.lib().cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), W, H, W, 1, H * W, s)
    else:
        k = int(what[-1])
        cf.sweeps_band(x, 0, y, 0, H, 0, H, k, 1.0, 0)
torch.cuda.synchronize()
print("ok", what)

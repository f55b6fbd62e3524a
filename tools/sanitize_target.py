"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1903_07189_b200 as cf
for (h, w) in [(1, 1), (5, 1), (3, 7), (17, 31), (70, 200), (130, 257)]:
    img = cf.synth_image(h, w, seed=h * w, n_rects=3, n_discs=3, sigma=0.1)
    d = torch.from_numpy(img).cuda()
    cf.wmc_half_laplace(d)
    cf.mc_flow(d, cf.FlowConfig(iters=7))
    cf.solve_l2_area(d, cf.SolverConfig(lam=2.0, dt=0.1, iters=5))
    for k in (1, 2, 3, 4):
        out = torch.empty_like(d)
        cf.sweeps_band(d, 0, out, 0, h, 0, h, k, 1.0, 0)
    cf.wmc_energy(d, 1.0); cf.wmc_histogram(d)
q = cf.synth_image(40, 64, seed=1, n_rects=3, n_discs=3, sigma=0.1, dtype="u8")
cf.mc_flow_u8(torch.from_numpy(np.stack([q, q])).cuda(), cf.FlowConfig(iters=4))
cf.mc_flow_image8(np.stack([q, q, q], axis=2), cf.FlowConfig(iters=3))
torch.cuda.synchronize()
print("sanitize target ok")

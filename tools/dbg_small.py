import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch, oracle
import paper_1903_07189_b200 as cf
for (h, w) in [(11, 1), (1, 9), (5, 1), (11, 2), (11, 3), (40, 1), (3, 3)]:
    img = np.random.default_rng(h * 7 + w).uniform(0, 1, (h, w)).astype(np.float32)
    for it in range(1, 6):
        got = cf.mc_flow(torch.from_numpy(img).cuda(), cf.FlowConfig(iters=it)).cpu().numpy()
        ref, _ = oracle.flow_f32(img, it, 1.0)
        bad = np.argwhere(got.view(np.uint32) != ref.view(np.uint32))
        if len(bad):
            print((h, w), 'iters', it, 'mismatch at', bad[:6].tolist(), got.ravel()[:6], ref.ravel()[:6])
    # band API single launch K=1..4
    d = torch.from_numpy(img).cuda()
    for k in (1, 2, 3, 4):
        out = torch.empty_like(d)
        cf.sweeps_band(d, 0, out, 0, h, 0, h, k, 1.0, 0)
        ref, _ = oracle.flow_f32(img, k, 1.0)
        bad = np.argwhere(out.cpu().numpy().view(np.uint32) != ref.view(np.uint32))
        if len(bad): print((h, w), 'band K', k, 'mismatch', bad[:6].tolist())
print('done')

"""Quick device-timing probe of the kernels (development tool, not the bench)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_07189_b200 as cf

def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3

res = {}
H = W = 16384
x = torch.rand((H, W), device="cuda")
y = torch.empty_like(x)
t = timeit(lambda: cf.lib().cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), W, H, W, 1, H*W, torch.cuda.current_stream().cuda_stream))
res["map16k_s"] = t; res["map16k_Gpx"] = H*W/t/1e9; res["map16k_GBs"] = 8*H*W/t/1e9
for k in (1, 2, 3, 4):
    t = timeit(lambda: cf.sweeps_band(x, 0, y, 0, H, 0, H, k, 1.0, 0))
    res[f"flowK{k}_Gupd"] = H*W*k/t/1e9
    res[f"flowK{k}_GBs"] = 8*H*W/t/1e9
# cfg2-size
x2 = torch.rand((1024, 1024), device="cuda")
t = timeit(lambda: cf.mc_flow(x2, cf.FlowConfig(iters=100), check_finite=False), reps=5)
res["cfg2_Gupd"] = 1024*1024*100/t/1e9
print(json.dumps(res, indent=1))

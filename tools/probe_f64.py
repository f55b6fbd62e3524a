"""Throughput of the SPEC-faithful fp64 path (cf_wmc_filter_f64 / map) on the
BASELINE configs: CUDA events, median of 5 runs (graph-cached repeats)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import CONFIGS, SUPPLEMENTAL  # noqa: E402

for name in (sys.argv[1:] or ["cfg1_16k", "cfg2", "cfg3", "cfg4", "cfg5"]):
    c = CONFIGS.get(name) or SUPPLEMENTAL[name]
    imgs = [cf.synth_image(c.h, c.w, c.seed(p), c.n_rects, c.n_discs, c.sigma,
                           dtype="u8" if c.u8 else "f32") for p in range(c.planes)]
    host = np.stack(imgs) if c.planes > 1 else imgs[0]
    if c.u8:
        src = torch.from_numpy(host).cuda()
        out = torch.empty(src.shape, dtype=torch.float64, device="cuda")
        nb = int(cf.lib().cf_wmc_filter_f64_workspace_bytes(c.w, c.h, c.w, c.planes, c.w * c.h))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        run = lambda: cf.mc_flow_u8(src, cf.FlowConfig(c.dt, c.iters), out=out, workspace=ws,  # noqa
                                    out_dtype="f64", check_finite=False)
    else:
        x0 = torch.from_numpy(host.astype(np.float64)).cuda()
        x = x0.clone()
        if c.iters == 0:
            y = torch.empty_like(x)
            s = torch.cuda.current_stream().cuda_stream
            P = c.planes
            run = lambda: cf.lib().cf_wmc_map_f64(x.data_ptr(), y.data_ptr(), c.w, c.h, c.w, P,  # noqa
                                                   c.w * c.h, s)
        else:
            nb = int(cf.lib().cf_wmc_filter_f64_workspace_bytes(c.w, c.h, c.w, c.planes,
                                                                 c.w * c.h))
            ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
            run = lambda: cf.mc_flow(x, cf.FlowConfig(c.dt, c.iters), inplace=True,  # noqa
                                     workspace=ws, check_finite=False)
    for _ in range(3):
        run()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    upd = c.updates
    print(json.dumps({"config": name, "precision": "fp64", "ms": round(ms, 3),
                      "Gupd_s": round(upd / ms / 1e6, 2),
                      "hbm_GBs_16B": round(upd * 16 / ms / 1e6, 1)}), flush=True)

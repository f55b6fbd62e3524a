"""Map throughput on the supplemental 16384^2 image (and cfg1): CUDA events,
median of 20 launches, 256 MiB L2 flush between launches for small images."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_07189_b200 as cf  # noqa: E402
from paper_1903_07189_b200.configs import CONFIGS, SUPPLEMENTAL  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
for name in (sys.argv[1:] or ["cfg1_16k", "cfg1"]):
    c = CONFIGS.get(name) or SUPPLEMENTAL[name]
    x = torch.from_numpy(cf.synth_image(c.h, c.w, c.seed(0), c.n_rects, c.n_discs, c.sigma)).cuda()
    y = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    L = cf.lib()
    for _ in range(3):
        assert L.cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), c.w, c.h, c.w, 1, c.w * c.h, s) == 0
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.cf_wmc_map_f32(x.data_ptr(), y.data_ptr(), c.w, c.h, c.w, 1, c.w * c.h, s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    gbs = c.w * c.h * 8 / ms / 1e6
    print(json.dumps({"config": name, "ms": round(ms, 4), "Gpx_s": round(c.w * c.h / ms / 1e6, 1),
                      "GBs": round(gbs, 1), "frac": round(gbs / peak, 4)}), flush=True)

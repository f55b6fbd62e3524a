"""Golden vectors (tests/golden/wmc_golden.npz, made by make_golden.py from
independent Python/numpy transcriptions) pin the C oracle -- and, on a GPU,
the kernels -- bit-exactly."""
import os

import numpy as np
import pytest

import oracle

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "wmc_golden.npz"))
CASES = sorted({k.split("/")[0] for k in G.files})


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_golden(case):
    img = G[f"{case}/in"]
    assert np.array_equal(bits(oracle.wmc_map_f64(img.astype(np.float64))), bits(G[f"{case}/map64"]))
    assert np.array_equal(bits(oracle.wmc_map_f32(img)), bits(G[f"{case}/map32"]))
    out, bad = oracle.flow_f32(img, 5, 1.0)
    assert bad == 0
    assert np.array_equal(bits(out), bits(G[f"{case}/flow5"]))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_matches_golden(case):
    import torch

    import paper_1903_07189_b200 as cf
    img = G[f"{case}/in"]
    d = torch.from_numpy(img).cuda()
    assert np.array_equal(bits(cf.wmc_half_laplace(d).cpu().numpy()), bits(G[f"{case}/map32"]))
    out = cf.mc_flow(d, cf.FlowConfig(dt=1.0, iters=5)).cpu().numpy()
    assert np.array_equal(bits(out), bits(G[f"{case}/flow5"]))

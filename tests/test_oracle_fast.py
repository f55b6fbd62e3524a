"""The vectorised oracle (oracle/wmc_fast.c) and the CPU-side generator
(oracle/synth_ref.c) pinned to the scalar oracle and to the product's
generator.  CPU only.

The vectorised functions are what the full-config GPU parity tests
(tests/test_gpu_configs.py) check the kernels against, so they must equal
the scalar restatement (oracle/wmc_oracle.c, itself pinned by
tests/test_oracle.py and tests/golden/) bit for bit.
"""
import numpy as np
import pytest

import oracle
from paper_1903_07189_b200.configs import CONFIGS, SUPPLEMENTAL

pytestmark = pytest.mark.skipif(not oracle.fast_supported(), reason="CPU without AVX2/FMA")

SHAPES = [(1, 1), (1, 2), (2, 1), (1, 3), (3, 2), (2, 3), (7, 5), (16, 16), (17, 33), (33, 17),
          (64, 130), (129, 257)]


def _same_f32(a, b):
    """Bitwise equal, NaN positions equal (NaN payloads may differ between
    scalar SSE and vector AVX operand orders)."""
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32))


def _same_f64(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


def test_weights_match():
    assert oracle.lib().or_fast_w64_matches() == 1


@pytest.mark.parametrize("shape", SHAPES)
def test_flow_f32_matches_scalar(shape):
    rng = np.random.default_rng(hash(shape) & 0xffff)
    a = rng.random(shape, dtype=np.float32)
    for iters, dt in ((1, 1.0), (2, 0.5), (5, 1.0), (9, 0.3)):
        r1, b1 = oracle.flow_f32(a, iters, dt, threads=3)
        r2, b2 = oracle.flow_f32_fast(a, iters, dt, threads=5)
        assert b1 == b2 == 0
        assert _same_f32(r1, r2), (shape, iters, dt)


@pytest.mark.parametrize("shape", SHAPES)
def test_map_matches_scalar(shape):
    rng = np.random.default_rng(7 + (hash(shape) & 0xffff))
    a = rng.random(shape, dtype=np.float32)
    m1, t1 = oracle.wmc_map_f32(a, threads=2, return_ties=True)
    m2, t2 = oracle.wmc_map_f32_fast(a, threads=7, return_ties=True)
    assert _same_f32(m1, m2) and np.array_equal(t1, t2)
    assert _same_f64(oracle.wmc_map_f64(a, threads=2), oracle.wmc_map_f64_fast(a, threads=3))


@pytest.mark.parametrize("shape", SHAPES)
def test_flow_f64_matches_scalar(shape):
    rng = np.random.default_rng(11 + (hash(shape) & 0xffff))
    a = rng.random(shape, dtype=np.float32)
    for iters, dt in ((1, 1.0), (4, 0.7)):
        r1, _ = oracle.flow_f64(a, iters, dt, threads=2)
        r2, _ = oracle.flow_f64_fast(a, iters, dt, threads=6)
        assert _same_f64(r1, r2)


def test_structured_images():
    """Ramps, constants, exact ties, quantised levels: selection tie paths."""
    h, w = 40, 67
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float32)
    cases = [np.full((h, w), 0.3, np.float32), (xx / w).astype(np.float32),
             ((xx + yy) / (w + h)).astype(np.float32), ((xx - 2 * yy) / 200).astype(np.float32),
             (np.random.default_rng(3).integers(0, 4, (h, w)) / 4).astype(np.float32),
             ((xx % 2) * 0.5).astype(np.float32)]
    for a in cases:
        r1, _ = oracle.flow_f32(a, 6, 1.0)
        r2, _ = oracle.flow_f32_fast(a, 6, 1.0)
        assert _same_f32(r1, r2)
        m1, t1 = oracle.wmc_map_f32(a, return_ties=True)
        m2, t2 = oracle.wmc_map_f32_fast(a, return_ties=True)
        assert _same_f32(m1, m2) and np.array_equal(t1, t2)
        assert _same_f64(oracle.flow_f64(a, 3)[0], oracle.flow_f64_fast(a, 3)[0])


def test_nonfinite_and_huge():
    rng = np.random.default_rng(5)
    for val, pos in ((np.nan, (3, 4)), (np.inf, (0, 0)), (-np.inf, (9, 12)), (3e38, (5, 5)),
                     (-3e38, (0, 12))):
        a = rng.random((10, 13), dtype=np.float32)
        a[pos] = val
        r1, b1 = oracle.flow_f32(a, 4, 1.0)
        r2, b2 = oracle.flow_f32_fast(a, 4, 1.0)
        assert b1 == b2 and b1 >= 1
        assert _same_f32(r1, r2)
        d1, c1 = oracle.flow_f64(a, 4, 1.0)
        d2, c2 = oracle.flow_f64_fast(a, 4, 1.0)
        assert c1 == c2 and _same_f64(d1, d2)
        m1, t1 = oracle.wmc_map_f32(a, return_ties=True)
        m2, t2 = oracle.wmc_map_f32_fast(a, return_ties=True)
        assert _same_f32(m1, m2) and np.array_equal(t1, t2)


def test_planes_batch():
    rng = np.random.default_rng(9)
    a = rng.random((3, 21, 34), dtype=np.float32)
    r1, _ = oracle.flow_f32(a, 5, 1.0)
    r2, _ = oracle.flow_f32_fast(a, 5, 1.0)
    assert _same_f32(r1, r2)
    m1 = oracle.wmc_map_f32(a)
    m2 = oracle.wmc_map_f32_fast(a)
    assert _same_f32(m1, m2)


def test_inplace_flow():
    a = np.random.default_rng(2).random((2, 30, 40), dtype=np.float32)
    ref, _ = oracle.flow_f32(a, 3, 1.0)
    b = a.copy()
    out, _ = oracle.flow_f32_fast(b, 3, 1.0, inplace=True)
    assert out.base is b or out is b
    assert _same_f32(ref, b)


# --------------------------------------------------------------- generator --
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_synth_matches_product(name):
    """oracle/synth_ref.c == cf_synth_* (the C-ABI generator is host code:
    no GPU needed), byte for byte, for two planes of each config."""
    import paper_1903_07189_b200 as cf
    c = CONFIGS[name]
    for p in range(min(2, c.planes)):
        a = cf.synth_image(c.h, c.w, c.seed(p), c.n_rects, c.n_discs, c.sigma,
                           dtype="u8" if c.u8 else "f32")
        b = oracle.synth(c.w, c.h, c.seed(p), c.n_rects, c.n_discs, c.sigma, u8=c.u8, threads=3)
        assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_synth_matches_product_large():
    """cfg4's generator parameters (2000 + 2000 shapes, sigma 0.1) at full
    height and a quarter of the width, and 512 rows of cfg1_16k's 16384-wide
    image (the generator's scene depends on (w, h), so these are complete
    images of their own size)."""
    import paper_1903_07189_b200 as cf
    c = CONFIGS["cfg4"]
    w, h = 4096, 16384
    a = cf.synth_image(h, w, c.seed(0), c.n_rects, c.n_discs, c.sigma)
    b = oracle.synth(w, h, c.seed(0), c.n_rects, c.n_discs, c.sigma)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    s = SUPPLEMENTAL["cfg1_16k"]
    a = cf.synth_image(512, s.w, s.seed(0), s.n_rects, s.n_discs, s.sigma)
    b = oracle.synth(s.w, 512, s.seed(0), s.n_rects, s.n_discs, s.sigma)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))

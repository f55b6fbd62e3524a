"""Generate tests/golden/wmc_golden.npz -- golden vectors for the WMC path.

The reference ships no fixtures, so these vectors come from
two small pure-Python/numpy transcriptions written independently of the C
oracle and of the CUDA kernels:

* fp64: Eqs. 27-28 taken literally: eight
  correlations with the exact-rational kernels lowered to double, row-major
  taps, clamp-to-edge, strict-< first minimum.
* fp32 canonical: the pinned fp32 operation sequence on numpy
  float32 scalars.  fmaf(a, b, c) is emulated as float32(double(a)*double(b) +
  double(c)); for every fma in the sequence a*b is exact in double and the
  sum of two float32-range terms of the magnitudes involved is exact in
  double, so the single final rounding equals the fused one.
* flow: 5 Jacobi iterations at dt = 1 of the fp32 sequence, with the step
  U' = fma(fl(dt * fl(1/12)), D_m, u) rounded once (exact rational
  arithmetic: that fma's sum is not always exact in double).

Run:  python tests/golden/make_golden.py   (writes the .npz next to it)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
f32 = np.float32

K12 = {  # PAPER.md:411-444 times 12, [row][col]
    1: [[2, 2, 0], [4, -12, 0], [2, 2, 0]], 2: [[2, 4, 2], [2, -12, 2], [0, 0, 0]],
    3: [[0, 2, 2], [0, -12, 4], [0, 2, 2]], 4: [[0, 0, 0], [2, -12, 2], [2, 4, 2]],
    5: [[2, 4, 1], [4, -12, 0], [1, 0, 0]], 6: [[1, 4, 2], [0, -12, 4], [0, 0, 1]],
    7: [[0, 0, 1], [0, -12, 4], [1, 4, 2]], 8: [[1, 0, 0], [4, -12, 0], [2, 4, 1]],
}
W64 = {i: [[0.0 if n == 0 else (-1.0 if n == -12 else n / 12.0) for n in row] for row in k]
       for i, k in K12.items()}


def nb(img, y, x):
    h, w = img.shape
    g = lambda yy, xx: img[min(max(yy, 0), h - 1), min(max(xx, 0), w - 1)]  # noqa: E731
    return [g(y + r, x + c) for r in (-1, 0, 1) for c in (-1, 0, 1)]


def px64(n9):
    best = None
    for i in range(1, 9):
        s = 0.0
        for t in range(9):
            s = s + W64[i][t // 3][t % 3] * float(n9[t])
        if best is None or abs(s) < abs(best):
            best = s
    return best


def fma32(a, b, c):
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def px32(n9):
    a, b, c, l, u, r, e, f, g = [f32(v) for v in n9]
    n12u = f32(u * f32(-12))
    Vl, Vc, Vr = f32(a + e), f32(b + f), f32(c + g)
    Wm, W0 = f32(Vl + Vc), f32(Vc + Vr)
    Ht, Hc, Hb = f32(a + c), f32(l + r), f32(e + g)
    Tm, T0 = f32(Ht + Hc), f32(Hc + Hb)
    D = [fma32(2, fma32(2, l, Wm), n12u), fma32(2, fma32(2, b, Tm), n12u),
         fma32(2, fma32(2, r, W0), n12u), fma32(2, fma32(2, f, T0), n12u)]
    K5, K6 = f32(f32(c + e) + n12u), f32(f32(a + g) + n12u)
    D += [fma32(4, f32(b + l), fma32(2, a, K5)),
          fma32(4, f32(b + r), fma32(2, c, K6)),
          fma32(4, f32(r + f), fma32(2, g, K5)),
          fma32(4, f32(l + f), fma32(2, e, K6))]
    pick = lambda lft, rgt: rgt if abs(rgt) < abs(lft) else lft  # noqa: E731
    best = pick(pick(pick(D[0], D[1]), pick(D[2], D[3])), pick(pick(D[4], D[5]), pick(D[6], D[7])))
    return D, n12u, best


C12 = f32(1.0) / f32(12.0)


def map32(img):
    h, w = img.shape
    out = np.empty_like(img)
    for y in range(h):
        for x in range(w):
            n9 = nb(img, y, x)
            D, n12u, best = px32(n9)
            T = min(abs(f32(d + best)) for d in D)
            tau = fma32(abs(n12u), f32(float.fromhex("0x1.8p-19")), f32(abs(best) * f32(float.fromhex("0x1.0p-20"))))
            if T <= tau and T < abs(best):
                out[y, x] = f32(px64(n9))
            else:
                out[y, x] = f32(best * C12)
    return out


def fma32_exact(a, b, c):
    """fl32(a*b + c) with ONE rounding, round-to-nearest-even, from exact
    rational arithmetic (a*b + c is not always exact in double)."""
    from fractions import Fraction
    a, b, c = f32(a), f32(b), f32(c)
    exact = Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c))
    if exact == 0:  # RN: exact zero sums are +0 unless both addends are -0
        p_neg = (np.signbit(a) != np.signbit(b))
        return f32(-0.0) if (p_neg and np.signbit(c)) else f32(0.0)
    cand = f32(float(exact))  # within one ulp of the answer
    best, best_err = None, None
    for v in (np.nextafter(cand, f32(-np.inf)), cand, np.nextafter(cand, f32(np.inf))):
        err = abs(Fraction(float(v)) - exact)
        if best is None or err < best_err or (err == best_err and
                                               (int(v.view(np.uint32)) & 1) == 0):
            best, best_err = v, err
    return f32(best)


def flow32(img, iters, dt=1.0):
    """The canonical flow step: U' = fma(fl(dt * fl(1/12)), D_m, u)."""
    c = f32(f32(dt) * C12)
    U = img.copy()
    for _ in range(iters):
        h, w = U.shape
        V = np.empty_like(U)
        for y in range(h):
            for x in range(w):
                _, _, best = px32(nb(U, y, x))
                V[y, x] = fma32_exact(c, best, U[y, x])
        U = V
    return U


def map64(img):
    h, w = img.shape
    return np.array([[px64(nb(img, y, x)) for x in range(w)] for y in range(h)])


def inputs():
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    cases = {}
    imp = np.zeros((3, 3), f32)
    imp[1, 1] = 1
    cases["impulse3"] = imp
    cases["ramp5"] = np.tile(np.arange(5, dtype=f32), (5, 1))
    cases["const6x7"] = np.full((6, 7), 0.3, f32)
    rng = np.random.default_rng(20190307)
    for i in range(3):
        cases[f"rand8_{i}"] = rng.uniform(0, 1, (8, 8)).astype(f32)
    cases["ragged1x9"] = rng.uniform(0, 1, (1, 9)).astype(f32)
    cases["ragged11x1"] = rng.uniform(0, 1, (11, 1)).astype(f32)
    try:
        import paper_1903_07189_b200 as cf
        cases["synth13x17"] = cf.synth_image(13, 17, seed=7, n_rects=3, n_discs=3, sigma=0.1)
        cases["synth24x20"] = cf.synth_image(24, 20, seed=8, n_rects=4, n_discs=4, sigma=0.05)
    except Exception:  # generator not built: keep the numpy cases only
        pass
    return cases


def main():
    data = {}
    for name, img in inputs().items():
        data[f"{name}/in"] = img
        data[f"{name}/map64"] = map64(img.astype(np.float64))
        data[f"{name}/map32"] = map32(img)
        data[f"{name}/flow5"] = flow32(img, 5)
    np.savez_compressed(os.path.join(HERE, "wmc_golden.npz"), **data)
    print("wrote", len(data) // 4, "cases")


if __name__ == "__main__":
    main()

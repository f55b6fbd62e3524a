"""CPU oracle for the WMC path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this package, always as the checker or the timed
reference CPU path; the product (paper_1903_07189_b200/) never does.

Wraps oracle/liboracle.so (wmc_oracle.c: fp64 SPEC-faithful + fp32 canonical
restatement) and, when built, oracle/_ref/libcf_ref.so (the fp64 restatement
run on the reference's own curveflow::parallel executor).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_REF = os.path.join(_HERE, "_ref", "libcf_ref.so")
_lib = None
_ref = None

_i32, _i64, _f32, _f64, _vp = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p
_pi32 = C.POINTER(C.c_int32)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = C.CDLL(_LIB)
        L.or_wmc_map_f64.argtypes = [_vp, _vp, _i32, _i32, _i32, _vp]
        L.or_wmc_map_f32.argtypes = [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32, _vp]
        L.or_wmc_flowmap_f32.argtypes = [_vp, _vp, _i32, _i32, _i32]
        L.or_wmc_flowmap_f32.restype = C.c_int
        L.or_flow_f32.argtypes = [_vp, _i32, _i32, _i64, _i32, _i64, _i32, _f32, _i32, _pi32]
        L.or_flow_f64.argtypes = [_vp, _i32, _i32, _i32, _f64, _i32, _pi32]
        L.or_u8_to_f32.argtypes = [_vp, _vp, _i64]
        L.or_quantize_u8.argtypes = [_vp, _vp, _i64]
        L.or_quantize_u8.restype = None
        L.or_solve_l2_area_f32.argtypes = [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32, _f32,
                                           _f32, _i32, _i32, _pi32]
        L.or_solve_l2_area_f32.restype = C.c_int
        L.or_solve_l1_area_f32.argtypes = [_vp, _vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32,
                                           _f32, _f32, _f32, _i32, _i32, _pi32]
        L.or_solve_l1_area_f32.restype = C.c_int
        L.or_l1_px.argtypes = [_f32, _f32, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.or_l1_px.restype = None
        L.or_fidelity.argtypes = [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _f64, _i32]
        L.or_fidelity.restype = C.c_double
        L.or_energy_from_map.argtypes = [_vp, _i32, _i32, _i32, _f64, _i32]
        L.or_energy_from_map.restype = C.c_double
        L.or_histogram_from_map.argtypes = [_vp, _i64, _f32, _f32, _f32, _i32, _vp]
        L.or_histogram_from_map.restype = None
        L.or_wmc_naive_f64.argtypes = [_vp, _vp, _i32, _i32]
        L.or_synth_f32.argtypes = [_vp, _i32, _i32, _i64, C.c_uint64, _i32, _i32, _f64, _i32]
        L.or_synth_f32.restype = C.c_int
        L.or_synth_u8.argtypes = [_vp, _i32, _i32, _i64, C.c_uint64, _i32, _i32, _f64, _i32]
        L.or_synth_u8.restype = C.c_int
        L.or_fast_supported.argtypes = []
        L.or_fast_supported.restype = C.c_int
        L.or_fast_w64_matches.argtypes = []
        L.or_fast_w64_matches.restype = C.c_int
        L.or_fast_flow_f32.argtypes = [_vp, _i32, _i32, _i64, _i32, _i64, _i32, _f32, _i32, _pi32]
        L.or_fast_flow_f32.restype = C.c_int
        L.or_fast_map_f32.argtypes = [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32, _vp]
        L.or_fast_map_f32.restype = C.c_int
        L.or_fast_flow_f64.argtypes = [_vp, _i32, _i32, _i32, _f64, _i32, _pi32]
        L.or_fast_flow_f64.restype = C.c_int
        L.or_fast_map_f64.argtypes = [_vp, _vp, _i32, _i32, _i32]
        L.or_fast_map_f64.restype = C.c_int
        L.or_kernel_bank_numerators.argtypes = [_pi32]
        for f in ("or_wmc_map_f64", "or_wmc_map_f32", "or_flow_f32", "or_flow_f64"):
            getattr(L, f).restype = C.c_int
        L.or_u8_to_f32.restype = None
        L.or_wmc_naive_f64.restype = None
        _lib = L
    return _lib


def ref_lib():
    """The reference-executor build, or None if it was never built."""
    global _ref
    if _ref is None and os.path.exists(_REF):
        L = C.CDLL(_REF)
        L.ref_wmc_map_f64.argtypes = [_vp, _vp, _i32, _i32, _i32]
        L.ref_flow_f64.argtypes = [_vp, _i32, _i32, _i32, _f64, _i32, _pi32]
        L.ref_wmc_map_f64.restype = C.c_int
        L.ref_flow_f64.restype = C.c_int
        _ref = L
    return _ref


def _threads(t):
    return os.cpu_count() or 1 if t is None else t


def wmc_map_f64(img, threads=None, return_argmin=False):
    a = np.ascontiguousarray(img, dtype=np.float64)
    h, w = a.shape
    out = np.empty_like(a)
    am = np.empty((h, w), dtype=np.int8) if return_argmin else None
    rc = lib().or_wmc_map_f64(a.ctypes.data, out.ctypes.data, w, h, _threads(threads),
                              am.ctypes.data if am is not None else None)
    assert rc == 0
    return (out, am) if return_argmin else out


def wmc_naive_f64(img):
    a = np.ascontiguousarray(img, dtype=np.float64)
    h, w = a.shape
    out = np.empty_like(a)
    lib().or_wmc_naive_f64(a.ctypes.data, out.ctypes.data, w, h)
    return out


def wmc_map_f32(img, threads=None, return_ties=False):
    """fp32 canonical map with the fp64 near-tie rule; img (H, W) or (P, H, W)."""
    a = np.ascontiguousarray(img, dtype=np.float32)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    out = np.empty_like(a3)
    ties = np.zeros(a3.shape, dtype=np.int8) if return_ties else None
    rc = lib().or_wmc_map_f32(a3.ctypes.data, out.ctypes.data, w, h, w, P, h * w,
                              _threads(threads), ties.ctypes.data if ties is not None else None)
    assert rc == 0
    res = out[0] if a.ndim == 2 else out
    if return_ties:
        return res, (ties[0] if a.ndim == 2 else ties)
    return res


def wmc_flowmap_f32(img, threads=None):
    """H^w as iterated by the flow (canonical fp32, no tie rule)."""
    a = np.ascontiguousarray(img, dtype=np.float32)
    h, w = a.shape
    out = np.empty_like(a)
    assert lib().or_wmc_flowmap_f32(a.ctypes.data, out.ctypes.data, w, h, _threads(threads)) == 0
    return out


def flow_f32(img, iters, dt=1.0, threads=None):
    """fp32 canonical mc_flow; returns (U^iters, first_bad_iter or 0)."""
    a = np.array(img, dtype=np.float32, order="C", copy=True)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    bad = C.c_int32(0)
    rc = lib().or_flow_f32(a3.ctypes.data, w, h, w, P, h * w, int(iters), float(dt),
                           _threads(threads), C.byref(bad))
    assert rc in (0, 3), rc
    return (a3[0] if a.ndim == 2 else a3), bad.value


def _f64_work(img, inplace):
    if inplace:  # filter a C-contiguous float64 array in place (no copy of big inputs)
        assert img.dtype == np.float64 and img.flags.c_contiguous
        return img
    return np.array(img, dtype=np.float64, order="C", copy=True)


def flow_f64(img, iters, dt=1.0, threads=None, inplace=False):
    a = _f64_work(img, inplace)
    h, w = a.shape
    bad = C.c_int32(0)
    rc = lib().or_flow_f64(a.ctypes.data, w, h, int(iters), float(dt), _threads(threads),
                           C.byref(bad))
    assert rc in (0, 3), rc
    return a, bad.value


def ref_flow_f64(img, iters, dt=1.0, threads=None, inplace=False):
    L = ref_lib()
    if L is None:
        raise RuntimeError("oracle/_ref/libcf_ref.so not built")
    a = _f64_work(img, inplace)
    h, w = a.shape
    bad = C.c_int32(0)
    rc = L.ref_flow_f64(a.ctypes.data, w, h, int(iters), float(dt), _threads(threads),
                        C.byref(bad))
    assert rc in (0, 3), rc
    return a, bad.value


def ref_wmc_map_f64(img, threads=None):
    L = ref_lib()
    if L is None:
        raise RuntimeError("oracle/_ref/libcf_ref.so not built")
    a = np.ascontiguousarray(img, dtype=np.float64)
    h, w = a.shape
    out = np.empty_like(a)
    assert L.ref_wmc_map_f64(a.ctypes.data, out.ctypes.data, w, h, _threads(threads)) == 0
    return out


def u8_to_f32(q):
    q = np.ascontiguousarray(q, dtype=np.uint8)
    out = np.empty(q.shape, dtype=np.float32)
    lib().or_u8_to_f32(q.ctypes.data, out.ctypes.data, q.size)
    return out


def kernel_bank_x12():
    buf = (C.c_int32 * 72)()
    lib().or_kernel_bank_numerators(buf)
    return np.array(list(buf), dtype=np.int32).reshape(8, 3, 3)


def quantize_u8(v):
    """Save-time quantisation: rint(clamp(v, 0, 1) * 255)."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    out = np.empty(v.shape, dtype=np.uint8)
    lib().or_quantize_u8(v.ctypes.data, out.ctypes.data, v.size)
    return out


def flow_image8(img8, iters, dt=1.0, threads=None):
    """Reference for mc_flow on an interleaved 8-bit image (H,W) / (H,W,3)."""
    a = np.asarray(img8, dtype=np.uint8)
    planes = a[None] if a.ndim == 2 else np.ascontiguousarray(np.moveaxis(a, 2, 0))
    f = u8_to_f32(planes)
    out, bad = flow_f32(f, iters, dt, threads)
    q = quantize_u8(out)
    return (q[0] if a.ndim == 2 else np.ascontiguousarray(np.moveaxis(q, 0, 2))), bad


def solve_l2_area_f32(f, iters, dt, lam, threads=None, u0=None):
    """fp32 canonical solve_l2_area (A = I); returns (U^iters, bad_iter).
    u0: continue from this iterate instead of U^0 = f."""
    a = np.ascontiguousarray(f, dtype=np.float32)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    u = (np.empty_like(a3) if u0 is None
         else np.array(np.asarray(u0, np.float32).reshape(a3.shape), copy=True))
    bad = C.c_int32(0)
    rc = lib().or_solve_l2_area_f32(a3.ctypes.data, u.ctypes.data, w, h, w, P, h * w, int(iters),
                                    float(dt), float(lam), int(u0 is None), _threads(threads),
                                    C.byref(bad))
    assert rc in (0, 3), rc
    return (u[0] if a.ndim == 2 else u), bad.value


def solve_l1_area_f32(f, iters, dt, lam, alpha, threads=None, state=None):
    """fp32 canonical solve_l1_area (A = I); returns (U, d, bad_iter).
    state = (u0, d0): continue from that iterate instead of U^0 = f, d^0 = 0."""
    a = np.ascontiguousarray(f, dtype=np.float32)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    if state is None:
        u, d = np.empty_like(a3), np.empty_like(a3)
    else:
        u = np.array(np.asarray(state[0], np.float32).reshape(a3.shape), copy=True)
        d = np.array(np.asarray(state[1], np.float32).reshape(a3.shape), copy=True)
    bad = C.c_int32(0)
    rc = lib().or_solve_l1_area_f32(a3.ctypes.data, u.ctypes.data, d.ctypes.data, w, h, w, P,
                                    h * w, int(iters), float(dt), float(lam), float(alpha),
                                    int(state is None), _threads(threads), C.byref(bad))
    assert rc in (0, 3), rc
    if a.ndim == 2:
        return u[0], d[0], bad.value
    return u, d, bad.value


def l1_px(r, alpha):
    """Eq. 36 shrinkage b and Eq. 37 dual d' for one residual (fp32)."""
    b, d = C.c_float(0), C.c_float(0)
    lib().or_l1_px(float(r), float(alpha), C.byref(b), C.byref(d))
    return b.value, d.value


def fidelity(u, f=None, q=1.0):
    """Fixed-order sum |u - f|^q (f None: sum |u|^q), as cf_wmc_fidelity_f64."""
    a = np.ascontiguousarray(u, dtype=np.float32)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    b3 = None
    if f is not None:
        b3 = np.ascontiguousarray(f, dtype=np.float32).reshape(a3.shape)
    qk = 1 if q == 1.0 else (2 if q == 2.0 else (3 if q == 0.5 else 0))
    return lib().or_fidelity(a3.ctypes.data, None if b3 is None else b3.ctypes.data, w, h, w, P,
                             h * w, float(q), qk)


def wmc_energy(img, q=1.0, threads=None):
    """Fixed-order energy sum |H^w|^q of the fp32 canonical map (tie rule)."""
    m = np.ascontiguousarray(wmc_map_f32(img, threads), dtype=np.float32)
    m3 = m[None] if m.ndim == 2 else m
    P, h, w = m3.shape
    qk = 1 if q == 1.0 else (2 if q == 2.0 else (3 if q == 0.5 else 0))
    return lib().or_energy_from_map(m3.ctypes.data, w, h, P, float(q), qk)


def wmc_histogram(img, scale=255.0, lo=-256.0, width=1.0, nbins=512, threads=None):
    m = np.ascontiguousarray(wmc_map_f32(img, threads), dtype=np.float32)
    counts = np.zeros(nbins, dtype=np.int64)
    lib().or_histogram_from_map(m.ctypes.data, m.size, float(scale), float(lo), float(width),
                                int(nbins), counts.ctypes.data)
    return counts


# ---------------------------------------------------------------------------
# Vectorised restatements (oracle/wmc_fast.c): the same sequences, bit-identical
# to the scalar functions above (tests/test_oracle_fast.py), fast enough for the
# full BASELINE configurations.  On a CPU without AVX2/FMA they run the scalar
# functions instead.

def fast_supported() -> bool:
    return bool(lib().or_fast_supported())


def flow_f32_fast(img, iters, dt=1.0, threads=None, inplace=False):
    """flow_f32, vectorised; img (H, W) or (P, H, W) float32.  inplace=True
    filters a C-contiguous float32 array in place (no copy of big inputs)."""
    if not fast_supported():
        return flow_f32(img, iters, dt, threads)
    if inplace:
        a = img
        assert a.dtype == np.float32 and a.flags.c_contiguous
    else:
        a = np.array(img, dtype=np.float32, order="C", copy=True)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    bad = C.c_int32(0)
    rc = lib().or_fast_flow_f32(a3.ctypes.data, w, h, w, P, h * w, int(iters), float(dt),
                                _threads(threads), C.byref(bad))
    assert rc in (0, 3), rc
    return (a3[0] if a.ndim == 2 else a3), bad.value


def wmc_map_f32_fast(img, threads=None, return_ties=False):
    """wmc_map_f32 (tie rule included), vectorised."""
    if not fast_supported():
        return wmc_map_f32(img, threads, return_ties)
    a = np.ascontiguousarray(img, dtype=np.float32)
    a3 = a[None] if a.ndim == 2 else a
    P, h, w = a3.shape
    out = np.empty_like(a3)
    ties = np.zeros(a3.shape, dtype=np.int8) if return_ties else None
    rc = lib().or_fast_map_f32(a3.ctypes.data, out.ctypes.data, w, h, w, P, h * w,
                               _threads(threads), ties.ctypes.data if ties is not None else None)
    assert rc == 0
    res = out[0] if a.ndim == 2 else out
    if return_ties:
        return res, (ties[0] if a.ndim == 2 else ties)
    return res


def flow_f64_fast(img, iters, dt=1.0, threads=None):
    """flow_f64 (SPEC-faithful fp64), vectorised; img (H, W)."""
    if not fast_supported():
        return flow_f64(img, iters, dt, threads)
    a = np.array(img, dtype=np.float64, order="C", copy=True)
    h, w = a.shape
    bad = C.c_int32(0)
    rc = lib().or_fast_flow_f64(a.ctypes.data, w, h, int(iters), float(dt), _threads(threads),
                                C.byref(bad))
    assert rc in (0, 3), rc
    return a, bad.value


def wmc_map_f64_fast(img, threads=None):
    """wmc_map_f64 (SPEC-faithful fp64), vectorised; img (H, W)."""
    if not fast_supported():
        return wmc_map_f64(img, threads)
    a = np.ascontiguousarray(img, dtype=np.float64)
    h, w = a.shape
    out = np.empty_like(a)
    assert lib().or_fast_map_f64(a.ctypes.data, out.ctypes.data, w, h, _threads(threads)) == 0
    return out


def synth(w, h, seed, n_rects, n_discs, sigma, u8=False, threads=None):
    """The seeded synthetic image from oracle/synth_ref.c --
    byte-identical to the product's cf_synth_f32 / cf_synth_u8, without
    loading the product library (bench.py's CPU legs)."""
    out = np.empty((h, w), dtype=np.uint8 if u8 else np.float32)
    fn = lib().or_synth_u8 if u8 else lib().or_synth_f32
    rc = fn(out.ctypes.data, int(w), int(h), int(w), int(seed) & (2**64 - 1), int(n_rects),
            int(n_discs), float(sigma), _threads(threads))
    assert rc == 0
    return out


def synth_config(cfg, planes=None, threads=None):
    """Input of a BASELINE config (paper_1903_07189_b200/configs.py WmcConfig):
    (H, W) for one plane, else (P, H, W); u8 configs give uint8."""
    n = cfg.planes if planes is None else planes
    imgs = [synth(cfg.w, cfg.h, cfg.seed(p), cfg.n_rects, cfg.n_discs, cfg.sigma, cfg.u8,
                  threads) for p in range(n)]
    return imgs[0] if n == 1 and planes is None else np.stack(imgs)

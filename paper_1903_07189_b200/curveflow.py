"""Host-side mirror of the reference's operator interface for the WMC path.

The reference (arXiv 1903.07189; /root/reference/SPEC.md) defines, in namespace
``curveflow``:

* ``wmc_half_laplace(img: Image2D) -> Image2D``
* ``mc_flow(img: Image2D, cfg: FlowConfig) -> Image2D``
* ``FlowConfig{dt, iters, scheme}``
* ``kernel(name)`` / ``KernelBank`` (h1..h8)
* ``split_channels`` / ``merge_channels``
* ``solve_l2_area`` / ``solve_l1_area`` / ``SolverConfig`` / ``SolveReport``
                                                          SPEC.md:286-311

Same names, argument meaning and error behaviour here; the arithmetic runs in
the sm_100a kernels of ``libcurveflow_b200.so`` through the C-ABI
(include/curveflow/capi.h).  There is no CPU fallback: every call needs the
native library and a B200.

Images are ``torch.Tensor`` (CUDA, float32, shape (H, W) or (P, H, W) for P
channel planes) or ``numpy.ndarray`` (host; copied to the device and back --
the end-to-end path).  Values are real intensities (the reference's 0-255
scale or [0, 1]; the operator is homogeneous).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from ._lib import CF_ENONFINITE, check, lib

__all__ = [
    "FlowConfig", "FlowError", "wmc_half_laplace", "mc_flow", "mc_flow_u8", "kernel",
    "kernel_bank", "split_channels", "merge_channels", "synth_image", "sweeps_band",
    "mc_flow_image8", "wmc_energy", "wmc_histogram", "SolverConfig", "SolveReport", "solve_l2_area",
    "solve_l1_area", "solve", "data_fidelity", "max_sweeps_per_launch", "workspace_bytes",
]

_HALF = ("h1", "h2", "h3", "h4", "h5", "h6", "h7", "h8")


class FlowError(RuntimeError):
    """mc_flow instability: a non-finite value appeared."""

    def __init__(self, iteration: int):
        super().__init__(f"mc_flow: non-finite value at iteration {iteration}")
        self.iteration = iteration


@dataclass(frozen=True)
class FlowConfig:
    """SPEC.md:250-253.  dt default 1.0 for half_laplace; dt <= 1."""

    dt: float = 1.0
    iters: int = 0
    scheme: str = "half_laplace"

    def validate(self) -> None:
        if self.scheme not in ("half_laplace", "half"):
            raise NotImplementedError(
                "scheme='fd' (central-difference WMC, SPEC.md:163-170) is outside this "
                "build's hot path; only scheme='half_laplace' is provided")
        if not (self.dt > 0.0) or self.dt > 1.0:
            raise ValueError("FlowConfig.dt must satisfy 0 < dt <= 1 for half_laplace "
                             "(SPEC.md:252)")
        if int(self.iters) != self.iters or self.iters < 0:
            raise ValueError("FlowConfig.iters must be a nonnegative integer")


def _torch():
    import torch
    return torch


def _stream_ptr(torch, dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _as_planes(t):
    """(H, W) -> (1, H, W); (P, H, W) stays.  Returns (tensor3d, squeeze)."""
    if t.dim() == 2:
        return t.unsqueeze(0), True
    if t.dim() == 3:
        return t, False
    raise ValueError("image must be (H, W) or (P, H, W)")


def _precision(img, precision):
    """"fp32" (the canonical fp32 sequence) or "fp64" (the
    reference CPU path's own fp64 arithmetic, bit-identical to it, DESIGN.md
    §3.6).  None: fp64 for float64 torch tensors, fp32 otherwise."""
    if precision is None:
        torch = _torch()
        return "fp64" if isinstance(img, torch.Tensor) and img.dtype == torch.float64 else "fp32"
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    return precision


def _device_image(img, precision="fp32"):
    torch = _torch()
    dt_np, dt_t = (np.float64, torch.float64) if precision == "fp64" else (np.float32,
                                                                            torch.float32)
    if isinstance(img, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(img, dtype=dt_np)).cuda(), True
    if not isinstance(img, torch.Tensor):
        raise TypeError("image must be a torch.Tensor or numpy.ndarray")
    if not img.is_cuda:
        return img.to(dtype=dt_t).contiguous().cuda(), True
    if img.dtype != dt_t:
        raise TypeError(f"device images must be {'float64' if precision == 'fp64' else 'float32'}"
                        f" for precision={precision!r}")
    return img, False


def wmc_half_laplace(img, *, precision=None):
    """Discrete WMC map d_m; returns a new image.
    precision="fp64" (or a float64 device tensor): the reference's fp64
    arithmetic, bit-identical to the reference CPU path (cf_wmc_map_f64)."""
    torch = _torch()
    prec = _precision(img, precision)
    src, host = _device_image(img, prec)
    x, squeeze = _as_planes(src)
    x = x if x.stride(-1) == 1 else x.contiguous()
    P, H, W = x.shape
    out = torch.empty((P, H, W), dtype=src.dtype, device=x.device)
    if P and H and W:
        pitch, plane = x.stride(1), x.stride(0)
        if out.stride(1) != pitch or out.stride(0) != plane:
            x = x.contiguous()
            pitch, plane = x.stride(1), x.stride(0)
        fn = lib().cf_wmc_map_f64 if prec == "fp64" else lib().cf_wmc_map_f32
        with torch.cuda.device(x.device):
            check(fn(x.data_ptr(), out.data_ptr(), W, H, pitch, P, plane,
                     _stream_ptr(torch, x.device)), "wmc_half_laplace")
    res = out[0] if squeeze else out
    if host:
        return res.cpu().numpy() if isinstance(img, np.ndarray) else res.cpu()
    return res


def workspace_bytes(h: int, w: int, planes: int = 1) -> int:
    return int(lib().cf_wmc_filter_workspace_bytes(w, h, w, planes, w * h))


def mc_flow(img, cfg: FlowConfig, *, check_finite: bool = True, workspace=None,
            inplace: bool = False, precision=None):
    """Mean-curvature flow, scheme=half_laplace.

    Returns U^iters.  Raises FlowError(iteration) if an iterate becomes
    non-finite.  ``inplace=True`` (device tensors only)
    overwrites ``img``.  ``check_finite=False`` skips the host sync the
    diagnostic needs (the device-side check still runs).
    ``precision="fp64"`` (or a float64 device tensor): fp64 images and the
    reference's fp64 arithmetic, bit-identical to the reference CPU path
    (cf_wmc_filter_f64).
    """
    torch = _torch()
    cfg.validate()
    prec = _precision(img, precision)
    src, host = _device_image(img, prec)
    if inplace and (host or not src.is_contiguous()):
        raise ValueError("inplace=True needs a contiguous CUDA tensor")
    x = src if inplace else src.clone(memory_format=torch.contiguous_format)
    x3, squeeze = _as_planes(x)
    P, H, W = x3.shape
    if cfg.iters > 0 and P and H and W:
        f64 = prec == "fp64"
        nbytes = int((lib().cf_wmc_filter_f64_workspace_bytes if f64 else
                      lib().cf_wmc_filter_workspace_bytes)(W, H, W, P, H * W))
        if workspace is None or workspace.numel() < nbytes:
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=x3.device)
        bad = C.c_int32(0)
        fn = lib().cf_wmc_filter_f64 if f64 else lib().cf_wmc_filter_f32
        with torch.cuda.device(x3.device):
            rc = fn(x3.data_ptr(), W, H, W, P, H * W, int(cfg.iters), float(cfg.dt),
                    workspace.data_ptr(), nbytes, C.byref(bad) if check_finite else None,
                    _stream_ptr(torch, x3.device))
        if rc == CF_ENONFINITE:
            raise FlowError(bad.value)
        check(rc, "mc_flow")
    res = x3[0] if squeeze else x3
    if host:
        return res.cpu().numpy() if isinstance(img, np.ndarray) else res.cpu()
    return res


def mc_flow_u8(img_u8, cfg: FlowConfig, *, check_finite: bool = True, workspace=None, out=None,
               out_dtype: str = "f32"):
    """8-bit input widened on device as q/255 (BASELINE cfg 5), then
    mc_flow; returns float32 U^iters of the same (P, H, W) / (H, W) shape, or,
    with out_dtype="u8", the frames re-quantised on device
    (rint(clamp(U, 0, 1) * 255), the reference's save-time rounding)."""
    torch = _torch()
    cfg.validate()
    if out_dtype not in ("f32", "u8", "f64"):
        raise ValueError("out_dtype must be 'f32', 'u8' or 'f64'")
    if isinstance(img_u8, np.ndarray):
        src = torch.from_numpy(np.ascontiguousarray(img_u8, dtype=np.uint8)).cuda()
        host = True
    else:
        src, host = img_u8.contiguous(), not img_u8.is_cuda
        if host:
            src = src.cuda()
    if src.dtype != torch.uint8:
        raise TypeError("mc_flow_u8 expects uint8 input")
    s3, squeeze = _as_planes(src)
    P, H, W = s3.shape
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    if out_dtype == "u8":
        if out is None:
            out = torch.empty((P, H, W), dtype=torch.uint8, device=s3.device)
        nbytes = int(lib().cf_wmc_filter_u8_u8_workspace_bytes(W, H, P))
        need_ws = True
    elif out_dtype == "f64":  # fp64 widening q/255 + the reference's fp64 arithmetic
        if out is None:
            out = torch.empty((P, H, W), dtype=torch.float64, device=s3.device)
        nbytes = int(lib().cf_wmc_filter_f64_workspace_bytes(W, H, W, P, H * W))
        need_ws = True
    else:
        if out is None:
            out = torch.empty((P, H, W), dtype=torch.float32, device=s3.device)
        nbytes = int(lib().cf_wmc_filter_workspace_bytes(W, H, W, P, H * W))
        need_ws = cfg.iters > 0
    if need_ws and (workspace is None or workspace.numel() < nbytes):
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=s3.device)
    bad = C.c_int32(0)
    bad_ptr = C.byref(bad) if check_finite else None
    with torch.cuda.device(s3.device):
        strm = _stream_ptr(torch, s3.device)
        if out_dtype == "f64":
            rc = lib().cf_wmc_filter_u8_f64(s3.data_ptr(), W, H * W, out.data_ptr(), W, H, W, P,
                                            H * W, int(cfg.iters), float(cfg.dt), ptr(workspace),
                                            nbytes, bad_ptr, strm)
        elif out_dtype == "u8":
            rc = lib().cf_wmc_filter_u8_u8(s3.data_ptr(), W, H * W, out.data_ptr(), W, H * W, W, H,
                                           P, int(cfg.iters), float(cfg.dt), ptr(workspace),
                                           nbytes, bad_ptr, strm)
        else:
            rc = lib().cf_wmc_filter_u8_f32(s3.data_ptr(), W, H * W, out.data_ptr(), W, H, W, P,
                                            H * W, int(cfg.iters), float(cfg.dt), ptr(workspace),
                                            nbytes if workspace is not None else 0, bad_ptr, strm)
    if rc == CF_ENONFINITE:
        raise FlowError(bad.value)
    check(rc, "mc_flow_u8")
    res = out[0] if squeeze else out
    if host:
        return res.cpu().numpy() if isinstance(img_u8, np.ndarray) else res.cpu()
    return res


def mc_flow_image8(img, cfg: FlowConfig, *, check_finite: bool = True):
    """mc_flow on an interleaved 8-bit image (H, W) or (H, W, 3): widened on
    load (q/255), filtered per channel, clamped and rounded back to uint8 at
    save time.  numpy in -> numpy out; torch CUDA uint8
    in -> torch CUDA uint8 out."""
    torch = _torch()
    cfg.validate()
    host = isinstance(img, np.ndarray)
    src = torch.from_numpy(np.ascontiguousarray(img, dtype=np.uint8)).cuda() if host else \
        img.contiguous()
    if src.dtype != torch.uint8:
        raise TypeError("mc_flow_image8 expects uint8 input")
    if src.dim() == 2:
        H, W, ch = src.shape[0], src.shape[1], 1
    elif src.dim() == 3 and src.shape[2] == 3:
        H, W, ch = src.shape[0], src.shape[1], 3
    else:
        raise ValueError("unsupported channel count (SPEC.md:65): expected 1 or 3")
    out = torch.empty_like(src)
    nbytes = int(lib().cf_wmc_filter_image8_workspace_bytes(W, H, ch))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=src.device)
    bad = C.c_int32(0)
    with torch.cuda.device(src.device):
        rc = lib().cf_wmc_filter_image8(src.data_ptr(), W * ch, out.data_ptr(), W * ch, W, H, ch,
                                        int(cfg.iters), float(cfg.dt), ws.data_ptr(), nbytes,
                                        C.byref(bad) if check_finite else None,
                                        _stream_ptr(torch, src.device))
    if rc == CF_ENONFINITE:
        raise FlowError(bad.value)
    check(rc, "mc_flow_image8")
    return out.cpu().numpy() if host else out


@dataclass
class SolverConfig:
    """SPEC.md:286-289 with operator A = identity.  model: "l2_area" (Eq. 30)
    or "l1_area" (Eqs. 32-38).  report=True runs iteration by iteration and
    fills the SolveReport series, stopping early once the relative update
    ||U^{t+1} - U^t|| / ||U^t|| drops below 1e-6; report=False
    fuses up to three iterations per launch and returns the final state."""

    lam: float = 0.0
    dt: float = 0.15
    iters: int = 500
    model: str = "l2_area"
    alpha: float = 1.0
    report: bool = False

    def validate(self) -> None:
        if self.model not in ("l2_area", "l1_area"):
            raise NotImplementedError(
                f"model={self.model!r}: only 'l2_area' (SPEC.md:296) and 'l1_area' (SPEC.md:304) "
                "run on the B200 WMC path; the eps-TV baseline solver is out of scope")
        if not (self.dt > 0.0) or not np.isfinite(self.dt):
            raise ValueError("SolverConfig.dt must be > 0")
        if not (self.lam >= 0.0) or not np.isfinite(self.lam):
            raise ValueError("SolverConfig.lam must be >= 0")
        if not (self.alpha > 0.0) or not (self.alpha <= 1e30):
            raise ValueError("SolverConfig.alpha must satisfy 0 < alpha <= 1e30 (SPEC.md:288)")
        if int(self.iters) != self.iters or self.iters < 0:
            raise ValueError("SolverConfig.iters must be a nonnegative integer")


@dataclass
class SolveReport:
    """SPEC.md:290-293.  fidelity: final data term (l2: 0.5*||U - f||^2,
    l1: ||U - f||_1, fp64).  With SolverConfig.report the per-iteration series
    (fidelity, regularization = sum |H^w(U)|, total = fidelity + lam * reg)
    have one entry per iteration run and `converged` says whether the
    relative update fell below 1e-6; otherwise they are None.  dual: the
    final d of the l1 model (None for l2)."""

    image: object
    iters: int
    fidelity: float
    fidelity_series: list | None = None
    regularization_series: list | None = None
    total_series: list | None = None
    converged: bool | None = None
    dual: object = None


CONVERGED_REL_UPDATE = 1e-6


def _fidelity_dev(torch, u3, f3, q: float) -> float:
    P, H, W = u3.shape
    nbytes = int(lib().cf_wmc_reduce_workspace_bytes(W, H, P))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=u3.device)
    out = torch.empty(1, dtype=torch.float64, device=u3.device)
    check(lib().cf_wmc_fidelity_f64(u3.data_ptr(), None if f3 is None else f3.data_ptr(), W, H,
                                    W, P, H * W, float(q), out.data_ptr(), ws.data_ptr(), nbytes,
                                    _stream_ptr(torch, u3.device)), "fidelity")
    return float(out.item())


def data_fidelity(u, f=None, q: float = 1.0) -> float:
    """sum |u - f|^q (f None: sum |u|^q), fp64, fixed order (csrc/wmc_reduce.cu)."""
    torch = _torch()
    a, _ = _device_image(u)
    a3, _ = _as_planes(a.contiguous())
    b3 = None
    if f is not None:
        b, _ = _device_image(f)
        b3, _ = _as_planes(b.contiguous())
        if b3.shape != a3.shape:
            raise ValueError("u and f must have the same shape")
    with torch.cuda.device(a3.device):
        return _fidelity_dev(torch, a3, b3, q)


def _solve(f, cfg: SolverConfig, model: str) -> SolveReport:
    torch = _torch()
    cfg.validate()
    if cfg.model != model:
        raise ValueError(f"cfg.model must be {model!r}")
    src, host = _device_image(f)
    f3, squeeze = _as_planes(src.contiguous())
    P, H, W = f3.shape
    l1 = model == "l1_area"
    u = torch.empty_like(f3)
    d = torch.empty_like(f3) if l1 else None
    nbytes = int(lib().cf_wmc_solve_l1_area_workspace_bytes(W, H, W, P, H * W) if l1
                 else lib().cf_wmc_filter_workspace_bytes(W, H, W, P, H * W))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=f3.device)
    bad = C.c_int32(0)
    q = 1.0 if l1 else 2.0
    scale = 1.0 if l1 else 0.5

    def step(iters: int, init: bool) -> None:
        strm = _stream_ptr(torch, f3.device)
        if l1:
            rc = lib().cf_wmc_solve_l1_area_f32(f3.data_ptr(), u.data_ptr(), d.data_ptr(), W, H,
                                                W, P, H * W, int(iters), float(cfg.dt),
                                                float(cfg.lam), float(cfg.alpha), int(init),
                                                ws.data_ptr(), nbytes, C.byref(bad), strm)
        else:
            rc = lib().cf_wmc_solve_l2_area_f32(f3.data_ptr(), u.data_ptr(), W, H, W, P, H * W,
                                                int(iters), float(cfg.dt), float(cfg.lam),
                                                int(init), ws.data_ptr(), nbytes, C.byref(bad),
                                                strm)
        if rc == CF_ENONFINITE:
            raise FlowError(done + bad.value)
        check(rc, "solve_" + model)

    done = 0
    fid_s = reg_s = tot_s = None
    converged = None
    with torch.cuda.device(f3.device):
        if not cfg.report:
            step(int(cfg.iters), True)
            done = int(cfg.iters)
        else:
            fid_s, reg_s, tot_s = [], [], []
            converged = False
            step(0, True)                     # U^0 = f (, d^0 = 0)
            prev = u.clone()
            for _ in range(int(cfg.iters)):
                step(1, False)
                done += 1
                fid = scale * _fidelity_dev(torch, u, f3, q)
                reg = wmc_energy(u, 1.0)
                fid_s.append(fid)
                reg_s.append(reg)
                tot_s.append(fid + cfg.lam * reg)
                num = _fidelity_dev(torch, u, prev, 2.0)
                den = _fidelity_dev(torch, prev, None, 2.0)
                rel = float(np.sqrt(num) / max(np.sqrt(den), np.finfo(np.float64).tiny))
                if rel < CONVERGED_REL_UPDATE:
                    converged = True
                    break
                prev.copy_(u)
        fidelity = scale * _fidelity_dev(torch, u, f3, q)

    def out(t):
        if t is None:
            return None
        r = t[0] if squeeze else t
        if host:
            r = r.cpu().numpy() if isinstance(f, np.ndarray) else r.cpu()
        return r

    return SolveReport(image=out(u), iters=done, fidelity=fidelity, fidelity_series=fid_s,
                       regularization_series=reg_s, total_series=tot_s, converged=converged,
                       dual=out(d))


def solve_l2_area(f, cfg: SolverConfig) -> SolveReport:
    """solve_l2_area (A = I): U^0 = f,
    U <- U + dt*((f - U) + lam*H^w(U)); raises FlowError(iteration) on a
    non-finite iterate."""
    return _solve(f, cfg, "l2_area")


def solve_l1_area(f, cfg: SolverConfig) -> SolveReport:
    """solve_l1_area (A = I): U^0 = f, d^0 = 0; per iteration
    r = U - f + d, d' = clamp(r, -alpha, alpha),
    U <- U + dt*(lam*H^w(U) - (2d' - d)/alpha); raises
    FlowError(iteration) on divergence."""
    return _solve(f, cfg, "l1_area")


def solve(f, cfg: SolverConfig) -> SolveReport:
    """Dispatch on cfg.model."""
    cfg.validate()
    return _solve(f, cfg, cfg.model)


def wmc_energy(img, q: float = 1.0) -> float:
    """WMC regularisation energy sum |H^w|^q, q > 0, with the
    deterministic fixed-order reduction of SPEC.md:236 (csrc/wmc_reduce.cu)."""
    torch = _torch()
    src, _ = _device_image(img)
    x, _ = _as_planes(src.contiguous())
    P, H, W = x.shape
    nbytes = int(lib().cf_wmc_reduce_workspace_bytes(W, H, P))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        check(lib().cf_wmc_energy_f64(x.data_ptr(), W, H, W, P, H * W, float(q), out.data_ptr(),
                                      ws.data_ptr(), nbytes, _stream_ptr(torch, x.device)),
              "wmc_energy")
    return float(out.item())


def wmc_histogram(img, scale: float = 255.0, lo: float = -256.0, width: float = 1.0,
                  nbins: int = 512) -> np.ndarray:
    """Histogram of wmc_half_laplace values: bins of `width`
    from `lo` on the `scale`d values (default: the reference's 0-255 scale,
    width 1 over [-256, 256]); returns int64 counts."""
    torch = _torch()
    src, _ = _device_image(img)
    x, _ = _as_planes(src.contiguous())
    P, H, W = x.shape
    nbytes = int(lib().cf_wmc_reduce_workspace_bytes(W, H, P))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    counts = torch.empty(nbins, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        check(lib().cf_wmc_histogram(x.data_ptr(), W, H, W, P, H * W, float(scale), float(lo),
                                     float(width), int(nbins), counts.data_ptr(), ws.data_ptr(),
                                     nbytes, _stream_ptr(torch, x.device)), "wmc_histogram")
    return counts.cpu().numpy()


def max_sweeps_per_launch() -> int:
    return int(lib().cf_wmc_max_sweeps_per_launch())


def sweeps_band(src, src_row0: int, dst, dst_row0: int, h: int, y0: int, y1: int, sweeps: int,
                dt: float, iter_base: int, flag=None) -> None:
    """Row-band primitive (C-ABI cf_wmc_sweeps_band_f32): `sweeps` fused Jacobi
    sweeps producing global rows [y0, y1) of a height-h image from a band buffer
    `src` holding global rows [src_row0, src_row0 + src.shape[0])."""
    torch = _torch()
    assert src.is_cuda and dst.is_cuda and src.dtype == torch.float32 and src.is_contiguous()
    W = src.shape[1]
    with torch.cuda.device(src.device):
        check(lib().cf_wmc_sweeps_band_f32(
            src.data_ptr(), src_row0, src.shape[0], dst.data_ptr(), dst_row0, W, h, W, y0, y1,
            sweeps, float(dt), iter_base, flag.data_ptr() if flag is not None else None,
            _stream_ptr(torch, src.device)), "sweeps_band")


def kernel_bank() -> dict:
    """h1..h8 as exact rationals, [row][col]."""
    buf = (C.c_int32 * 72)()
    lib().cf_kernel_bank_x12(buf)
    bank = {}
    for i, name in enumerate(_HALF):
        bank[name] = [[Fraction(buf[i * 9 + r * 3 + c], 12) for c in range(3)] for r in range(3)]
    return bank


def kernel(name: str):
    """SPEC.md:105 kernel(name) for the half-Laplace kernels h1..h8."""
    bank = kernel_bank()
    if name not in bank:
        raise KeyError(f"kernel {name!r}: this build carries h1..h8 (the hot path); "
                       "the Laplace diagnostics k1..k4 are out of scope")
    return bank[name]


def split_channels(img: np.ndarray):
    """(H, W) -> [plane]; (H, W, 3) -> 3 planes; else format error."""
    a = np.asarray(img)
    if a.ndim == 2:
        return [a]
    if a.ndim == 3 and a.shape[2] == 3:
        return [np.ascontiguousarray(a[:, :, c]) for c in range(3)]
    raise ValueError("unsupported channel count (SPEC.md:65): expected 1 or 3")


def merge_channels(planes):
    if len(planes) == 1:
        return np.asarray(planes[0])
    if len(planes) == 3:
        return np.stack([np.asarray(p) for p in planes], axis=2)
    raise ValueError("unsupported channel count (SPEC.md:65): expected 1 or 3")


def synth_image(h: int, w: int, seed: int, n_rects: int, n_discs: int, sigma: float,
                dtype: str = "f32", threads: int = 0) -> np.ndarray:
    """Seeded synthetic image (host), DESIGN.md §6 / csrc/synth.cpp."""
    if dtype == "f32":
        out = np.empty((h, w), dtype=np.float32)
        fn = lib().cf_synth_f32
    elif dtype == "u8":
        out = np.empty((h, w), dtype=np.uint8)
        fn = lib().cf_synth_u8
    else:
        raise ValueError("dtype must be 'f32' or 'u8'")
    check(fn(out.ctypes.data, w, h, w, int(seed) & (2**64 - 1), n_rects, n_discs, float(sigma),
             threads), "synth_image")
    return out


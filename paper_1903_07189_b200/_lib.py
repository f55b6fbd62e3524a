"""ctypes binding of libcurveflow_b200.so (the C-ABI in include/curveflow/capi.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_1903_07189_b200/csrc``).  There is no fallback: if it is missing or does
not load, every entry point raises ``CurveflowLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcurveflow_b200.so")

CF_OK, CF_EINVAL, CF_ECUDA, CF_ENONFINITE, CF_ENODEV = 0, 1, 2, 3, 4


class CurveflowLibraryError(RuntimeError):
    """The native library is missing or failed to load (no CPU fallback exists)."""


_lock = threading.Lock()
_lib = None

_i32, _i64, _u64, _f32, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
_vp, _sz = C.c_void_p, C.c_size_t
_pi32 = C.POINTER(C.c_int32)

# name -> (restype, argtypes); must match include/curveflow/capi.h exactly.
SIGNATURES = {
    "cf_version": (C.c_char_p, []),
    "cf_status_string": (C.c_char_p, [C.c_int]),
    "cf_last_cuda_error": (C.c_int, []),
    "cf_wmc_map_f32": (C.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _vp]),
    "cf_wmc_filter_workspace_bytes": (_sz, [_i32, _i32, _i64, _i32, _i64]),
    "cf_wmc_filter_u8_fused": (_i32, [_vp, _i64, _i64, _i32, _i32]),
    "cf_wmc_filter_f32": (C.c_int, [_vp, _i32, _i32, _i64, _i32, _i64, _i32, _f32, _vp, _sz,
                                    _pi32, _vp]),
    "cf_wmc_filter_query_nonfinite": (C.c_int, [_vp, _pi32, _vp]),
    "cf_wmc_filter_u8_f32": (C.c_int, [_vp, _i64, _i64, _vp, _i32, _i32, _i64, _i32, _i64,
                                       _i32, _f32, _vp, _sz, _pi32, _vp]),
    "cf_wmc_solve_l2_area_f32": (C.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32, _f32,
                                           _f32, _i32, _vp, _sz, _pi32, _vp]),
    "cf_wmc_solve_l1_area_workspace_bytes": (_sz, [_i32, _i32, _i64, _i32, _i64]),
    "cf_wmc_solve_l1_area_f32": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i64, _i32, _i64, _i32,
                                           _f32, _f32, _f32, _i32, _vp, _sz, _pi32, _vp]),
    "cf_shard_plan_init": (C.c_int, [_i32, _i32, _i32, _i32, _vp]),
    "cf_wmc_filter_sharded_f32": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _f32, _pi32]),
    "cf_wmc_sweeps_band_peer_f32": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _i32, _i32, _i64, _i32,
                                              _i32, _i32, _f32, _i32, _vp, _vp, _i32, _i32, _vp,
                                              _i32, _i32, _vp]),
    "cf_device_alloc": (C.c_int, [_sz, C.POINTER(_vp)]),
    "cf_device_free": (C.c_int, [_vp]),
    "cf_device_memset": (C.c_int, [_vp, C.c_int, _sz, _vp]),
    "cf_copy": (C.c_int, [_vp, _vp, _sz, _vp]),
    "cf_ipc_mem_handle": (C.c_int, [_vp, _vp]),
    "cf_ipc_open_mem": (C.c_int, [_vp, C.POINTER(_vp)]),
    "cf_ipc_close_mem": (C.c_int, [_vp]),
    "cf_ipc_event_create": (C.c_int, [C.POINTER(_vp)]),
    "cf_ipc_event_handle": (C.c_int, [_vp, _vp]),
    "cf_ipc_open_event": (C.c_int, [_vp, C.POINTER(_vp)]),
    "cf_event_record": (C.c_int, [_vp, _vp]),
    "cf_stream_wait_event": (C.c_int, [_vp, _vp]),
    "cf_event_destroy": (C.c_int, [_vp]),
    "cf_stream_synchronize": (C.c_int, [_vp]),
    "cf_wmc_max_sweeps_per_launch": (_i32, []),
    "cf_wmc_filter_launches": (_i32, [_i32, _i32, _i32, _i32]),
    "cf_wmc_filter_sweeps_per_launch": (_i32, [_i32, _i32, _i32]),
    "cf_wmc_sweeps_band_f32": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _i32, _i32, _i64, _i32,
                                         _i32, _i32, _f32, _i32, _vp, _vp]),
    "cf_image8_to_planes_f32": (C.c_int, [_vp, _i64, _i32, _i32, _i32, _vp, _i64, _i64, _vp]),
    "cf_planes_f32_to_image8": (C.c_int, [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _vp]),
    "cf_wmc_filter_u8_u8_workspace_bytes": (_sz, [_i32, _i32, _i32]),
    "cf_wmc_filter_u8_u8": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _i32,
                                      _f32, _vp, _sz, _pi32, _vp]),
    "cf_wmc_filter_image8_workspace_bytes": (_sz, [_i32, _i32, _i32]),
    "cf_wmc_filter_image8_fused": (_i32, [_vp, _i64, _i32, _i32, _i32]),
    "cf_wmc_filter_image8": (C.c_int, [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _f32, _vp,
                                       _sz, _pi32, _vp]),
    "cf_wmc_reduce_workspace_bytes": (_sz, [_i32, _i32, _i32]),
    "cf_wmc_energy_f64": (C.c_int, [_vp, _i32, _i32, _i64, _i32, _i64, _f64, _vp, _vp, _sz, _vp]),
    "cf_wmc_histogram": (C.c_int, [_vp, _i32, _i32, _i64, _i32, _i64, _f32, _f32, _f32, _i32,
                                   _vp, _vp, _sz, _vp]),
    "cf_wmc_fidelity_f64": (C.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _f64, _vp, _vp,
                                      _sz, _vp]),
    "cf_synth_f32": (C.c_int, [_vp, _i32, _i32, _i64, _u64, _i32, _i32, _f64, _i32]),
    "cf_synth_u8": (C.c_int, [_vp, _i32, _i32, _i64, _u64, _i32, _i32, _f64, _i32]),
    "cf_kernel_bank_x12": (None, [_pi32]),
    # the SPEC-faithful fp64 path (csrc/wmc_f64.cu)
    "cf_wmc_map_f64": (C.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, _i64, _vp]),
    "cf_wmc_filter_f64_workspace_bytes": (_sz, [_i32, _i32, _i64, _i32, _i64]),
    "cf_wmc_filter_f64": (C.c_int, [_vp, _i32, _i32, _i64, _i32, _i64, _i32, _f64, _vp, _sz,
                                    _pi32, _vp]),
    "cf_wmc_filter_u8_f64": (C.c_int, [_vp, _i64, _i64, _vp, _i32, _i32, _i64, _i32, _i64,
                                       _i32, _f64, _vp, _sz, _pi32, _vp]),
    "cf_wmc_filter_f64_query_nonfinite": (C.c_int, [_vp, _pi32, _vp]),
}


CF_MAX_PARTS = 64


class CfShardPlan(C.Structure):
    """cf_shard_plan (include/curveflow/capi.h)."""
    _fields_ = [("h", _i32), ("w", _i32), ("parts", _i32), ("k", _i32),
                ("row0", _i32 * CF_MAX_PARTS), ("row1", _i32 * CF_MAX_PARTS),
                ("top", _i32 * CF_MAX_PARTS), ("bot", _i32 * CF_MAX_PARTS),
                ("rows", _i32 * CF_MAX_PARTS)]


def lib():
    """Load (once) and return the native library; raise if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CurveflowLibraryError(
                    f"{LIB_PATH} not built; run __graft_entry__.build() "
                    "(there is no CPU fallback for the WMC path)")
            try:
                L = C.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover - environment specific
                raise CurveflowLibraryError(f"cannot load {LIB_PATH}: {e}") from e
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


class CurveflowError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        L = lib()
        msg = L.cf_status_string(status).decode()
        if status == CF_ECUDA:
            msg += f" (cudaError {L.cf_last_cuda_error()})"
        super().__init__(f"{what}: {msg}" if what else msg)
        self.status = status


def check(status: int, what: str = "") -> None:
    if status != CF_OK:
        raise CurveflowError(status, what)

"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/curveflow/capi.h declares, validates arguments before touching CUDA,
and its host-only pieces (generator, kernel bank, schedule) behave."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1903_07189_b200 as cf
from paper_1903_07189_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "curveflow", "capi.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"CF_API\s+[\w\s\*]+?\b(cf_\w+)\s*\(", txt)))


def test_header_and_binding_agree():
    syms = declared_symbols()
    assert len(syms) >= 14
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    L = cf.lib()
    for s in declared_symbols():
        assert getattr(L, s) is not None
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s
    # internal symbols are hidden (only the C-ABI is exported)
    assert not re.search(r"\bT _ZN3cfk", out)


def test_version_and_status():
    L = cf.lib()
    assert b"sm_100a" in L.cf_version()
    for st in range(5):
        assert len(L.cf_status_string(st)) > 0


def test_invalid_arguments_rejected_before_cuda():
    L = cf.lib()
    EINVAL = _lib.CF_EINVAL
    dummy = C.c_void_p(16)
    assert L.cf_wmc_map_f32(None, dummy, 4, 4, 4, 1, 16, None) == EINVAL
    assert L.cf_wmc_map_f32(dummy, dummy, 4, 4, 4, 1, 16, None) == EINVAL      # aliasing
    assert L.cf_wmc_map_f32(dummy, C.c_void_p(32), 0, 4, 4, 1, 16, None) == EINVAL
    assert L.cf_wmc_map_f32(dummy, C.c_void_p(32), 5, 4, 4, 1, 16, None) == EINVAL  # pitch<w
    ws = cf.lib().cf_wmc_filter_workspace_bytes(4, 4, 4, 1, 16)
    assert ws >= 256 + 64
    for dt in (0.0, -1.0, 1.5, float("nan")):
        assert L.cf_wmc_filter_f32(dummy, 4, 4, 4, 1, 16, 3, dt, dummy, ws, None, None) == EINVAL
    assert L.cf_wmc_filter_f32(dummy, 4, 4, 4, 1, 16, -1, 1.0, dummy, ws, None, None) == EINVAL
    assert L.cf_wmc_filter_f32(dummy, 4, 4, 4, 1, 16, 3, 1.0, dummy, ws - 1, None, None) == EINVAL
    assert L.cf_wmc_filter_f32(dummy, 4, 4, 4, 1, 16, 0, 1.0, None, 0, None, None) == 0  # identity
    assert L.cf_wmc_sweeps_band_f32(dummy, 0, 4, dummy, 0, 4, 4, 4, 0, 4, 9, 1.0, 0, None,
                                    None) == EINVAL                               # sweeps > max
    assert L.cf_wmc_sweeps_band_f32(dummy, 2, 2, dummy, 0, 4, 8, 4, 0, 4, 2, 1.0, 0, None,
                                    None) == EINVAL                               # src too short


@pytest.mark.parametrize("w,h,planes,levels", [(1024, 1024, 1, 2), (2048, 2048, 1, 2),
                                               (16384, 16384, 1, 2), (1920, 1080, 256, 2),
                                               (3840, 2160, 3, 2)])
def test_filter_schedule_is_even(w, h, planes, levels):
    """Sweeps per launch; an even launch count for iters >= 2
    so the ping-pong ends in the caller's buffer."""
    L = cf.lib()
    assert L.cf_wmc_filter_sweeps_per_launch(w, h, planes) == levels
    assert L.cf_wmc_filter_sweeps_per_launch(0, h, planes) == 0
    assert L.cf_wmc_filter_launches(w, h, planes, 0) == 0
    assert L.cf_wmc_filter_launches(w, h, planes, 1) == 1
    for it in (2, 3, 5, 20, 50, 99, 100, 200):
        n = L.cf_wmc_filter_launches(w, h, planes, it)
        assert n % 2 == 0 and n >= it / levels and n <= it


def test_generator_deterministic_and_in_range():
    a = cf.synth_image(123, 257, seed=42, n_rects=20, n_discs=20, sigma=0.1, threads=1)
    for t in (2, 7, 0):
        assert np.array_equal(cf.synth_image(123, 257, 42, 20, 20, 0.1, threads=t), a)
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() <= 1
    b = cf.synth_image(123, 257, seed=43, n_rects=20, n_discs=20, sigma=0.1)
    assert not np.array_equal(a, b)
    q = cf.synth_image(123, 257, seed=42, n_rects=20, n_discs=20, sigma=0.1, dtype="u8")
    assert q.dtype == np.uint8
    assert np.abs(q / 255.0 - a).max() <= 0.5 / 255 + 1e-6
    # noise level: sigma of the residual from a 3x3 median is ~ the configured sigma
    flat = cf.synth_image(256, 256, seed=1, n_rects=0, n_discs=0, sigma=0.05)
    resid = flat[1:-1, 1:-1] - 0.25 * (flat[:-2, 1:-1] + flat[2:, 1:-1] + flat[1:-1, :-2]
                                       + flat[1:-1, 2:])
    assert 0.035 < resid.std() / np.sqrt(1.25) < 0.065


def test_python_api_validation():
    with pytest.raises(ValueError):
        cf.FlowConfig(dt=1.5, iters=3).validate()
    with pytest.raises(ValueError):
        cf.FlowConfig(dt=0.5, iters=-1).validate()
    with pytest.raises(NotImplementedError):
        cf.FlowConfig(scheme="fd", iters=3).validate()
    with pytest.raises(KeyError):
        cf.kernel("k4")
    rgb = np.random.default_rng(0).integers(0, 255, (2, 2, 3)).astype(np.uint8)
    planes = cf.split_channels(rgb)
    assert len(planes) == 3 and np.array_equal(cf.merge_channels(planes), rgb)
    assert len(cf.split_channels(rgb[:, :, 0])) == 1
    with pytest.raises(ValueError):
        cf.split_channels(np.zeros((2, 2, 4)))


def test_product_has_no_oracle_dependency():
    """The shipped package never imports or links the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_1903_07189_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", "Makefile")):
                path = os.path.join(dirpath, f)
                if f.endswith(".py"):
                    import ast
                    for node in ast.walk(ast.parse(open(path).read())):
                        if isinstance(node, ast.Import):
                            assert not any("oracle" in a.name for a in node.names), f
                        if isinstance(node, ast.ImportFrom):
                            assert "oracle" not in (node.module or ""), f
                else:
                    for line in open(path):
                        if line.lstrip().startswith("#include") or f == "Makefile":
                            assert "oracle" not in line, (f, line)


def test_cpp_cli_built():
    exe = os.path.join(os.path.dirname(_lib.LIB_PATH), "curveflow_b200")
    assert os.access(exe, os.X_OK)
    r = __import__("subprocess").run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr


def test_shard_plan_follows_for_rows():
    """cf_shard_plan_init: parallel.hpp:36 ceil-div bands, k halo rows."""
    from paper_1903_07189_b200 import sharded
    for h, parts, k in [(10, 4, 1), (16384, 8, 3), (100, 3, 2), (7, 1, 4)]:
        pl = sharded.plan(h, 33, parts, k)
        assert [(pl.row0[p], pl.row1[p]) for p in range(parts)] == sharded.band_bounds(h, parts)
        for p in range(parts):
            assert pl.top[p] == (k if p > 0 else 0) and pl.bot[p] == (k if p < parts - 1 else 0)
            assert pl.rows[p] == pl.top[p] + pl.row1[p] - pl.row0[p] + pl.bot[p]
    L = cf.lib()
    import ctypes as C
    from paper_1903_07189_b200._lib import CF_EINVAL as EINVAL, CfShardPlan
    pl = CfShardPlan()
    assert L.cf_shard_plan_init(3, 8, 4, 1, C.addressof(pl)) == EINVAL    # parts > h
    assert L.cf_shard_plan_init(10, 8, 4, 3, C.addressof(pl)) == EINVAL   # band < k rows
    assert L.cf_shard_plan_init(10, 8, 2, 9, C.addressof(pl)) == EINVAL   # k > max sweeps
    assert L.cf_shard_plan_init(10, 8, 65, 1, C.addressof(pl)) == EINVAL  # > CF_MAX_PARTS
    assert L.cf_wmc_filter_sharded_f32(None, None, None, None, None, None, 3, 1.0, None) == EINVAL

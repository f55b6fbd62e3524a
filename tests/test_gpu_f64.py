"""The SPEC-faithful fp64 path (csrc/wmc_f64.cu) against the
reference CPU path: BIT-exact, not a tolerance.

The reference evaluates in fp64.  cf_wmc_map_f64 /
cf_wmc_filter_f64 / cf_wmc_filter_u8_f64 follow its arithmetic operation for
operation, so their outputs must equal, bit for bit:
  * the oracle's fp64 SPEC-faithful restatement (oracle/wmc_oracle.c
    or_wmc_map_f64 / or_flow_f64, and its vectorised twin wmc_fast.c pinned
    to it by tests/test_oracle_fast.py), and
  * the same restatement run on the reference's own executor
    (oracle/_ref/libcf_ref.so, parallel.hpp:26-47) where that build exists,
on odd shapes, pitches, planes, dt < 1, odd iteration counts, the non-finite
abort, and every BASELINE config at full size (cfg4: the whole 16384^2 x 200
run).  Records go to $CF_PARITY_LOG when set.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1903_07189_b200 as cf
from paper_1903_07189_b200.configs import CONFIGS, SUPPLEMENTAL

pytestmark = pytest.mark.gpu


def _record(name, **kv):
    kv = {"config": name, "precision": "fp64", **kv}
    print(json.dumps(kv))
    path = os.environ.get("CF_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kv) + "\n")


def _same(got, ref, what):
    g = np.ascontiguousarray(got, dtype=np.float64).view(np.uint64)
    r = np.ascontiguousarray(ref, dtype=np.float64).view(np.uint64)
    n = int(np.count_nonzero(g != r))
    assert n == 0, f"{what}: {n} of {g.size} pixels differ from the fp64 reference path"


def _img(h, w, seed, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (h, w))


def _ref_map(img):
    ref = oracle.wmc_map_f64(img)
    if oracle.ref_lib() is not None:
        _same(oracle.ref_wmc_map_f64(img), ref, "oracle vs _ref (map)")
    return ref


def _ref_flow(img, iters, dt):
    ref, bad = oracle.flow_f64(img, iters, dt)
    if oracle.ref_lib() is not None:
        r2, b2 = oracle.ref_flow_f64(img, iters, dt)
        assert b2 == bad
        if bad == 0:
            _same(r2, ref, "oracle vs _ref (flow)")
    return ref, bad


@pytest.mark.parametrize("h,w", [(1, 1), (1, 7), (5, 1), (2, 2), (3, 33), (37, 65), (64, 64),
                                 (129, 257)])
def test_map_f64_shapes(h, w):
    img = _img(h, w, h * 1000 + w)
    got = cf.wmc_half_laplace(torch.from_numpy(img).cuda()).cpu().numpy()
    _same(got, _ref_map(img), f"map {h}x{w}")


def test_map_f64_precision_keyword_numpy():
    img = _img(40, 50, 3)
    got = cf.wmc_half_laplace(img, precision="fp64")
    assert got.dtype == np.float64
    _same(got, _ref_map(img), "map via precision='fp64'")


@pytest.mark.parametrize("h,w,iters,dt", [(1, 1, 3, 1.0), (7, 5, 1, 1.0), (33, 47, 2, 0.5),
                                          (64, 80, 5, 0.37), (101, 67, 12, 1.0),
                                          (256, 256, 9, 0.8)])
def test_flow_f64_shapes(h, w, iters, dt):
    img = _img(h, w, iters * 7 + h)
    got = cf.mc_flow(torch.from_numpy(img).cuda(), cf.FlowConfig(dt=dt, iters=iters)).cpu().numpy()
    ref, bad = _ref_flow(img, iters, dt)
    assert bad == 0
    _same(got, ref, f"flow {h}x{w} x{iters} dt={dt}")


def test_flow_f64_planes_pitch_graph_replay():
    # 3 planes in one call, repeated (the second and third identical calls
    # replay the cached graph); each plane equals the reference's filter
    imgs = np.stack([_img(45, 70, s) for s in range(3)])
    cfg = cf.FlowConfig(dt=1.0, iters=6)
    x = torch.from_numpy(imgs).cuda()
    ws = torch.empty(int(cf.lib().cf_wmc_filter_f64_workspace_bytes(70, 45, 70, 3, 45 * 70)),
                     dtype=torch.uint8, device="cuda")
    for _ in range(3):
        y = x.clone()
        cf.mc_flow(y, cfg, inplace=True, workspace=ws)
        for p in range(3):
            _same(y[p].cpu().numpy(), _ref_flow(imgs[p], 6, 1.0)[0], f"plane {p}")


def test_flow_f64_nonfinite_names_iteration():
    # values near the fp64 maximum overflow within a few iterations; the
    # first bad iteration must be the reference's
    img = _img(20, 24, 11, -1.0, 1.0) * 1.7e308
    _, bad = _ref_flow(img, 10, 1.0)
    assert bad > 0
    with pytest.raises(cf.FlowError) as e:
        cf.mc_flow(torch.from_numpy(img).cuda(), cf.FlowConfig(dt=1.0, iters=10))
    assert e.value.iteration == bad


def test_u8_f64_widening_every_byte():
    q = np.arange(256, dtype=np.uint8).reshape(16, 16)
    got = cf.mc_flow_u8(torch.from_numpy(q).cuda(), cf.FlowConfig(dt=1.0, iters=0),
                        out_dtype="f64").cpu().numpy()
    _same(got, q.astype(np.float64) / 255.0, "q/255 in fp64")


# ------------------------------------------------- the BASELINE configs ---
def _input(c):
    imgs = [cf.synth_image(c.h, c.w, c.seed(p), c.n_rects, c.n_discs, c.sigma,
                           dtype="u8" if c.u8 else "f32", threads=0) for p in range(c.planes)]
    return np.stack(imgs) if c.planes > 1 else imgs[0]


@pytest.mark.parametrize("name", ["cfg1", "cfg1_16k"])
def test_f64_map_config(name):
    c = CONFIGS.get(name) or SUPPLEMENTAL[name]
    img = _input(c).astype(np.float64)
    got = cf.wmc_half_laplace(torch.from_numpy(img).cuda()).cpu().numpy()
    ref = oracle.wmc_map_f64_fast(img)
    if c.h <= 1024:
        _same(ref, _ref_map(img), "fast oracle vs scalar")
    _same(got, ref, f"{name} fp64 map")
    _record(name, op="wmc_half_laplace", bitexact_fp64=True, pixels=int(img.size))


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_f64_filter_config(name):
    c = CONFIGS[name]
    img = _input(c).astype(np.float64)
    x = torch.from_numpy(img).cuda()
    got = cf.mc_flow(x, cf.FlowConfig(dt=c.dt, iters=c.iters), inplace=True).cpu().numpy()
    del x
    planes = img if img.ndim == 3 else img[None]
    gots = got if got.ndim == 3 else got[None]
    for p in range(planes.shape[0]):
        ref, bad = oracle.flow_f64_fast(planes[p], c.iters, c.dt)
        assert bad == 0
        _same(gots[p], ref, f"{name} fp64 filter, plane {p}")
    if name == "cfg2":  # the scalar restatement and the reference executor too
        _same(got, _ref_flow(img, c.iters, c.dt)[0], "cfg2 vs scalar / _ref")
    _record(name, op="mc_flow", bitexact_fp64=True, pixels=int(img.size), iters=c.iters)


def test_f64_filter_cfg5_u8():
    c = CONFIGS["cfg5"]
    frames = _input(c)  # (256, 1080, 1920) u8
    got = cf.mc_flow_u8(torch.from_numpy(frames).cuda(), cf.FlowConfig(dt=c.dt, iters=c.iters),
                        out_dtype="f64").cpu().numpy()
    for i in range(c.planes):
        ref, bad = oracle.flow_f64_fast(frames[i].astype(np.float64) / 255.0, c.iters, c.dt)
        assert bad == 0
        _same(got[i], ref, f"cfg5 fp64 filter, frame {i}")
    _record("cfg5", op="mc_flow_u8", bitexact_fp64=True, pixels=int(frames.size), iters=c.iters)

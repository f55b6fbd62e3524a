"""Minimal compute-sanitizer target without torch: the map (flat + streaming,
edge and interior warps), the filter, the u8 paths, the fp64 path and the
reductions through the C-ABI on small images (ctypes + numpy only)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1903_07189_b200._lib import lib  # noqa: E402

L = lib()


def dev(nbytes):
    p = C.c_void_p()
    assert L.cf_device_alloc(max(nbytes, 4), C.byref(p)) == 0
    return p.value


def h2d(arr):
    a = np.ascontiguousarray(arr)
    p = dev(a.nbytes)
    assert L.cf_copy(p, a.ctypes.data, a.nbytes, None) == 0
    return p


rng = np.random.default_rng(0)
for (h, w) in [(1, 1), (3, 7), (37, 65), (600, 1000), (130, 700)]:
    img = rng.random((h, w), dtype=np.float32)
    src, dst = h2d(img), dev(img.nbytes)
    assert L.cf_wmc_map_f32(src, dst, w, h, w, 1, h * w, None) == 0      # flat / streaming
    nb = L.cf_wmc_filter_workspace_bytes(w, h, w, 1, h * w)
    ws = dev(nb)
    bad = C.c_int32(0)
    assert L.cf_wmc_filter_f32(src, w, h, w, 1, h * w, 5, 1.0, ws, nb, C.byref(bad), None) == 0
    rb = L.cf_wmc_reduce_workspace_bytes(w, h, 1)
    rws, out = dev(rb), dev(8)
    assert L.cf_wmc_energy_f64(src, w, h, w, 1, h * w, 1.0, out, rws, rb, None) == 0
    cnt = dev(512 * 8)
    assert L.cf_wmc_histogram(src, w, h, w, 1, h * w, 255.0, -256.0, 1.0, 512, cnt, rws, rb,
                              None) == 0
    img64 = img.astype(np.float64)
    s64, d64 = h2d(img64), dev(img64.nbytes)
    assert L.cf_wmc_map_f64(s64, d64, w, h, w, 1, h * w, None) == 0
    nb64 = L.cf_wmc_filter_f64_workspace_bytes(w, h, w, 1, h * w)
    ws64 = dev(nb64)
    assert L.cf_wmc_filter_f64(s64, w, h, w, 1, h * w, 3, 1.0, ws64, nb64, C.byref(bad), None) == 0
q = (rng.random((2, 40, 64)) * 255).astype(np.uint8)
qs = h2d(q)
fo = dev(q.size * 4)
nb = L.cf_wmc_filter_workspace_bytes(64, 40, 64, 2, 40 * 64)
ws = dev(nb)
assert L.cf_wmc_filter_u8_f32(qs, 64, 40 * 64, fo, 64, 40, 64, 2, 40 * 64, 4, 1.0, ws, nb,
                              C.byref(bad), None) == 0
nb8 = L.cf_wmc_filter_u8_u8_workspace_bytes(64, 40, 2)
ws8, o8 = dev(nb8), dev(q.size)
assert L.cf_wmc_filter_u8_u8(qs, 64, 40 * 64, o8, 64, 40 * 64, 64, 40, 2, 4, 1.0, ws8, nb8,
                             C.byref(bad), None) == 0
assert L.cf_stream_synchronize(None) == 0
print("sanitize_min ok")

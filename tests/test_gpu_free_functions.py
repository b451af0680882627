"""Device evaluation of the reference's public free functions vs the oracle, bit-exact,
plus the reference's own KATs (test_tsdf_integrator.cpp:12-109) on the device."""
import ctypes

import numpy as np
import pytest

from paper_1611_03631_b200 import VOXEL_DTYPE, WeightMode, measurement_weight, projective_distance, raycast
from paper_1611_03631_b200 import update_tsdf_voxels
from paper_1611_03631_b200._capi import VxgVoxel
from oracle_bindings import oracle_lib

pytestmark = pytest.mark.gpu


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def test_projective_distance_kats(gpu):
    x = np.array([[0, 0, 2], [0, 0, 1], [0, 0, 2.5]], np.float32)
    p = np.array([[0, 0, 2]] * 3, np.float32)
    s = np.zeros((3, 3), np.float32)
    out = projective_distance(x, p, s)
    assert out[0] == 0.0
    assert abs(out[1] - 1.0) < 1e-5 and abs(out[2] + 0.5) < 1e-5


def test_projective_distance_random(gpu):
    rng = np.random.default_rng(1)
    n = 20000
    x, p, s = (rng.uniform(-5, 5, (n, 3)).astype(np.float32) for _ in range(3))
    out = projective_distance(x, p, s)
    L = oracle_lib()
    ref = np.array([L.vxo_projective_distance(_fp(x[i]), _fp(p[i]), _fp(s[i])) for i in range(n)], np.float32)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_measurement_weight(gpu):
    t, e = 0.4, 0.1
    assert measurement_weight(WeightMode.kConstant, 3.0, 0.2, t, e)[0] == 1.0
    assert abs(measurement_weight(WeightMode.kInverseZ2, 2.0, 0.0, t, e)[0] - 0.25) < 1e-6
    w = lambda d: measurement_weight(WeightMode.kInverseZ2Dropoff, 1.0, d, t, e)[0]
    assert abs(w(-t)) < 1e-5 and abs(w(-(t + e) / 2) - 0.5) < 1e-5 and abs(w(0.05) - 1.0) < 1e-5
    assert w(-t - 0.01) == 0.0
    rng = np.random.default_rng(2)
    z = rng.uniform(0.05, 20, 5000).astype(np.float32)
    d = rng.uniform(-0.6, 0.6, 5000).astype(np.float32)
    L = oracle_lib()
    for mode in WeightMode:
        out = measurement_weight(mode, z, d, t, e)
        ref = np.array([L.vxo_measurement_weight(int(mode), float(z[i]), float(d[i]), t, e) for i in range(len(z))],
                       np.float32)
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32)), mode


def test_update_voxel_random_folds(gpu):
    """Sequential folds incl. weight clamping and colour rounding, bit-exact."""
    rng = np.random.default_rng(3)
    nv, per = 500, 40
    starts = np.arange(0, nv * per + 1, per, dtype=np.uint64)
    d = rng.uniform(-1, 1, nv * per).astype(np.float32)
    w = rng.uniform(0.0, 300, nv * per).astype(np.float32)
    w[::7] = 0.0
    rgb = rng.integers(0, 256, (nv * per, 3), dtype=np.uint8)
    v0 = np.zeros(nv, VOXEL_DTYPE)
    out = update_tsdf_voxels(v0, starts, d, w, 0.4, 1000.0, rgb)
    L = oracle_lib()
    for i in range(nv):
        vx = VxgVoxel(0.0, 0.0, 0, 0, 0, 0)
        for j in range(int(starts[i]), int(starts[i + 1])):
            c = np.ascontiguousarray(rgb[j])
            L.vxo_update_voxel(ctypes.byref(vx), float(d[j]), float(w[j]), 0.4, 1000.0, c.ctypes.data_as(ctypes.c_void_p))
        assert np.float32(vx.distance).view(np.uint32) == out[i]["distance"].view(np.uint32)
        assert np.float32(vx.weight).view(np.uint32) == out[i]["weight"].view(np.uint32)
        assert (vx.r, vx.g, vx.b) == (out[i]["r"], out[i]["g"], out[i]["b"])


def test_raycast_random(gpu):
    """Exact DDA incl. axis-aligned rays and boundary starts: same voxel sequence."""
    rng = np.random.default_rng(4)
    n = 3000
    v = 0.1
    start = rng.uniform(-3, 3, (n, 3)).astype(np.float32)
    end = (start + rng.uniform(-2, 2, (n, 3))).astype(np.float32)
    end[::5, 1] = start[::5, 1]          # axis-aligned components
    start[::7] = np.round(start[::7] / v) * v  # starts on voxel boundaries
    walks = raycast(start, end, v)
    L = oracle_lib()
    for i in range(n):
        buf = np.zeros((4096, 3), np.int32)
        k = L.vxo_raycast(_fp(start[i]), _fp(end[i]), v, buf.ctypes.data_as(ctypes.c_void_p), 4096)
        assert np.array_equal(walks[i], buf[:k]), i
        gs, ge = np.floor(start[i] / np.float32(v)), np.floor(end[i] / np.float32(v))
        assert k == int(np.abs(ge - gs).sum()) + 1  # always span+1 voxels


def test_fast_fold_selftest(gpu):
    """The apply kernel's fast fold (shared reciprocal, colour-stationarity
    skip) must equal the reference-order update_tsdf_voxel bit-for-bit:
    2^28 random divisions over exponents [-70, 70] and 20k random fold
    sequences of 2000 steps (incl. weight saturation)."""
    from paper_1611_03631_b200._capi import check, lib
    out = (ctypes.c_uint64 * 2)()
    check(lib().vxg_selftest_fold(0, 1 << 28, 20000, 2000, 12345, out))
    assert out[0] == 0, f"{out[0]} division mismatches"
    assert out[1] == 0, f"{out[1]} fold-sequence mismatches"


@pytest.mark.parametrize("n", [1, 31, 4095, 4096, 4097, 8193, 70_001, 1_000_003, 20_000_001])
def test_device_primitives_selftest(gpu, n):
    """The in-house prefix sums and pair sorts (vxg_sort.cuh) against the
    host at tile-boundary sizes, for both sort tile shapes (inputs under / over
    16 M items), 32- and 64-bit keys, ascending and descending, with ties (the
    sorts must be stable)."""
    from paper_1611_03631_b200 import TsdfLayer
    from paper_1611_03631_b200._capi import check, lib
    layer = TsdfLayer(0.05, 16)
    for bits, desc in ((8, 0), (21, 0), (32, 0), (46, 0), (64, 1), (19, 1)):
        if n > 2_000_000 and (bits, desc) not in ((32, 0), (46, 0)):
            continue
        out = (ctypes.c_uint64 * 4)()
        check(lib().vxg_selftest_prims(layer.handle, n, bits, desc, 777 + n + bits, out))
        assert list(out) == [0, 0, 0, 0], f"n={n} bits={bits} desc={desc}: mismatches {list(out)}"

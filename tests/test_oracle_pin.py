"""CPU: pins the oracle restatement (oracle/vxf_oracle.cpp) to the reference.

* the reference's own doctest suites for this path run against the
  unmodified reference sources (oracle/_ref/unit_tests_ref, built with
  oracle/eigen_shim + oracle/doctest_shim);
* oracle vs the shim-compiled reference (oracle/_ref/libvxfref.so): bit-exact
  VXBLX bytes and counters on seeded scans over every merge x weight mode,
  random poses and all configs; free functions on random inputs;
* oracle vs the committed golden fixtures (generated from the reference).
_ref only exists where /root/reference was present at build time; the golden
fixtures pin the oracle everywhere else.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from golden_io import fixtures, load
from oracle_bindings import REF_TESTS, OracleLayer, RefLayer, oracle_lib, ref_available, ref_lib
from paper_1611_03631_b200 import MergeMode, TsdfConfig, WeightMode
from paper_1611_03631_b200 import workload as W
from paper_1611_03631_b200._capi import VxgVoxel

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference here)")


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="oracle/_ref/unit_tests_ref not built")
def test_reference_doctests_pass_on_shim_build():
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0 | assertions:" in r.stdout and "test cases: 16" in r.stdout, r.stdout


@pytest.mark.parametrize("path", fixtures(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_golden(path):
    meta, cfg, frames, expected = load(path)
    ora = OracleLayer(cfg, meta["voxel_size"], meta["vps"])
    stats = [list(ora.integrate(x, c, p)) for (x, c, p) in frames]
    assert stats == [list(s) for s in meta["stats"]]
    assert ora.save_bytes() == expected


def _random_pose(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                  [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                  [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
    t = rng.uniform(-2, 2, 3)
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32).reshape(12)


@needs_ref
@pytest.mark.parametrize("merge", list(MergeMode))
@pytest.mark.parametrize("weight", list(WeightMode))
def test_oracle_vs_reference_random_scans(merge, weight):
    rng = np.random.default_rng(100 + 3 * int(merge) + int(weight))
    v = float(rng.choice([0.05, 0.1, 0.13]))
    cfg = TsdfConfig.for_voxel_size(v)
    cfg.merge_mode, cfg.weight_mode = merge, weight
    cfg.max_weight = float(rng.choice([20.0, 1e4]))
    ora, ref = OracleLayer(cfg, v, 8), RefLayer(cfg, v, 8)
    for _ in range(3):
        n = int(rng.integers(50, 800))
        pts = rng.normal(size=(n, 3)).astype(np.float32) * np.float32(1.5)
        rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8) if rng.random() < 0.7 else None
        pose = _random_pose(rng)
        assert ora.integrate(pts, rgb, pose) == ref.integrate(pts, rgb, pose)
    assert ora.save_bytes() == ref.save_bytes()


@needs_ref
@pytest.mark.parametrize("cfg_id", [0, 1, 2, 3])
def test_oracle_vs_reference_configs(cfg_id):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    ora, ref = OracleLayer(cfg, wc.voxel_size, wc.vps), RefLayer(cfg, wc.voxel_size, wc.vps)
    for f in range(2 if cfg_id else 1):
        x, c, p = W.frame(cfg_id, 13 * f + 1, 0.12)
        assert ora.integrate(x, c, p) == ref.integrate(x, c, p)
    assert ora.save_bytes() == ref.save_bytes()


@needs_ref
def test_config_validation_messages_match():
    O, R = oracle_lib(), ref_lib()
    for tr, eps, wmax, mn, mx in [(0.1, 0.1, 1e4, 0.05, 5), (0.4, 0.1, 0, 0.05, 5), (0.4, 0.1, 1, 5, 5),
                                  (0.4, -1, 1, 0, 5), (0.4, 0.1, 1, -1, 5), (0.4, 0.1, 1e4, 0.05, 10)]:
        c = TsdfConfig(truncation=tr, dropoff_epsilon=eps, max_weight=wmax, min_ray_length=mn,
                       max_ray_length=mx).to_c()
        a, b = ctypes.create_string_buffer(200), ctypes.create_string_buffer(200)
        ra = O.vxo_config_validate(ctypes.byref(c), a, 200)
        rb = R.vxr_config_validate(ctypes.byref(c), b, 200)
        assert ra == rb and a.value == b.value


@needs_ref
def test_free_functions_vs_reference():
    O, R = oracle_lib(), ref_lib()
    fp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    rng = np.random.default_rng(9)
    for _ in range(3000):
        x, p, s = (rng.uniform(-3, 3, 3).astype(np.float32) for _ in range(3))
        a = np.float32(O.vxo_projective_distance(fp(x), fp(p), fp(s)))
        b = np.float32(R.vxr_projective_distance(fp(x), fp(p), fp(s)))
        assert a.view(np.uint32) == b.view(np.uint32)
        mode, z, d = int(rng.integers(0, 3)), float(rng.uniform(0.05, 9)), float(rng.uniform(-0.5, 0.5))
        assert np.float32(O.vxo_measurement_weight(mode, z, d, 0.4, 0.1)).view(np.uint32) == \
            np.float32(R.vxr_measurement_weight(mode, z, d, 0.4, 0.1)).view(np.uint32)
        g = rng.integers(-3000, 3000, 3).astype(np.int32)
        assert O.vxo_index_hash(*map(int, g)) == R.vxr_index_hash(*map(int, g))
    for _ in range(300):
        st = rng.uniform(-3, 3, 3).astype(np.float32)
        en = (st + rng.uniform(-2, 2, 3)).astype(np.float32)
        a, b = np.zeros((2048, 3), np.int32), np.zeros((2048, 3), np.int32)
        ka = O.vxo_raycast(fp(st), fp(en), 0.1, a.ctypes.data_as(ctypes.c_void_p), 2048)
        kb = R.vxr_raycast(fp(st), fp(en), 0.1, b.ctypes.data_as(ctypes.c_void_p), 2048)
        assert ka == kb and np.array_equal(a[:ka], b[:kb])
    for _ in range(200):
        va, vb = VxgVoxel(0, 0, 0, 0, 0, 0), VxgVoxel(0, 0, 0, 0, 0, 0)
        for _ in range(30):
            d, w = float(rng.uniform(-1, 1)), float(rng.uniform(0, 50))
            col = rng.integers(0, 256, 3, dtype=np.uint8)
            cp = col.ctypes.data_as(ctypes.c_void_p)
            O.vxo_update_voxel(ctypes.byref(va), d, w, 0.4, 200.0, cp)
            R.vxr_update_voxel(ctypes.byref(vb), d, w, 0.4, 200.0, cp)
        assert bytes(va) == bytes(vb)


def test_reference_kats_on_oracle():
    """test_tsdf_integrator.cpp:12-38 and test_voxel_store.cpp:13-21 KATs."""
    O = oracle_lib()
    fp = lambda *v: np.array(v, np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    assert O.vxo_projective_distance(fp(0, 0, 2), fp(0, 0, 2), fp(0, 0, 0)) == 0.0
    assert abs(O.vxo_projective_distance(fp(0, 0, 1), fp(0, 0, 2), fp(0, 0, 0)) - 1.0) < 1e-5
    assert abs(O.vxo_projective_distance(fp(0, 0, 2.5), fp(0, 0, 2), fp(0, 0, 0)) + 0.5) < 1e-5
    assert O.vxo_measurement_weight(0, 3.0, 0.2, 0.4, 0.1) == 1.0
    assert abs(O.vxo_measurement_weight(1, 2.0, 0.0, 0.4, 0.1) - 0.25) < 1e-6
    assert O.vxo_measurement_weight(2, 1.0, -0.41, 0.4, 0.1) == 0.0
    out = np.zeros(3, np.int32)
    O.vxo_global_index(fp(0.25, -0.05, 0.10), 0.1, out.ctypes.data_as(ctypes.c_void_p))
    assert out.tolist() == [2, -1, 1]  # floor(-0.5) = -1

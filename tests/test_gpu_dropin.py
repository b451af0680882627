"""The reference's OWN doctest suites (proj/tests/test_tsdf_integrator.cpp,
test_voxel_store.cpp) linked against the B200 drop-in
(paper_1611_03631_b200/dropin/vxf_tsdf_integrator_vxg.cpp) instead of the
reference's src/tsdf_integrator.cpp: every vxf::TsdfIntegrator call in them
runs through the C ABI on the GPU. Built in the container where
/root/reference exists (oracle/Makefile -> oracle/_ref/unit_tests_vxg)."""
import os
import subprocess

import pytest

from oracle_bindings import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "unit_tests_vxg")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/unit_tests_vxg not built (needs /root/reference)")
def test_reference_doctests_on_gpu_dropin(gpu):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "test cases: 16 | failed: 0" in r.stdout, r.stdout


MESH_REF = os.path.join(ROOT, "oracle", "_ref", "unit_tests_ref_mesh")
MESH_VXG = os.path.join(ROOT, "oracle", "_ref", "unit_tests_vxg_mesh")


@pytest.mark.skipif(not (os.path.exists(MESH_REF) and os.path.exists(MESH_VXG)),
                    reason="oracle/_ref mesh test binaries not built (needs /root/reference)")
def test_reference_mesh_doctests_on_gpu_dropin(gpu):
    """The reference's test_mesh_extractor.cpp against the GPU MeshExtractor
    drop-in reports exactly what it reports against the reference's own
    mesh_extractor.cpp (5 cases; the plane case's REQUIRE(interpolation at every
    vertex) fails for the reference itself in this build: vertices on the
    field's last voxel layer need voxel 18 of a 0..17 field)."""
    ref = subprocess.run([MESH_REF], capture_output=True, text=True, timeout=600)
    vxg = subprocess.run([MESH_VXG], capture_output=True, text=True, timeout=600)
    assert "test cases: 5" in ref.stdout, ref.stdout[-2000:]
    assert vxg.stdout == ref.stdout, "drop-in:\n" + vxg.stdout[-3000:] + "\nreference:\n" + ref.stdout[-3000:]


INS_REF = os.path.join(ROOT, "oracle", "_ref", "bench_insert_ref")
INS_VXG = os.path.join(ROOT, "oracle", "_ref", "bench_insert_vxg")


@pytest.mark.skipif(not (os.path.exists(INS_REF) and os.path.exists(INS_VXG)),
                    reason="oracle/_ref/bench_insert_* not built (needs /root/reference)")
def test_per_scan_insert_through_dropin(gpu):
    """A caller of the reference's C++ API inserting 30 cfg1 scans one by one
    (oracle/bench_insert.cpp, timed like cli.cpp:168-186), linked against the
    reference's integrator and against the B200 drop-in: same update and block
    counts, and the drop-in's median insert is well below the reference's
    (the full 100-scan numbers are in profiles/r3_dropin_cfg1.json)."""
    from dropin_insert_timing import run
    out = run(1, 30)
    assert out["vxg"]["updates"] == out["ref"]["updates"] and out["vxg"]["blocks"] == out["ref"]["blocks"]
    assert out["vxg"]["median_ms"] < 0.5 * out["ref"]["median_ms"], out

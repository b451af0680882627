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

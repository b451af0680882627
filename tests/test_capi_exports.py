"""CPU: the C-ABI library loads and exports every symbol include/*.h declares
(no compute calls without a GPU), and refuses to run without a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(vxg_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared("vxg.h")
    for n in ["vxg_create", "vxg_destroy", "vxg_integrate", "vxg_integrate_batch", "vxg_integrate_packed",
              "vxg_export_blocks", "vxg_query_voxels", "vxg_save_vxblx", "vxg_load_vxblx", "vxg_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1611_03631_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared("vxg.h") if not hasattr(lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in _capi.SIGNATURES}
    assert set(declared("vxg.h")) <= bound, set(declared("vxg.h")) - bound


def test_library_is_sm100a_only():
    from paper_1611_03631_b200 import _capi
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_no_cpu_fallback_without_device():
    """Without a CUDA device vxg_create fails loudly (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1611_03631_b200 import TsdfLayer
    with pytest.raises(RuntimeError, match="no CUDA device|CUDA"):
        TsdfLayer(0.1, 16)


def test_oracle_library_exports():
    from oracle_bindings import oracle_lib
    L = oracle_lib()
    for n in ["vxo_integrate", "vxo_save_vxblx", "vxo_grouped_ray_order", "vxo_bucket_schedule"]:
        assert hasattr(L, n)

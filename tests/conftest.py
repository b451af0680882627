import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: larger CPU-oracle cases")
    # Build products if this snapshot lacks them (nvcc cross-compiles without a GPU).
    need = [os.path.join(ROOT, "paper_1611_03631_b200", "libvxg.so"),
            os.path.join(ROOT, "paper_1611_03631_b200", "workload", "libworkload.so"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "-j8", "lib", "workload", "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def gpu():
    """Fails (not skips) if a GPU test runs without a usable device: the CUDA path
    must be the one that runs, never a silent fallback."""
    from paper_1611_03631_b200 import _capi
    import ctypes
    buf = ctypes.create_string_buffer(256)
    rc = _capi.lib().vxg_device_info(0, buf, 256)
    assert rc == 0, f"no usable CUDA device: {_capi.lib().vxg_last_error().decode()}"
    return buf.value.decode()

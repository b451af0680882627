"""Scan I/O (host side, CPU): vxg_tum_load, the ascii PLY path of
vxg_ply_load, vxg_save_ply_mesh and the PLY header errors against the
reference's own scan.cpp compiled in oracle/_ref — bitwise values, identical
bytes, identical exception texts."""
import numpy as np
import pytest

from io_helpers import write_ply, write_tum
from oracle_bindings import ref_available, ref_load_ply, ref_load_tum, ref_save_ply_mesh
from paper_1611_03631_b200 import Mesh, load_ply_points, load_tum_trajectory, save_ply_mesh

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _err(fn, *a):
    try:
        fn(*a)
    except RuntimeError as e:
        return str(e)
    return None


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("crlf", [False, True])
def test_tum_trajectory(tmp_path, seed, crlf):
    p = str(tmp_path / "traj.txt")
    write_tum(p, 200, seed, crlf=crlf)
    ts, ps = ref_load_tum(p)
    got = load_tum_trajectory(p)
    assert len(got) == len(ts) == 200
    assert np.array_equal(np.array([g.timestamp for g in got]), ts)
    assert np.array_equal(np.stack([g.pose for g in got]).view(np.uint32), ps.view(np.uint32))


def test_tum_errors(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("# c\n1.0 0 0 0 0 0 0 1\n2.0 1 2 3 0.1 0.2\n")
    nonunit = tmp_path / "nonunit.txt"
    nonunit.write_text("1.0 0 0 0 0 0 0 1\n2.0 0 0 0 0.5 0.5 0.5 0.2\n")
    for p in (str(bad), str(nonunit), str(tmp_path / "missing.txt")):
        e = _err(load_tum_trajectory, p)
        assert e is not None and e == _err(ref_load_tum, p)


@pytest.mark.parametrize("props,colors", [
    ([("float", "x"), ("float", "y"), ("float", "z")], False),
    ([("double", "x"), ("float", "nx"), ("double", "y"), ("int", "z"), ("uchar", "red"), ("uchar", "green"),
      ("uchar", "blue"), ("uchar", "alpha")], True),
    ([("short", "z"), ("ushort", "y"), ("int8", "x"), ("float", "red"), ("uint", "green"), ("int16", "blue")], True),
])
@pytest.mark.parametrize("crlf", [False, True])
def test_ascii_ply(tmp_path, props, colors, crlf):
    p = str(tmp_path / "a.ply")
    write_ply(p, props, 500, 7, binary=False, crlf=crlf, extra_elements=True)
    xyz, rgb = ref_load_ply(p)
    s = load_ply_points(p)
    assert np.array_equal(s.points.view(np.uint32), xyz.view(np.uint32))
    assert (s.colors is not None) == colors == (rgb is not None)
    if colors:
        assert np.array_equal(s.colors, rgb)


def test_ply_header_errors(tmp_path):
    cases = {
        "notply.ply": b"plx\nformat ascii 1.0\n",
        "fmt.ply": b"ply\nformat binary_big_endian 1.0\nelement vertex 1\nproperty float x\nend_header\n",
        "list.ply": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar int x\nend_header\n",
        "noxyz.ply": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nproperty float y\nend_header\n0 0\n",
        "trunc.ply": b"ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\nproperty float z\n"
                     b"end_header\n1 2 3\n4 5 6\n",
        "malformed.ply": b"ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\n"
                         b"property float z\nend_header\n1 2 3\n4 five 6\n",
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        e = _err(load_ply_points, str(p))
        assert e is not None and e == _err(ref_load_ply, str(p)), name
    missing = str(tmp_path / "missing.ply")
    assert _err(load_ply_points, missing) == _err(ref_load_ply, missing)


@pytest.mark.parametrize("colors", [True, False])
def test_save_ply_mesh_bytes(tmp_path, colors):
    rng = np.random.default_rng(5)
    T = 300
    v = rng.normal(size=(3 * T, 3)).astype(np.float32)
    n = rng.normal(size=(3 * T, 3)).astype(np.float32)
    c = rng.integers(0, 256, (3 * T, 3)).astype(np.uint8) if colors else np.zeros((0, 3), np.uint8)
    tri = np.arange(3 * T, dtype=np.uint32).reshape(T, 3)
    a, b = str(tmp_path / "a.ply"), str(tmp_path / "b.ply")
    save_ply_mesh(Mesh(v, n, c, tri), a)
    ref_save_ply_mesh(b, v, n, c if colors else None, tri)
    assert open(a, "rb").read() == open(b, "rb").read()

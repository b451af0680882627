"""Binary PLY ingestion decoded on the device (vxg_ply_load) vs the
reference's load_ply_points (oracle/_ref): every supported property type and
order, extra properties, host and device outputs, error texts; then a PLY
scan decoded straight into device memory and integrated."""
import numpy as np
import pytest

from io_helpers import write_ply
from oracle_bindings import OracleLayer, ref_available, ref_load_ply
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer, load_ply_points
from paper_1611_03631_b200 import workload as W

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]

PROPS = [
    ([("float", "x"), ("float", "y"), ("float", "z")], False),
    ([("float", "x"), ("float", "y"), ("float", "z"), ("uchar", "red"), ("uchar", "green"), ("uchar", "blue")], True),
    ([("double", "x"), ("float", "nx"), ("double", "y"), ("int", "z"), ("uchar", "red"), ("uint8", "green"),
      ("uchar", "blue"), ("uchar", "alpha"), ("int64", "stamp")], True),
    ([("short", "z"), ("ushort", "y"), ("int8", "x"), ("float", "red"), ("uint", "green"), ("int16", "blue"),
      ("float64", "extra")], True),
    ([("int32", "x"), ("uint32", "y"), ("float32", "z"), ("char", "red"), ("ushort", "green"), ("double", "blue")],
     True),
]


@pytest.mark.parametrize("k", range(len(PROPS)))
def test_binary_ply_host_and_device(gpu, tmp_path, k):
    import torch
    props, colors = PROPS[k]
    p = str(tmp_path / "b.ply")
    write_ply(p, props, 100003, 11 + k, binary=True, extra_elements=(k % 2 == 1))
    xyz, rgb = ref_load_ply(p)
    s = load_ply_points(p)
    assert np.array_equal(s.points.view(np.uint32), xyz.view(np.uint32))
    assert (rgb is not None) == colors
    if colors:
        assert np.array_equal(s.colors, rgb)
    dx, dc = load_ply_points(p, device=0)
    assert np.array_equal(dx.cpu().numpy().view(np.uint32), xyz.view(np.uint32))
    if colors:
        assert np.array_equal(dc.cpu().numpy(), rgb)
    torch.cuda.synchronize()


def test_binary_ply_errors(gpu, tmp_path):
    p = tmp_path / "t.ply"
    write_ply(str(p), [("float", "x"), ("float", "y"), ("float", "z")], 10, 3, binary=True)
    data = p.read_bytes()
    p.write_bytes(data[:-5])
    bad = tmp_path / "i64.ply"
    write_ply(str(bad), [("int64", "x"), ("float", "y"), ("float", "z")], 4, 3, binary=True)
    badtype = tmp_path / "bt.ply"
    badtype.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\nproperty float x\n"
                        b"property float y\nproperty quad z\nend_header\n" + b"\0" * 16)
    for f in (p, bad, badtype):
        with pytest.raises(RuntimeError) as e:
            load_ply_points(str(f))
        with pytest.raises(RuntimeError) as r:
            ref_load_ply(str(f))
        assert str(e.value) == str(r.value)


def test_ply_scan_integrated_from_device(gpu, tmp_path):
    """A cfg1 frame written as binary PLY, decoded on the device and integrated
    from device memory: the layer equals the oracle's on the same frame."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    x, c, pose = W.frame(1, 4)
    p = str(tmp_path / "f.ply")
    a = np.zeros(len(x), [("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("red", "u1"), ("green", "u1"), ("blue", "u1")])
    a["x"], a["y"], a["z"] = x[:, 0], x[:, 1], x[:, 2]
    a["red"], a["green"], a["blue"] = c[:, 0], c[:, 1], c[:, 2]
    with open(p, "wb") as f:
        f.write(b"ply\nformat binary_little_endian 1.0\nelement vertex %d\n" % len(x))
        f.write(b"property float x\nproperty float y\nproperty float z\n")
        f.write(b"property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n")
        f.write(a.tobytes())
    dx, dc = load_ply_points(p, device=0)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    st = integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), np.array([0, len(x)], np.uint64),
                                np.asarray(pose, np.float32).reshape(1, 12), True)
    o = OracleLayer(cfg, wc.voxel_size, wc.vps)
    assert tuple(int(v) for v in st[0]) == o.integrate(x, c, pose)
    assert layer.save_bytes() == o.save_bytes()

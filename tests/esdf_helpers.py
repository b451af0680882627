"""ESDF VXBLX decoding and checks shared by the ESDF pin (CPU) and GPU tests."""
import numpy as np

from paper_1611_03631_b200.tsdf import ESDF_VOXEL_DTYPE

OBSERVED, FIXED = 1, 2  # voxel.h:24-25


def decode(data: bytes):
    """(header bytes, block index [B,3] i64, voxels [B, vps^3] ESDF_VOXEL_DTYPE)."""
    assert data[:6] == b"VXBLX\0" and data[22] == 1, "not an ESDF layer file"
    vps = int(np.frombuffer(data[18:22], dtype="<u4")[0])
    count = int(np.frombuffer(data[23:31], dtype="<u8")[0])
    rec = np.dtype([("idx", "<i8", (3,)), ("vox", ESDF_VOXEL_DTYPE, (vps ** 3,))])
    arr = np.frombuffer(data, dtype=rec, count=count, offset=31)
    assert 31 + count * rec.itemsize == len(data)
    return data[:31], arr["idx"], arr["vox"], vps


def same_distances_and_flags(a: bytes, b: bytes) -> None:
    """Bit-exact header, block set, distances and flags (parents excluded)."""
    ha, ia, va, _ = decode(a)
    hb, ib, vb, _ = decode(b)
    assert ha == hb
    assert np.array_equal(ia, ib)
    assert np.array_equal(va["distance"].view(np.uint32), vb["distance"].view(np.uint32))
    assert np.array_equal(va["flags"], vb["flags"])


def check_parents(data: bytes, voxel_size: float, d_max: float) -> int:
    """Every lowered voxel's parent is an observed 26-neighbour whose
    RN(distance + step) equals the voxel's distance (relax_neighbors
    esdf_integrator.cpp:258-292); fixed, unobserved and never-lowered voxels
    have none. Returns the number of lowered voxels."""
    _h, idx, vox, vps = decode(data)
    steps = np.float32(voxel_size) * np.sqrt(np.arange(4, dtype=np.float32)).astype(np.float32)
    lut = {tuple(int(x) for x in b): k for k, b in enumerate(idx)}
    lin = np.arange(vps ** 3)
    lx, ly, lz = lin % vps, (lin // vps) % vps, lin // (vps * vps)
    lowered = 0
    for k, b in enumerate(idx):
        v = vox[k]
        obs = (v["flags"] & OBSERVED) != 0
        fixed = (v["flags"] & FIXED) != 0
        low = obs & ~fixed & (v["distance"] < np.float32(d_max))
        par = v["parent"].astype(np.int64)
        assert not par[~low].any(), "parent on a voxel that was never lowered"
        for i in np.nonzero(low)[0]:
            p = par[i]
            assert np.abs(p).max() == 1, "quasi-Euclidean parents are unit offsets"
            g = np.array([b[0] * vps + lx[i], b[1] * vps + ly[i], b[2] * vps + lz[i]]) + p
            nb = tuple(int(x) for x in np.floor_divide(g, vps))
            assert nb in lut
            nl = g - np.array(nb) * vps
            src = vox[lut[nb]][nl[0] + vps * (nl[1] + vps * nl[2])]
            assert src["flags"] & OBSERVED
            cand = np.float32(src["distance"]) + steps[int((p * p).sum())]
            assert np.float32(cand) == v["distance"][i]
        lowered += int(low.sum())
    return lowered

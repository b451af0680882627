"""Layers for the meshing parity tests: analytic fields written block by block
(the reference tests' oracles::analytic_tsdf, tests/oracles.h:103-119) and
seeded random fields with unobserved voxels, negative block indices and
straddling cubes."""
import numpy as np

from paper_1611_03631_b200.tsdf import VOXEL_DTYPE


def _blocks_from_field(fn, lo, hi, v, vps, trunc, rng=None, p_unobserved=0.0):
    """Blocks covering voxels lo..hi (inclusive); voxels outside the range stay default (unobserved)."""
    lo, hi = np.asarray(lo), np.asarray(hi)
    b_lo, b_hi = np.floor_divide(lo, vps), np.floor_divide(hi, vps)
    idx, vox = [], []
    lin = np.arange(vps ** 3)
    lx, ly, lz = lin % vps, (lin // vps) % vps, lin // (vps * vps)
    for bz in range(b_lo[2], b_hi[2] + 1):
        for by in range(b_lo[1], b_hi[1] + 1):
            for bx in range(b_lo[0], b_hi[0] + 1):
                g = np.stack([bx * vps + lx, by * vps + ly, bz * vps + lz], 1)
                inside = np.all((g >= lo) & (g <= hi), axis=1)
                c = ((g.astype(np.float32) + np.float32(0.5)) * np.float32(v)).astype(np.float32)
                d = np.clip(fn(c), -trunc, trunc).astype(np.float32)
                b = np.zeros(vps ** 3, dtype=VOXEL_DTYPE)
                b["distance"] = np.where(inside, d, 0)
                w = np.where(inside, 1.0, 0.0).astype(np.float32)
                if rng is not None:
                    w = np.where(rng.random(len(w)) < p_unobserved, 0.0, w * rng.uniform(0.5, 3.0, len(w))).astype(
                        np.float32)
                    b["r"] = rng.integers(0, 256, len(w))
                    b["g"] = rng.integers(0, 256, len(w))
                    b["b"] = rng.integers(0, 256, len(w))
                b["weight"] = w
                idx.append((bx, by, bz))
                vox.append(b)
    return np.array(idx, np.int32), np.stack(vox)


def sphere_layer(v=0.05, vps=8, center=(0.52, 0.48, 0.5), radius=0.31, lo=(0, 0, 0), hi=(20, 20, 20)):
    c = np.asarray(center, np.float32)
    fn = lambda p: (np.sqrt(((p - c) ** 2).sum(1)) - np.float32(radius)).astype(np.float32)  # noqa: E731
    return _blocks_from_field(fn, lo, hi, v, vps, 10.0)


def random_layer(seed, v=0.1, vps=8, lo=(-11, -5, -9), hi=(12, 9, 6), p_unobserved=0.05):
    """A wavy seeded field (many crossings) with random weights, colours and holes."""
    rng = np.random.default_rng(seed)
    k = rng.uniform(2.0, 6.0, 3).astype(np.float32)
    ph = rng.uniform(0, 6.28, 3).astype(np.float32)
    fn = lambda p: (0.3 * np.sin(k[0] * p[:, 0] + ph[0]) * np.cos(k[1] * p[:, 1] + ph[1])  # noqa: E731
                    + 0.3 * np.sin(k[2] * p[:, 2] + ph[2]) - 0.05).astype(np.float32)
    return _blocks_from_field(fn, lo, hi, v, vps, 0.3, rng, p_unobserved)

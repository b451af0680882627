"""CPU: the oracle's interpolate_distance / surface_error restatement against
the reference itself (oracle/_ref: interpolation.h + analysis.cpp compiled
unmodified), bit for bit, on layers both built from the same scans."""
import os

import numpy as np
import pytest

from oracle_bindings import REF_SO, OracleLayer, RefLayer
from paper_1611_03631_b200 import workload as W

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def _query_points(frames, n_extra=2000, seed=7):
    """World points of the scans (near the surface), jittered copies, lattice
    points (exact voxel-centre coordinates) and far points (absent)."""
    rng = np.random.default_rng(seed)
    pts = []
    for x, _c, p in frames:
        P = np.asarray(p, dtype=np.float32).reshape(3, 4)
        w = (x.astype(np.float32) @ P[:, :3].T + P[:, 3]).astype(np.float32)
        pts.append(w[:: max(1, len(w) // 3000)])
    q = np.concatenate(pts)
    jit = (q + rng.normal(0, 0.03, q.shape)).astype(np.float32)
    lattice = ((np.round(q[:500] / 0.05) + 0.5) * 0.05).astype(np.float32)
    far = rng.uniform(-50, 50, (n_extra, 3)).astype(np.float32)
    return np.concatenate([q, jit, lattice, far]).astype(np.float32)


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_oracle_interpolation_matches_reference(cfg_id):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=2, scale=0.25, start=3)
    ora, ref = OracleLayer(cfg, wc.voxel_size, wc.vps), RefLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in frames:
        ora.integrate(x, c, p)
        ref.integrate(x, c, p)
    q = _query_points(frames)
    od, of = ora.interpolate_distance(q)
    rd, rf = ref.interpolate_distance(q)
    assert of.sum() > 100 and (~of).sum() > 100
    assert np.array_equal(of, rf)
    assert np.array_equal(od.view(np.uint32), rd.view(np.uint32))
    assert ora.surface_error(q, wc.truncation) == ref.surface_error(q, wc.truncation)

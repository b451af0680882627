"""GPU: batched interpolate_distance (interpolation.h:28-60) and surface_error
(analysis.cpp:41-59) on the device slab vs the oracle, bit for bit."""
import numpy as np
import pytest

from oracle_bindings import OracleLayer
from paper_1611_03631_b200 import Scan, TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from test_interpolation_pin import _query_points

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_id,count,scale", [(1, 3, 0.5), (2, 2, 0.5), (3, 2, 0.25), (1, 20, 1.0)])
def test_interpolation_matches_oracle(gpu, cfg_id, count, scale):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=count, scale=scale, start=2)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    integ.integrate_batch([Scan(x, c, p) for x, c, p in frames])
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in frames:
        ora.integrate(x, c, p)
    assert layer.save_bytes() == ora.save_bytes()
    q = _query_points(frames)
    gd, gf = layer.interpolate_distance(q)
    od, of = ora.interpolate_distance(q)
    assert gf.sum() > 100 and (~gf).sum() > 100
    assert np.array_equal(gf, of)
    assert np.array_equal(gd.view(np.uint32), od.view(np.uint32))
    assert layer.surface_error(q, wc.truncation) == ora.surface_error(q, wc.truncation)


def test_interpolation_empty_and_edges(gpu):
    wc = W.CONFIGS[1]
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    q = np.array([[0, 0, 0], [-1e-7, 0.025, -0.025], [1e6, -1e6, 3]], np.float32)
    d, f = layer.interpolate_distance(q)
    assert not f.any() and (d == 0).all()
    assert layer.surface_error(q, 0.1) == {"rms": 0.0, "mean": 0.0, "max": 0.0, "count": 0, "unknown_fraction": 1.0}
    d, f = layer.interpolate_distance(np.zeros((0, 3), np.float32))
    assert len(d) == 0 and len(f) == 0

"""GPU: the occupancy-seeded ESDF (EsdfIntegrator::build_from_occupancy,
esdf_integrator.cpp:303-330) on the device slab vs the oracle restatement
(pinned to the reference by tests/test_esdf_pin.py): header, block set,
distances and flags bit for bit for every queue mode; parents are valid
minimising neighbours (the reference's own tie choice is queue-order
dependent); config errors carry the reference's texts."""
import numpy as np
import pytest

from esdf_helpers import check_parents, decode, same_distances_and_flags
from oracle_bindings import OracleLayer
from paper_1611_03631_b200 import (DistanceMetric, EsdfConfig, EsdfIntegrator, FixedBandMode, QueueMode, Scan,
                                   TsdfIntegrator, TsdfLayer)
from paper_1611_03631_b200 import workload as W

pytestmark = pytest.mark.gpu


def _build(cfg_id, count, scale, start=2):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=count, scale=scale, start=start)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    TsdfIntegrator(cfg, layer).integrate_batch([Scan(x, c, p) for x, c, p in frames])
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in frames:
        ora.integrate(x, c, p)
    assert layer.save_bytes() == ora.save_bytes()
    return wc, layer, ora


@pytest.mark.parametrize("cfg_id,count,scale,d_max", [(1, 3, 0.5, 2.0), (2, 2, 0.5, 4.0), (3, 1, 0.25, 3.0),
                                                      (1, 20, 1.0, 4.0)])
def test_esdf_occupancy_matches_oracle(gpu, cfg_id, count, scale, d_max):
    wc, layer, ora = _build(cfg_id, count, scale)
    for band in FixedBandMode:
        c = EsdfConfig(d_max=d_max, band_mode=band, truncation=wc.truncation)
        esdf = EsdfIntegrator.build_from_occupancy(layer, c)
        assert esdf.block_count() == layer.block_count()
        g = esdf.save_bytes()
        for q in QueueMode:
            c.queue_mode = q
            same_distances_and_flags(g, ora.esdf_occupancy_bytes(c))
        assert check_parents(g, wc.voxel_size, d_max) > 1000
        _h, _i, vox, _ = decode(g)
        assert (vox["distance"] == np.float32(0)).any() and (vox["distance"] < np.float32(d_max)).sum() > 1000


def test_esdf_after_more_frames_and_empty_layer(gpu):
    """Rebuild after further integration (new blocks) and on an empty layer."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    c = EsdfConfig(d_max=1.5, truncation=wc.truncation)
    empty = EsdfIntegrator.build_from_occupancy(layer, c)
    assert empty.block_count() == 0 and len(empty.save_bytes()) == 31
    integ = TsdfIntegrator(cfg, layer)
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    for k, (x, col, p) in enumerate(W.frames(1, count=4, scale=0.3, start=0)):
        integ.integrate(Scan(x, col, p))
        ora.integrate(x, col, p)
        if k in (0, 3):
            same_distances_and_flags(EsdfIntegrator.build_from_occupancy(layer, c).save_bytes(),
                                     ora.esdf_occupancy_bytes(c))


def test_esdf_config_errors(gpu):
    wc, layer, ora = _build(1, 1, 0.1)
    for c in [EsdfConfig(d_max=0.04, truncation=wc.truncation),
              EsdfConfig(band_mode=FixedBandMode.kHalfTruncation, truncation=0.0),
              EsdfConfig(band_mode=FixedBandMode.kOneVoxel, truncation=0.01)]:
        with pytest.raises(ValueError) as e_gpu:
            EsdfIntegrator.build_from_occupancy(layer, c)
        with pytest.raises(ValueError) as e_ora:
            ora.esdf_occupancy_bytes(c)
        assert str(e_gpu.value) == str(e_ora.value)
    with pytest.raises(ValueError, match="quasi-Euclidean"):
        EsdfIntegrator.build_from_occupancy(layer, EsdfConfig(metric=DistanceMetric.kEuclidean,
                                                              truncation=wc.truncation))

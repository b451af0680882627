"""CPU: the oracle's ESDF restatement (build_from_occupancy, esdf_integrator.cpp:
303-330) against the reference itself (oracle/_ref: esdf_integrator.cpp compiled
unmodified), byte for byte — distances, flags AND parents, for every queue
mode, both metrics and both band modes — on layers both built from the same
scans; plus the property the GPU path rests on: with the quasi-Euclidean
metric the reference's distances and flags do not depend on the queue mode."""
import os

import pytest

from esdf_helpers import check_parents, same_distances_and_flags
from oracle_bindings import REF_SO, OracleLayer, RefLayer
from paper_1611_03631_b200 import DistanceMetric, EsdfConfig, FixedBandMode, QueueMode
from paper_1611_03631_b200 import workload as W

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def _layers(cfg_id, count=2, scale=0.25):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    ora, ref = OracleLayer(cfg, wc.voxel_size, wc.vps), RefLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in W.frames(cfg_id, count=count, scale=scale, start=2):
        ora.integrate(x, c, p)
        ref.integrate(x, c, p)
    assert ora.save_bytes() == ref.save_bytes()
    return wc, ora, ref


@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_oracle_esdf_occupancy_matches_reference(cfg_id):
    wc, ora, ref = _layers(cfg_id, **({"count": 1, "scale": 0.1} if cfg_id == 3 else {}))
    for metric in DistanceMetric:
        for band in FixedBandMode:
            for q in QueueMode:
                c = EsdfConfig(d_max=1.0 if cfg_id == 3 else 2.0, band_mode=band, truncation=wc.truncation, metric=metric, queue_mode=q)
                assert ora.esdf_occupancy_bytes(c) == ref.esdf_occupancy_bytes(c), (metric, band, q)


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_quasi_occupancy_is_queue_order_independent(cfg_id):
    """The reference's own output, three queue orders: identical distances and
    flags; parents differ only among valid minimising neighbours."""
    wc, _ora, ref = _layers(cfg_id)
    outs = [ref.esdf_occupancy_bytes(EsdfConfig(d_max=2.0, truncation=wc.truncation, queue_mode=q))
            for q in QueueMode]
    for o in outs[1:]:
        same_distances_and_flags(outs[0], o)
    for o in outs:
        assert check_parents(o, wc.voxel_size, 2.0) > 1000


def test_esdf_config_errors_match_reference():
    wc, ora, ref = _layers(1, count=1, scale=0.1)
    bad = [EsdfConfig(d_max=0.04, truncation=wc.truncation),                      # d_max <= band radius
           EsdfConfig(band_mode=FixedBandMode.kHalfTruncation, truncation=0.0),  # band radius 0
           EsdfConfig(band_mode=FixedBandMode.kOneVoxel, truncation=0.01)]       # band radius > truncation
    for c in bad:
        with pytest.raises(ValueError) as e_ref:
            ref.esdf_occupancy_bytes(c)
        with pytest.raises(ValueError) as e_ora:
            ora.esdf_occupancy_bytes(c)
        assert str(e_ref.value) == str(e_ora.value)

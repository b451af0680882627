"""A batch's ordered fold may outlive vxg_integrate_* ("across
calls"): the next batch's bundling overlaps it, vxg_reset is deferred until the
folds in flight are done, and every entry point that reads the map joins them.
These sequences must give exactly the layers of the synchronous reference
(tsdf_integrator.cpp:111-127 returns with the layer updated)."""
import numpy as np
import pytest

from paper_1611_03631_b200 import Scan, TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from oracle_bindings import OracleLayer
from parity_helpers import diff_report

pytestmark = pytest.mark.gpu


def _frames(start, count, scale=0.3):
    return W.frames(1, count=count, scale=scale, start=start)


def _oracle(cfg, wc, batches):
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    stats = [[ora.integrate(x, c, p) for (x, c, p) in b] for b in batches]
    return ora, stats


def _gpu_batch(integ, frames):
    rows = integ.integrate_batch([Scan(x, c, p) for (x, c, p) in frames])
    return [tuple(int(v) for v in r) for r in rows]


def test_batches_back_to_back_then_reset(gpu):
    """Two batches whose folds chain on the device, a deferred reset while the
    second may still be folding, a third batch: the layer is the third batch's."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    a, b, c = _frames(0, 3), _frames(10, 3), _frames(20, 3)
    _, (sa, sb) = _oracle(cfg, wc, [a, b])
    assert _gpu_batch(integ, a) == sa
    assert _gpu_batch(integ, b) == sb
    layer.reset()
    assert layer.block_count() == 0
    ora_c, (sc,) = _oracle(cfg, wc, [c])
    assert _gpu_batch(integ, c) == sc
    gb, ob = layer.save_bytes(), ora_c.save_bytes()
    assert gb == ob, diff_report(gb, ob)


def test_reset_then_read_is_empty(gpu):
    """A read right after a deferred reset applies it (after the fold in flight)."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _gpu_batch(integ, _frames(0, 4))
    layer.reset()
    empty = OracleLayer(cfg, wc.voxel_size, wc.vps)
    assert layer.save_bytes() == empty.save_bytes()
    # and the layer keeps working from empty
    d = _frames(30, 2)
    ora, (sd,) = _oracle(cfg, wc, [d])
    assert _gpu_batch(integ, d) == sd
    gb, ob = layer.save_bytes(), ora.save_bytes()
    assert gb == ob, diff_report(gb, ob)


def test_accumulating_batches_with_interleaved_queries(gpu):
    """Batches accumulate into one layer; a voxel query between them sees the
    previous batch's complete fold, and the final layer equals the oracle's."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    for k, start in enumerate((0, 7, 14, 21)):
        fr = _frames(start, 2)
        so = [ora.integrate(x, c, p) for (x, c, p) in fr]
        assert _gpu_batch(integ, fr) == so
        if k % 2 == 0:
            gb, ob = layer.save_bytes(), ora.save_bytes()
            assert gb == ob, diff_report(gb, ob)
    gb, ob = layer.save_bytes(), ora.save_bytes()
    assert gb == ob, diff_report(gb, ob)


def test_flush_then_stream_sync(gpu):
    """vxg_flush orders the handle's stream after the fold: after flush and a
    sync of that stream only, the stage timer of the apply stage is complete."""
    import torch
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    stream = torch.cuda.current_stream()
    layer.set_stream(stream.cuda_stream)
    integ = TsdfIntegrator(cfg, layer)
    layer.profile(True)
    layer.stage_times(reset=True)
    _gpu_batch(integ, _frames(0, 3))
    layer.flush()
    stream.synchronize()
    st = layer.stage_times(reset=True)
    assert st["apply"][0] > 0.0
    layer.profile(False)


def test_reset_then_empty_batch(gpu):
    """A batch without rays after a deferred reset still leaves an empty layer."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _gpu_batch(integ, _frames(0, 2))
    layer.reset()
    empty_pts = np.zeros((0, 3), np.float32)
    pose = np.eye(4, dtype=np.float32)[:3]
    stats = integ.integrate_batch([Scan(empty_pts, None, pose)])
    assert int(stats[0, 0]) == 0
    assert layer.block_count() == 0
    assert layer.save_bytes() == OracleLayer(cfg, wc.voxel_size, wc.vps).save_bytes()

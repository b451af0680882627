"""GPU: the sharded (multi-GPU) path, exercised on one B200 through the
loopback group (vxg_group_*): the same sharded kernels (record-balanced ray
slices, owner partition, localize at the owner, sort + fold), with
device-to-device copies standing in for the NCCL all-to-all. The union of the
shards must equal the single-GPU layer and the oracle bit-for-bit
(SURVEY.md §8e parity)."""
import pytest

from paper_1611_03631_b200 import MergeMode, Scan, ShardGroup, TsdfIntegrator, TsdfLayer, WeightMode
from paper_1611_03631_b200 import workload as W
from oracle_bindings import OracleLayer
from parity_helpers import diff_report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_sharded_equals_oracle(gpu, world, cfg_id):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=3, scale=0.2)
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    o_stats = [list(ora.integrate(*f)) for f in frames]
    g = ShardGroup(cfg, wc.voxel_size, wc.vps, world=world)
    stats = [[int(v) for v in r] for r in g.integrate_batch([Scan(*f) for f in frames])]
    assert stats == o_stats
    got, exp = g.save_bytes(), ora.save_bytes()
    assert got == exp, diff_report(got, exp)
    counts = g.shard_block_counts()
    assert sum(counts) == ora.block_count()
    if world > 1:
        assert sum(1 for c in counts if c > 0) > 1  # blocks really are spread over owners


@pytest.mark.parametrize("merge", [MergeMode.kSimpleRaycast, MergeMode.kGroupedAntiGraze])
def test_sharded_modes(gpu, merge):
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc, merge_mode=int(merge), weight_mode=int(WeightMode.kInverseZ2Dropoff))
    frames = W.frames(1, count=2, scale=0.15, start=11)
    single = TsdfLayer(wc.voxel_size, wc.vps)
    TsdfIntegrator(cfg, single).integrate_batch([Scan(*f) for f in frames])
    g = ShardGroup(cfg, wc.voxel_size, wc.vps, world=4)
    g.integrate_batch([Scan(*f) for f in frames])
    assert g.save_bytes() == single.save_bytes()


def test_sharded_full_frames(gpu):
    """Full-size cfg1 frames over 4 shards equal the single-GPU layer."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    frames = W.frames(1, count=4, start=40)
    single = TsdfLayer(wc.voxel_size, wc.vps)
    s1 = TsdfIntegrator(cfg, single).integrate_batch([Scan(*f) for f in frames])
    g = ShardGroup(cfg, wc.voxel_size, wc.vps, world=4, block_capacity=64)
    s4 = g.integrate_batch([Scan(*f) for f in frames])
    assert (s1 == s4).all()
    assert g.save_bytes() == single.save_bytes()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg_id", [1, 3])
def test_replicated_traversal_equals_oracle(gpu, world, cfg_id):
    """SURVEY.md 8e fallback: every shard walks all rays and keeps only its own
    blocks' records (no record exchange); same layer, same counters."""
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=3, scale=0.2, start=4)
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    o_stats = [list(ora.integrate(*f)) for f in frames]
    g = ShardGroup(cfg, wc.voxel_size, wc.vps, world=world, replicated=True)
    stats = [[int(v) for v in r] for r in g.integrate_batch([Scan(*f) for f in frames])]
    assert stats == o_stats
    got, exp = g.save_bytes(), ora.save_bytes()
    assert got == exp, diff_report(got, exp)
    assert sum(1 for c in g.shard_block_counts() if c > 0) > 1


@pytest.mark.parametrize("cfg_id", [1, 3])
def test_nccl_one_rank_exchange(gpu, cfg_id):
    """The real NCCL path (ncclSend/ncclRecv of the counts and records in a
    group, ncclAllReduce of the per-frame counters, vxg_tsdf.cu nccl_exchange /
    nccl_reduce_updates) over a 1-rank communicator: one GPU exchanges with
    itself, so the same protocol a multi-GPU run uses executes on hardware.
    The layer equals the single-GPU one and the oracle."""
    from paper_1611_03631_b200 import nccl_unique_id
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    frames = W.frames(cfg_id, count=3, scale=0.3, start=5)
    ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
    o_stats = [list(ora.integrate(*f)) for f in frames]
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    layer.shard_init(0, 1, nccl_unique_id())
    integ = TsdfIntegrator(cfg, layer)
    stats = [[int(v) for v in r] for r in integ.integrate_batch([Scan(*f) for f in frames])]
    assert stats == o_stats
    # a second call through the same communicator, frame by frame
    for f in W.frames(cfg_id, count=2, scale=0.3, start=9):
        o = list(ora.integrate(*f))
        assert [integ.integrate(Scan(*f)), integ.raycasts_last_scan(), integ.skipped_points_last_scan()] == o
    got, exp = layer.save_bytes(), ora.save_bytes()
    assert got == exp, diff_report(got, exp)

"""GPU parity through the C ABI: the B200 pipeline vs the CPU oracle, bit-exact.

The bar (BASELINE.json north_star): allocated block set, voxel keys and the
per-voxel (distance, weight, colour) must match; the order-preserving fold
makes them bit-exact, so every comparison here is on the VXBLX bytes
(serialization.cpp:141-168) plus the integrate() counters.
"""
import numpy as np
import pytest

from paper_1611_03631_b200 import MergeMode, Scan, TsdfConfig, TsdfIntegrator, TsdfLayer, WeightMode
from paper_1611_03631_b200 import workload as W
from oracle_bindings import ref_available
from parity_helpers import diff_report, run_pair

pytestmark = pytest.mark.gpu


def _check(layer, integ, cfg, wc, frames, batch=False):
    g, o, gb, ob = run_pair(layer, integ, cfg, wc.voxel_size, wc.vps, frames, batch=batch)
    assert g == o, f"stats differ: gpu={g} oracle={o}"
    assert gb == ob, diff_report(gb, ob)


@pytest.mark.parametrize("cfg_id", [0, 1, 2, 3])
@pytest.mark.parametrize("batch", [False, True])
def test_configs_reduced_scale(gpu, cfg_id, batch):
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    frames = W.frames(cfg_id, count=3 if cfg_id else 1, scale=0.2, start=0, n_frames=wc.frames)
    _check(layer, integ, cfg, wc, frames, batch)


@pytest.mark.parametrize("merge", [MergeMode.kSimpleRaycast, MergeMode.kGroupedRaycast, MergeMode.kGroupedAntiGraze])
@pytest.mark.parametrize("weight", [WeightMode.kConstant, WeightMode.kInverseZ2, WeightMode.kInverseZ2Dropoff])
def test_all_modes(gpu, merge, weight):
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc, merge_mode=int(merge), weight_mode=int(weight))
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    frames = W.frames(1, count=2, scale=0.15, start=5)
    _check(layer, integ, cfg, wc, frames, batch=True)


def test_cfg1_full_scale_frames(gpu):
    """Three full-size 640x480 merged frames (~2M updates each), bit-exact."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(1, count=3, start=0), batch=True)


def test_cfg0_full_scale(gpu):
    """The full cfg0 frame (simple, constant weight, ~2.9e7 updates), bit-exact."""
    wc = W.CONFIGS[0]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(0, count=1), batch=False)


def test_batch_equals_sequential(gpu):
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    frames = W.frames(1, count=6, scale=0.3, start=20)
    a = TsdfLayer(wc.voxel_size)
    ia = TsdfIntegrator(cfg, a)
    sa = [ia.integrate(Scan(*f)) for f in frames]
    b = TsdfLayer(wc.voxel_size)
    ib = TsdfIntegrator(cfg, b)
    sb = ib.integrate_batch([Scan(*f) for f in frames])
    assert [int(x) for x in sb[:, 0]] == sa
    assert a.save_bytes() == b.save_bytes()


def test_slab_growth_replay(gpu):
    """Start with a 1-block slab: allocation overflows, the slab grows and the
    batch is replayed; the result must still match the oracle exactly."""
    wc = W.CONFIGS[2]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(2, count=2, scale=0.2), batch=True)


def test_empty_and_out_of_range(gpu):
    v = 0.1
    cfg = TsdfConfig.for_voxel_size(v)
    cfg.merge_mode = MergeMode.kSimpleRaycast
    cfg.weight_mode = WeightMode.kConstant
    cfg.min_ray_length, cfg.max_ray_length = 0.5, 2.0
    layer = TsdfLayer(v, 16)
    integ = TsdfIntegrator(cfg, layer)
    assert integ.integrate(Scan(np.zeros((0, 3), np.float32))) == 0
    assert layer.block_count() == 0
    pts = np.array([[0.2, 0, 0], [5.0, 0, 0]], np.float32)  # too close, too far
    assert integ.integrate(Scan(pts)) == 0
    assert integ.skipped_points_last_scan() == 2
    assert layer.block_count() == 0
    pts = np.array([[0.2, 0, 0], [5.0, 0, 0], [1.0, 0, 0]], np.float32)
    assert integ.integrate(Scan(pts)) > 0
    assert integ.skipped_points_last_scan() == 2  # test_tsdf_integrator.cpp:206-218


def test_colour_mismatch_raises(gpu):
    layer = TsdfLayer(0.1)
    integ = TsdfIntegrator(TsdfConfig.for_voxel_size(0.1), layer)
    with pytest.raises(ValueError, match="scan colors must parallel points"):
        integ.integrate(Scan(np.ones((3, 3), np.float32), np.zeros((2, 3), np.uint8)))


def test_invalid_config_raises():
    with pytest.raises(ValueError, match="0 < dropoff_epsilon < truncation"):
        TsdfIntegrator(TsdfConfig(truncation=0.1, dropoff_epsilon=0.1), None)


def test_mixed_colour_batch(gpu):
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    fr = W.frames(1, count=3, scale=0.15, start=40)
    fr[1] = (fr[1][0], None, fr[1][2])
    layer = TsdfLayer(wc.voxel_size)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, fr, batch=True)


def test_query_and_absence(gpu):
    layer = TsdfLayer(0.1)
    integ = TsdfIntegrator(TsdfConfig.for_voxel_size(0.1), layer)
    assert layer.voxel_ptr((1, 2, 3)) is None
    integ.integrate(Scan(np.array([[1.0, 0.05, 0.05]], np.float32)))
    v = layer.voxel_ptr((10, 0, 0))
    assert v is not None and v["weight"] > 0
    assert layer.voxel_ptr((1000, 1000, 1000)) is None


def test_vxblx_round_trip_and_resume(gpu, tmp_path):
    """save -> load -> continue integrating equals integrating without the round trip."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    fr = W.frames(1, count=4, scale=0.15, start=60)
    a = TsdfLayer(wc.voxel_size)
    ia = TsdfIntegrator(cfg, a)
    ia.integrate_batch([Scan(*f) for f in fr[:2]])
    path = str(tmp_path / "layer.vxblx")
    a.save_file(path)
    b = TsdfLayer(wc.voxel_size)
    b.load_bytes(open(path, "rb").read())
    assert b.save_bytes() == a.save_bytes()
    ib = TsdfIntegrator(cfg, b)
    ia.integrate_batch([Scan(*f) for f in fr[2:]])
    ib.integrate_batch([Scan(*f) for f in fr[2:]])
    assert a.save_bytes() == b.save_bytes()


def _dup_image(data: bytes, extra_from: int, modify) -> bytes:
    """A VXBLX image whose block list repeats block `extra_from` (a modified
    copy appended at the end): the reference's load keeps the LAST copy whole."""
    import struct
    nb = struct.unpack_from("<Q", data, 23)[0]
    vps = struct.unpack_from("<I", data, 18)[0]
    bs = 24 + 12 * vps ** 3
    blk = bytearray(data[31 + extra_from * bs: 31 + (extra_from + 1) * bs])
    modify(blk)
    return data[:23] + struct.pack("<Q", nb + 1) + data[31:] + bytes(blk)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_vxblx_load_duplicate_blocks(gpu):
    """Duplicate block indices in a VXBLX file: the device load equals the
    reference's load_tsdf_layer (last copy wins whole)."""
    from oracle_bindings import ref_load_resave
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    a = TsdfLayer(wc.voxel_size)
    TsdfIntegrator(cfg, a).integrate_batch([Scan(*f) for f in W.frames(1, count=2, scale=0.15)])
    good = a.save_bytes()

    def scramble(blk):
        for i in range(24, len(blk), 12 * 37):
            blk[i:i + 8] = bytes([7, 0, 128, 63, 0, 0, 32, 65])  # d = 1.0000008, w = 10
    img = _dup_image(good, 1, scramble)
    want = ref_load_resave(img)
    b = TsdfLayer(wc.voxel_size)
    for _ in range(2):  # twice: nondeterministic slot races would show
        b.load_bytes(img)
        assert b.save_bytes() == want
    assert want != good


def test_parse_errors(gpu):
    from paper_1611_03631_b200 import ParseError
    layer = TsdfLayer(0.1)
    good = layer.save_bytes()
    with pytest.raises(ParseError, match="bad magic"):
        layer.load_bytes(b"Z" + good[1:])
    with pytest.raises(ParseError, match="truncated"):
        layer.load_bytes(good[:10])


def test_consumers(gpu):
    layer = TsdfLayer(0.1, 8)
    layer.register_consumer("esdf")
    layer.register_consumer("mesh")
    integ = TsdfIntegrator(TsdfConfig.for_voxel_size(0.1), layer)
    integ.integrate(Scan(np.array([[1.0, 0.3, 0.1]], np.float32)))
    s1 = layer.drain_updated("esdf")
    assert len(s1) == layer.block_count() > 0
    assert layer.drain_updated("esdf") == set()
    assert layer.drain_updated("mesh") == s1
    with pytest.raises(ValueError, match="unknown updated-block consumer"):
        layer.drain_updated("nobody")


@pytest.mark.parametrize("max_weight", [5.0, 60.0])
def test_weight_saturation(gpu, max_weight):
    """Low max_weight saturates most voxels: exercises the fold's saturated,
    colour-stationary fast lane and its exact fallback, bit-exact vs the oracle."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    cfg.max_weight = max_weight
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(1, count=4, scale=0.5, start=30), batch=True)


def test_long_chains_full_trajectory_slice(gpu):
    """20 full-size frames in one batch: fold chains of several 10^4 records
    (warp-cooperative path), bit-exact vs the oracle."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(1, count=20, start=0), batch=True)
    assert layer.batch_info()["max_chain"] > 4096


def test_cfg1_bench_workload_bit_exact(gpu):
    """The exact bench.py step: all 100 full-size cfg1 frames in one batch
    (2.4e8 updates, fold chains up to 77k records, the custom radix sort at
    3 passes), bit-exact vs the oracle's 100 sequential integrate() calls."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1024)
    integ = TsdfIntegrator(cfg, layer)
    layer.batch_info(reset=True)
    _check(layer, integ, cfg, wc, W.frames(1), batch=True)
    info = layer.batch_info()
    assert info["max_chain"] > 50000 and info["sort_passes"] == 3


@pytest.mark.parametrize("cfg_id,count,scale", [(2, 3, 1.0), (3, 3, 1.0), (4, 1, 0.5)])
def test_configs_full_size_frames(gpu, cfg_id, count, scale):
    """Full-size frames of the other configs (cfg2 752x480 stereo-like, cfg3
    64-beam LiDAR with 80 m rays, cfg4 at 1024x1024), bit-exact."""
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, W.frames(cfg_id, count=count, scale=scale, start=1), batch=True)


def test_rehash_epochs_on_device(gpu):
    """Scans whose bucketing map rehashes while it is filled (every point in a
    voxel of its own: > N/4 distinct terminal voxels, three rehashes at N =
    20k) between ordinary frames, in one batch: the device epoch emulation of
    the libstdc++ iteration order (k_rh_*) gives the reference's ray order,
    bit-exact vs the oracle."""
    rng = np.random.default_rng(7)
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    frames = [W.frame(1, 3, scale=0.2)]
    for n in (20000, 5000):
        pts = rng.uniform(-2.0, 2.0, size=(n, 3)).astype(np.float32)
        pts[:, 2] = np.abs(pts[:, 2]) + 0.5
        col = rng.integers(0, 256, size=(n, 3), dtype=np.uint8)
        frames.append((pts, col, W.pose(1, 40)))
    frames.append(W.frame(1, 7, scale=0.2))
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    _check(layer, integ, cfg, wc, frames, batch=True)


def test_cfg4_full_frames(gpu):
    """Two full 2048x2048 cfg4 frames (v = 2 cm, 4.2e6 points and ~1e9 updates
    each) in one batch against the REFERENCE's own layer for them
    (tests/golden/full_digests.json: sha256 of oracle/_ref's VXBLX bytes,
    made by tests/golden/make_full_digests.py; too large to commit as bytes)."""
    import hashlib
    import json
    import os
    from golden_full import input_digest
    d = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_digests.json")))["cfg4_full_f1_f2"]
    wc = W.CONFIGS[d["config"]]
    cfg = W.tsdf_config(wc)
    frames = W.frames(d["config"], count=d["count"], start=d["start"])
    assert input_digest(frames) == d["input_sha256"], "workload generator drift"
    layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=8192)
    integ = TsdfIntegrator(cfg, layer)
    stats = integ.integrate_batch([Scan(*f) for f in frames])
    assert [[int(v) for v in row] for row in stats] == d["stats"]
    assert layer.block_count() == d["blocks"]
    b = layer.save_bytes()
    assert len(b) == d["vxblx_bytes"] and hashlib.sha256(b).hexdigest() == d["vxblx_sha256"]


@pytest.mark.parametrize("case", ["cfg1_bench_x100", "cfg2_x40", "cfg3_x40"])
def test_full_batches_against_reference_digests(gpu, case):
    """Full-size batches against the REFERENCE ITSELF (not the restatement):
    the 100-frame cfg1 batch bench.py times, and 40-frame prefixes of cfg2 and
    cfg3, each integrated in one call; the layer's VXBLX bytes and the per-frame
    counters must equal oracle/_ref's (tests/golden/full_digests.json)."""
    import hashlib
    import json
    import os
    from golden_full import input_digest
    d = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_digests.json")))[case]
    wc = W.CONFIGS[d["config"]]
    cfg = W.tsdf_config(wc)
    frames = W.frames(d["config"], count=d["count"], start=d["start"])
    assert input_digest(frames) == d["input_sha256"], "workload generator drift"
    layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1024)
    integ = TsdfIntegrator(cfg, layer)
    stats = integ.integrate_batch([Scan(*f) for f in frames])
    assert [[int(v) for v in row] for row in stats] == d["stats"]
    assert layer.block_count() == d["blocks"]
    b = layer.save_bytes()
    assert len(b) == d["vxblx_bytes"] and hashlib.sha256(b).hexdigest() == d["vxblx_sha256"]


def test_batch_split_invariance_full_size(gpu):
    """Property at full size (no oracle): the same 40 frames integrated as one
    batch, as 4 batches of 10 and as 40 single calls give identical bytes."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    fr = [Scan(x, c, p) for (x, c, p) in W.frames(1, count=40, start=10)]
    out = []
    for parts in (1, 4, 40):
        layer = TsdfLayer(wc.voxel_size, wc.vps)
        integ = TsdfIntegrator(cfg, layer)
        n = len(fr) // parts
        for i in range(parts):
            integ.integrate_batch(fr[i * n:(i + 1) * n])
        out.append(layer.save_bytes())
    assert out[0] == out[1] == out[2]


def test_streaming_staged_equals_packed(gpu):
    """Streaming ingestion: batches staged ahead (double-buffered H2D on the copy
    stream, batch k+1 staged before batch k is integrated) give the same layer
    bytes and stats as synchronous integrate_packed calls; staging a third
    batch while two are pending is rejected."""
    import torch
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    batches = [W.pack(W.frames(1, count=4, scale=0.5, start=4 * k)) for k in range(4)]
    ref = TsdfLayer(wc.voxel_size, wc.vps)
    iref = TsdfIntegrator(cfg, ref)
    sref = [iref.integrate_packed(x.ctypes.data, c.ctypes.data, o, p, False) for (x, c, o, p) in batches]
    pinned = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(c).pin_memory(), o, p) for (x, c, o, p) in batches]
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    slot = integ.stage_packed(pinned[0][0].data_ptr(), pinned[0][1].data_ptr(), pinned[0][2])
    got = []
    for k in range(len(pinned)):
        nxt = None
        if k + 1 < len(pinned):
            nxt = integ.stage_packed(pinned[k + 1][0].data_ptr(), pinned[k + 1][1].data_ptr(), pinned[k + 1][2])
            with pytest.raises(Exception):  # two batches pending: no third slot
                integ.stage_packed(pinned[k][0].data_ptr(), pinned[k][1].data_ptr(), pinned[k][2])
        got.append(integ.integrate_staged(slot, pinned[k][3]))
        slot = nxt
    for a, b in zip(got, sref):
        assert np.array_equal(a, b)
    assert layer.save_bytes() == ref.save_bytes()

"""CPU, world_size 2 (gloo): the host-side logic of the sharded map (SURVEY.md
§8e), the protocol the GPU path runs (vxg_tsdf.cu shard_front/shard_back):

  1. every rank derives the same update records in ray order (here: the
     oracle's update trace, standing in for the redundant bundling + walk);
  2. rank r takes the ray-aligned slice holding records
     [r*T/W, (r+1)*T/W) (first ray whose record offset reaches each bound);
  3. records are stably partitioned by block owner = mix64(packed block) % W;
  4. all-to-all (gloo here, NCCL ncclSend/ncclRecv on the GPUs);
  5. each owner concatenates what it received in SOURCE-RANK order, stably
     sorts by voxel and folds each voxel's records in that order.

The union of the shards must equal the single-process oracle layer bit for
bit, which holds only if steps 2-5 preserve each voxel's ray order."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

M64 = (1 << 64) - 1


def mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def pack_block(b):  # vxg_device.cuh pack_block (21 bits per axis, biased by 2^20)
    x, y, z = (int(v) + (1 << 20) for v in b)
    return (x << 42) | (y << 21) | z


def owner_of(b, world):
    return mix64(pack_block(b)) % world


def floor_div(a, b):
    return a // b  # Python floor division == core.h floor_div for b > 0


def trace_scan(cfg_id, vps):
    """(records [N,7] uint32, oracle layer bytes, voxel size) for a small seeded scan."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    from oracle_bindings import OracleLayer, oracle_lib
    from paper_1611_03631_b200 import workload as W
    wc = W.CONFIGS[cfg_id]
    cfg = W.tsdf_config(wc)
    x, c, p = W.frame(cfg_id, 3, 0.12)
    L = oracle_lib()
    L.vxo_trace_updates.restype = ctypes.c_size_t
    L.vxo_trace_updates.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.POINTER(ctypes.c_float), ctypes.c_void_p, ctypes.c_size_t]
    lay = OracleLayer(cfg, wc.voxel_size, vps)
    c_cfg = cfg.to_c()
    pose = np.ascontiguousarray(p, np.float32)
    cap = 5_000_000
    out = np.zeros((cap, 7), np.uint32)
    n = L.vxo_trace_updates(lay.h, ctypes.byref(c_cfg), x.ctypes.data, None if c is None else c.ctypes.data, len(x),
                            pose.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.ctypes.data, cap)
    return out[:n].copy(), lay, cfg, wc.voxel_size


def fold_records(recs, cfg, vps):
    """Fold each voxel's records in the given (stable) order with the oracle's update_tsdf_voxel."""
    from oracle_bindings import oracle_lib
    from paper_1611_03631_b200._capi import VxgVoxel
    L = oracle_lib()
    g = recs[:, 1:4].view(np.int32)
    keys = [tuple(r) for r in g.tolist()]
    order = sorted(range(len(recs)), key=lambda i: keys[i])  # Python sort is stable
    state = {}
    for i in order:
        v = state.setdefault(keys[i], VxgVoxel(0, 0, 0, 0, 0, 0))
        d = float(recs[i, 4:5].view(np.float32)[0])
        w = float(recs[i, 5:6].view(np.float32)[0])
        col = int(recs[i, 6])
        rgb = np.array([col & 255, (col >> 8) & 255, (col >> 16) & 255], np.uint8)
        L.vxo_update_voxel(ctypes.byref(v), d, w, cfg.truncation, cfg.max_weight,
                           rgb.ctypes.data_as(ctypes.c_void_p) if col >> 31 else None)
    return {k: bytes(v) for k, v in state.items()}


def _worker(rank, world, port, cfg_id, vps, result_path, replicated=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs, lay, cfg, v = trace_scan(cfg_id, vps)  # step 1: identical on every rank
        T = len(recs)
        ray = recs[:, 0].astype(np.int64)
        if replicated:
            # replicated traversal (SURVEY.md 8e fallback): every rank walks all
            # rays and keeps the records of the blocks it owns; no exchange
            g = recs[:, 1:4].view(np.int32)
            owners = np.array([owner_of([floor_div(int(a), vps) for a in row], world) for row in g], np.int64)
            got = np.ascontiguousarray(recs[owners == rank])
        else:
            # step 2: ray-aligned slice of the record range
            lo, hi = T * rank // world, T * (rank + 1) // world
            starts = np.searchsorted(ray, np.unique(ray))  # record offset of each ray (records grouped by ray)
            roff = np.append(starts, T)
            first = lambda target: int(roff[np.searchsorted(roff, target)])  # first ray offset >= target
            s0, s1 = first(lo), first(hi)
            mine = recs[s0:s1]
            # step 3: stable partition by block owner
            g = mine[:, 1:4].view(np.int32)
            owners = np.array([owner_of([floor_div(int(a), vps) for a in row], world) for row in g], np.int64)
            send = [np.ascontiguousarray(mine[owners == o]) for o in range(world)]
            # step 4: all-to-all (counts, then records)
            sc = torch.tensor([len(s) for s in send], dtype=torch.int64)
            rc = torch.zeros(world, dtype=torch.int64)
            dist.all_to_all_single(rc, sc)
            send_t = torch.from_numpy(np.concatenate(send).view(np.int32).reshape(-1, 7)) if T else torch.zeros((0, 7), dtype=torch.int32)
            recv_t = torch.zeros((int(rc.sum()), 7), dtype=torch.int32)
            dist.all_to_all_single(recv_t, send_t, output_split_sizes=rc.tolist(), input_split_sizes=sc.tolist())
            got = recv_t.numpy().view(np.uint32)  # step 5: source-rank order preserved by all_to_all_single
        shard = fold_records(got, cfg, vps)
        shards = [None] * world
        dist.all_gather_object(shards, shard)
        if rank == 0:
            union = {}
            for sh in shards:
                assert not (set(sh) & set(union)), "a voxel was folded on two shards"
                union.update(sh)
            full = fold_records(recs, cfg, vps)  # single-process fold of the same trace
            ok_fold = union == full
            # and the single-process fold equals the oracle layer itself
            from oracle_bindings import oracle_lib
            from paper_1611_03631_b200._capi import VxgVoxel
            L = oracle_lib()
            ok_layer = True
            for k, val in full.items():
                vx = VxgVoxel(0, 0, 0, 0, 0, 0)
                L.vxo_voxel(lay.h, k[0], k[1], k[2], ctypes.byref(vx))
                ok_layer &= bytes(vx) == val
            busy = sum(1 for sh in shards if sh)
            with open(result_path, "w") as f:
                f.write(f"{int(ok_fold)} {int(ok_layer)} {busy} {len(full)}")
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("replicated", [False, True])
@pytest.mark.parametrize("cfg_id,vps", [(1, 16), (3, 8)])
def test_sharded_protocol_world2(tmp_path, cfg_id, vps, replicated):
    result = tmp_path / "result.txt"
    mp.spawn(_worker, args=(2, _free_port(), cfg_id, vps, str(result), replicated), nprocs=2, join=True)
    ok_fold, ok_layer, busy, nvox = map(int, result.read_text().split())
    assert nvox > 1000
    assert ok_layer, "single-process fold of the trace differs from the oracle layer"
    assert ok_fold, "sharded fold differs from the single-process fold"
    assert busy == 2, "both shards should own voxels"

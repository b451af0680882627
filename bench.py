#!/usr/bin/env python3
"""Benchmark: TSDF voxel-updates/s and ms/frame on B200 vs the CPU reference.

Workload (BASELINE.json configs[1], the metric's config): the 100-frame seeded
640x480 RGB-D trajectory, merged integrator, 1/z^2 weight + linear drop-off,
voxel 0.05 m, truncation 0.10 m. One STEP = integrate the whole trajectory
into a fresh layer (reset + 100 frames, one batched call; results identical to
100 sequential integrate() calls). Inputs (~460 MB) exceed the 126 MB L2, so no
explicit flush between steps.

  value : updates/s with inputs resident in HBM (device pointers), device time
          from CUDA events on the library's stream, max over ranks.
  e2e   : the same through the C ABI with pinned HOST buffers (H2D of points +
          colours inside the timed region, stats D2H at the end of each call),
          fed as a stream: vxg_stage_packed starts step k+1's copy before
          vxg_integrate_staged integrates step k (double-buffered staging), so
          the copy overlaps compute. e2e.sync_one_call = vxg_integrate_packed
          (copy, then compute, per call).
  --impl reference : the reference's own CPU integrator (oracle/_ref: the
          unmodified reference sources compiled with the Eigen shim), 1 thread.
Multi-GPU (torchrun, one process per GPU): ONE map sharded by block-key
ownership over the ranks: every rank bundles the 100 frames,
walks a record-balanced slice of the ray order and routes update records to
the block owners with an NCCL all-to-all inside the library; the total work is
fixed (strong scaling), value = total updates / max-over-ranks step time.
Ranks > 0 of the reference arm exit without work.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tsdf_voxel_updates_per_sec"
UNIT = "updates/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_workload(cfg_id: int, n_frames: int):
    from paper_1611_03631_b200 import workload as W
    wc = W.CONFIGS[cfg_id]
    fr = [W.frame(cfg_id, i % wc.frames, 1.0, wc.frames) for i in range(n_frames)]
    return wc, W.pack(fr)


def cpu_reference_run(wc, packed, frames: int):
    """The unmodified reference integrator (oracle/_ref) on `frames` frames, 1 thread."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import RefLayer, ref_available
    from paper_1611_03631_b200 import workload as W
    if not ref_available():
        return None
    xyz, rgb, off, poses = packed
    layer = RefLayer(W.tsdf_config(wc), wc.voxel_size, wc.vps)
    upd = 0
    t0 = time.perf_counter()
    for f in range(frames):
        a, b = int(off[f]), int(off[f + 1])
        u, _, _ = layer.integrate(xyz[a:b], None if rgb is None else rgb[a:b], poses[f])
        upd += u
    dt = time.perf_counter() - t0
    return upd, dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    wc, packed = load_workload(args.config, args.ref_frames)
    res = cpu_reference_run(wc, packed, 1)  # warm-up-free probe that the library loads
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libvxfref.so not built"}))
        return
    times, upds = [], []
    for i in range(args.warmup + args.steps):
        u, dt = cpu_reference_run(wc, packed, args.ref_frames)
        if i >= args.warmup:
            times.append(dt)
            upds.append(u)
    value = sum(upds) / sum(times)
    ms_frame = 1e3 * sum(times) / (len(times) * args.ref_frames)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "ms_per_frame": ms_frame, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32+f64", "data": "synthetic (seeded analytic room, workload.c)",
        "config": {"workload": wc.name, "frames_per_step": args.ref_frames, "merge": "grouped",
                   "weight": "inverse_z2_dropoff", "voxel_size": wc.voxel_size},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"first {args.ref_frames} frames of {wc.name} per step (reference is single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vxg", choices=["vxg", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--frames", type=int, default=100)
    ap.add_argument("--ref-frames", type=int, default=10)
    ap.add_argument("--cpu-frames", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicated", action="store_true",
                    help="N>1: replicated traversal (every rank walks all rays, no record exchange)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)

    from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
    from paper_1611_03631_b200 import workload as W

    wc, packed = load_workload(args.config, args.frames)
    xyz, rgb, off, poses = packed
    F = len(poses)
    P = int(off[-1])
    cfg = W.tsdf_config(wc)

    stream = torch.cuda.current_stream()
    layer = TsdfLayer(wc.voxel_size, wc.vps, device=local, block_capacity=1024)
    layer.set_stream(stream.cuda_stream)
    if world > 1:
        from paper_1611_03631_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        layer.shard_init(rank, world, obj[0], replicated=args.replicated)
    integ = TsdfIntegrator(cfg, layer)

    d_xyz = torch.from_numpy(xyz).cuda()
    d_rgb = torch.from_numpy(rgb).cuda() if rgb is not None else None
    h_xyz = torch.from_numpy(xyz).pin_memory()
    h_rgb = torch.from_numpy(rgb).pin_memory() if rgb is not None else None

    def step(device_input: bool):
        layer.reset()
        if device_input:
            return integ.integrate_packed(d_xyz.data_ptr(), d_rgb.data_ptr() if d_rgb is not None else None, off,
                                          poses, True)
        return integ.integrate_packed(h_xyz.data_ptr(), h_rgb.data_ptr() if h_rgb is not None else None, off, poses,
                                      False)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (allocates scratch, grows the slab, caches the bucket schedule)
    for _ in range(args.warmup):
        stats = step(True)
    updates_per_step = int(stats[:, 0].sum())

    # ---- timed: device-resident inputs
    layer.profile(True)
    layer.batch_info(reset=True)
    layer.stage_times(reset=True)
    layer.kernel_launches(reset=True)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        t0.record(stream)
        for _ in range(args.steps):
            stats = step(True)
        layer.flush()  # the last batch's fold (it may outlive the call) inside the timed region
        t1.record(stream)
        barrier()
    dev_ms = t0.elapsed_time(t1)
    stages = layer.stage_times(reset=True)
    launches = layer.kernel_launches(reset=True)
    info = layer.batch_info(reset=True)
    layer.profile(False)
    ms = torch.tensor([dev_ms], device="cuda")
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dev_ms = float(ms.item())
    ms_step = dev_ms / args.steps
    total_updates = updates_per_step  # one sharded map: stats are global on every rank
    value = total_updates / (ms_step / 1e3)

    # ---- e2e: pinned host inputs through the C ABI. Headline: the streaming
    # API (vxg_stage_packed / vxg_integrate_staged) as a continuous feed would
    # use it — step k+1's H2D is staged before step k is integrated, so the copy
    # overlaps step k's compute; every step's H2D and its stats D2H are inside
    # the timed region. Also timed: the synchronous one-call path
    # (vxg_integrate_packed from host memory, H2D then compute).
    hx = h_xyz.data_ptr()
    hc = h_rgb.data_ptr() if h_rgb is not None else None

    def timed(fn):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        layer.flush()
        e1.record(stream)
        barrier()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def streamed():
        slot = integ.stage_packed(hx, hc, off)
        for k in range(args.steps):
            layer.reset()
            nxt = integ.stage_packed(hx, hc, off) if k + 1 < args.steps else None
            integ.integrate_staged(slot, poses)
            slot = nxt

    def synchronous():
        for _ in range(args.steps):
            step(False)

    for _ in range(2):
        step(False)
    e2e_sync_ms = timed(synchronous)
    e2e_ms = timed(streamed)
    h2d = P * 12 + (P * 3 if rgb is not None else 0) + 8 * (F + 1) + 48 * F
    d2h = 24 * F

    # ---- rooflines (SURVEY.md 8d accounting): HBM-bound stages,
    # achieved = algorithmic bytes / the stage's CUDA-event time on the launching stream
    peak, peak_src = _peaks()
    dom = max(("emit", "record_sort", "runs", "apply", "bundle", "ray_order", "ray_setup"), key=lambda k: stages[k][0])
    n_upd = updates_per_step
    n_vox = info["n_vox"] / args.steps
    n_rec = info["records"] / args.steps
    passes = info["sort_passes"]
    prof_path = os.path.join(ROOT, "profiles", "roofline_inputs.json")
    prof = {}
    try:
        with open(prof_path) as f:
            prof = json.load(f)
    except Exception:
        pass

    def roof(stage, kernels, alg_bytes, model):
        t_ms = stages[stage][0] / args.steps
        ach = alg_bytes / (t_ms / 1e3) / 1e9 if t_ms > 0 else 0.0
        return {"bound": "hbm", "kernel": kernels, "stage": stage, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": prof.get(f"{stage}_dram_bytes_per_step"),
                "algorithmic_bytes": alg_bytes, "ms_per_step": t_ms, "peak_source": peak_src, "model": model}

    roof_sort = roof("record_sort", "k_sort_upsweep + k_sort_downsweep (x passes)", 20.0 * n_rec * passes,
                     f"LSD radix sort of 8-byte (voxel key, ray id) records, {passes} passes x (4 B upsweep read "
                     f"+ 8 B read + 8 B write) per record")
    roof_apply = roof("apply", "k_fold_all (long-run producer/consumer pairs + short runs, one grid)", 16.0 * n_upd + 24.0 * n_vox,
                      "16 B/update + 24 B/distinct voxel (SURVEY.md 8d); bound in practice by the longest "
                      "per-voxel chain (work.longest_fold_chain sequential steps)")
    roofline = roof_sort if stages["record_sort"][0] >= stages["apply"][0] else roof_apply

    # ---- CPU baseline (the reference, rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = cpu_reference_run(wc, packed, args.cpu_frames)
        if res is not None:
            u, dt = res
            cpu = {"value": u / dt, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"first {args.cpu_frames} frames of {wc.name}; unmodified reference sources (Eigen shim), "
                             f"g++ -O3, 1 thread, {dt:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_frame": ms_step / F,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic (seeded analytic room, workload.c; EuRoC/KITTI/Cow absent)",
            "config": {"workload": wc.name, "frames_per_step": F, "points_per_step": P, "updates_per_step": n_upd,
                       "merge": "grouped", "weight": "inverse_z2_dropoff", "voxel_size": wc.voxel_size,
                       "truncation": wc.truncation, "l2": "inputs 460 MB > 126 MB L2 (no flush)",
                       "parallelism": ((f"map sharded by block owner over {world} ranks, replicated traversal "
                                        f"(no record exchange)" if args.replicated else
                                        f"map sharded by block owner over {world} ranks, NCCL all-to-all of update "
                                        f"records") if world > 1 else "1 GPU")},
            "e2e": {"value": total_updates / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "api": "vxg_stage_packed + vxg_integrate_staged (pinned host input, step k+1 staged before "
                           "step k is integrated)",
                    "sync_one_call": {"value": total_updates / (e2e_sync_ms / 1e3), "ms_per_step": e2e_sync_ms,
                                      "api": "vxg_integrate_packed (pinned host input, H2D then compute)"}},
            "roofline": roofline,
            "roofline_stages": {"record_sort": roof_sort, "apply": roof_apply},
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
            "work": {"records_per_step": n_rec, "n_vox_per_step": n_vox,
                     "longest_fold_chain": info["max_chain"], "blocks": info["blocks"], "sort_passes": passes},
            "dominant_stage": dom,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

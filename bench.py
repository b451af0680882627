#!/usr/bin/env python3
"""Benchmark: TSDF voxel-updates/s and ms/frame on B200 vs the CPU reference.

Workloads (BASELINE.json configs, seeded synthetic scenes from
paper_1611_03631_b200/workload; the paper's datasets are not in the image):
  --config 1 (default, the metric's config): the 100-frame 640x480 RGB-D
      trajectory, merged integrator, 1/z^2 weight + drop-off, v = 0.05 m.
  --config 0: one 640x480 frame, simple integrator, constant weight.
  --config 2: 200 stereo-like 752x480 frames, v = 0.10 m.
  --config 3: 500 64-beam LiDAR scans (~120k returns), v = 0.20 m, 80 m rays.
  --config 4: 300 frames of 2048x2048, v = 0.02 m (integrated in batches of
      --frames-per-call frames: a whole step does not fit one call's records).
One STEP = integrate the whole trajectory into a fresh layer (reset + every
frame, batched; results identical to sequential integrate() calls).

  value : updates/s with inputs resident in HBM (device pointers), device time
          from CUDA events on the library's stream, max over ranks.
  e2e   : the same through the C ABI with pinned HOST buffers (H2D of points +
          colours and the per-frame stats D2H inside the timed region), fed as
          a stream (vxg_stage_packed starts step k+1's copy before
          vxg_integrate_staged integrates step k); e2e.sync_one_call =
          vxg_integrate_packed (copy, then compute, per call).
  latency_f1 : per-scan latency the way the reference's CLI times an insert
          (cli.cpp:168-174): one vxg_integrate call per frame from host
          memory, completed (vxg_flush) before the next; median / p90 beside
          the reference's median insert.
  --impl reference : the reference's own CPU integrator (oracle/_ref: the
          unmodified reference sources compiled with the Eigen shim), 1 thread
          pinned to one core (the reference is single-threaded), same frames.
Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) unless
already under torchrun. ONE map sharded by block-key ownership over the ranks
(SURVEY.md §8e): every rank bundles the batch, walks a record-balanced slice
of the ray order and routes update records to the block owners with an NCCL
all-to-all inside the library; total work is fixed (strong scaling), value =
total updates / max-over-ranks step time. Ranks > 0 of the reference arm exit
without work.
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

# frames per step (= the config's trajectory) and frames per integrate call
STEP = {0: (1, 1), 1: (100, 100), 2: (200, 200), 3: (500, 500), 4: (300, 4)}
CPU_BUDGET_S = 20.0  # cpu_baseline sample: whole trajectory, or the first frames within ~this


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
            self._stop.wait(0.1)

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


def common_config(wc, frames: int) -> dict:
    """`config` shared by both arms (same workload => same dict)."""
    return {"workload": wc.name, "frames_per_step": frames,
            "merge": ["simple", "grouped", "grouped_anti_graze"][wc.merge_mode],
            "weight": ["constant", "inverse_z2", "inverse_z2_dropoff"][wc.weight_mode],
            "voxel_size": wc.voxel_size, "truncation": wc.truncation, "max_ray": wc.max_ray,
            "l2": "inputs and per-step records exceed the 126 MB L2 (no flush needed)"}


def pin_one_core():
    """taskset -c <first allowed core>: the reference is single-threaded."""
    try:
        cores = sorted(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cores[0]})
        return cores[0]
    except Exception:
        return None


def cpu_reference_run(wc, packed, frames: int, budget_s: float = 0.0):
    """The unmodified reference integrator (oracle/_ref), 1 thread, frames in
    order into a fresh layer. Per-frame time = steady_clock around integrate()
    inside the reference library (benchmark.cpp:93-95). budget_s > 0 stops
    after the frame that crosses the budget. Returns (updates, seconds,
    per-frame seconds) or None when _ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import RefLayer, ref_available
    from paper_1611_03631_b200 import workload as W
    if not ref_available():
        return None
    xyz, rgb, off, poses = packed
    layer = RefLayer(W.tsdf_config(wc), wc.voxel_size, wc.vps)
    upd, per = 0, []
    for f in range(frames):
        a, b = int(off[f]), int(off[f + 1])
        u, _, _ = layer.integrate(xyz[a:b], None if rgb is None else rgb[a:b], poses[f])
        per.append(layer.last_integrate_seconds())
        upd += u
        if budget_s > 0 and sum(per) > budget_s:
            break
    return upd, sum(per), per


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    core = pin_one_core()
    F = args.frames
    wc, packed = load_workload(args.config, F)
    if cpu_reference_run(wc, packed, 1) is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libvxfref.so not built"}))
        return
    # warm-up steps integrate one frame (a CPU integrator has no warm-up state to build)
    for _ in range(args.warmup):
        cpu_reference_run(wc, packed, 1)
    times, upds, per = [], [], []
    ref_frames = F if args.ref_frames is None else min(F, args.ref_frames)
    for _ in range(args.steps):
        u, dt, pf = cpu_reference_run(wc, packed, ref_frames)
        times.append(dt)
        upds.append(u)
        per += pf
    value = sum(upds) / sum(times)
    same = ref_frames == F
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "ms_per_frame": 1e3 * sum(times) / (len(times) * ref_frames),
        "median_insert_ms": 1e3 * statistics.median(per),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32+f64", "data": "synthetic (seeded analytic scenes, workload.c)",
        "config": common_config(wc, F if same else ref_frames),
        "same_config": same,
        "parallelism": f"1 thread pinned to core {core} of {os.cpu_count()} (the reference is single-threaded)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"frames 0..{ref_frames - 1} of {wc.name} per step; steady_clock around "
                                   f"integrate() (benchmark.cpp:93-95); warm-up steps integrate 1 frame",
                         "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: relaunch this script as N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vxg", choices=["vxg", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(STEP))
    ap.add_argument("--frames", type=int, default=None, help="frames per step (default: the config's trajectory)")
    ap.add_argument("--frames-per-call", type=int, default=None)
    ap.add_argument("--ref-frames", type=int, default=None, help="reference arm: frames per step (default: all)")
    ap.add_argument("--cpu-budget", type=float, default=CPU_BUDGET_S)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--sharded-nccl", action="store_true",
                    help="run the sharded NCCL path even at N=1 (1-rank communicator, NCCL self send/recv)")
    ap.add_argument("--replicated", action="store_true",
                    help="N>1: replicated traversal (every rank walks all rays, no record exchange)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.frames is None:
        args.frames = STEP[args.config][0]
    if args.frames_per_call is None:
        args.frames_per_call = min(args.frames, STEP[args.config][1])

    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        sys.exit(spawn_ranks(args))
    if world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)

    if args.impl == "reference":
        run_reference_arm(args)
        return
    run_vxg_arm(args)


def run_vxg_arm(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
    from paper_1611_03631_b200 import workload as W

    wc, packed = load_workload(args.config, args.frames)
    xyz, rgb, off, poses = packed
    F = len(poses)
    P = int(off[-1])
    FC = args.frames_per_call
    calls = [(f0, min(F, f0 + FC)) for f0 in range(0, F, FC)]
    cfg = W.tsdf_config(wc)

    stream = torch.cuda.current_stream()
    layer = TsdfLayer(wc.voxel_size, wc.vps, device=local, block_capacity=1024)
    layer.set_stream(stream.cuda_stream)
    if world > 1:
        from paper_1611_03631_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        layer.shard_init(rank, world, obj[0], replicated=args.replicated)
    elif args.sharded_nccl:
        from paper_1611_03631_b200 import nccl_unique_id
        layer.shard_init(0, 1, nccl_unique_id(), replicated=args.replicated)
    integ = TsdfIntegrator(cfg, layer)

    d_xyz = torch.from_numpy(xyz).cuda()
    d_rgb = torch.from_numpy(rgb).cuda() if rgb is not None else None
    h_xyz = torch.from_numpy(xyz).pin_memory()
    h_rgb = torch.from_numpy(rgb).pin_memory() if rgb is not None else None
    offs = [np.ascontiguousarray(off[a:b + 1]) for a, b in calls]

    def step(device_input: bool):
        layer.reset()
        out = []
        for (a, b), o in zip(calls, offs):
            if device_input:
                out.append(integ.integrate_packed(d_xyz.data_ptr(), d_rgb.data_ptr() if d_rgb is not None else None,
                                                  o, poses[a:b], True))
            else:
                out.append(integ.integrate_packed(h_xyz.data_ptr(), h_rgb.data_ptr() if h_rgb is not None else None,
                                                  o, poses[a:b], False))
        return np.concatenate(out)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
    dev_ms = max_over_ranks(t0.elapsed_time(t1))
    stages = layer.stage_times(reset=True)
    launches = layer.kernel_launches(reset=True)
    info = layer.batch_info(reset=True)
    layer.profile(False)
    ms_step = dev_ms / args.steps
    total_updates = updates_per_step  # one sharded map: stats are global on every rank
    value = total_updates / (ms_step / 1e3)

    # ---- e2e: pinned host inputs through the C ABI (every step's H2D and its
    # stats D2H inside the timed region). Streamed: step k+1's batch is staged
    # (vxg_stage_packed) before step k is integrated (vxg_integrate_staged), so
    # the copy overlaps compute. Also timed: the synchronous one-call path.
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
        return max_over_ranks(e0.elapsed_time(e1) / args.steps)

    def streamed():
        seq = [(k, c) for k in range(args.steps) for c in range(len(calls))]
        slot = integ.stage_packed(hx, hc, offs[0])
        for i, (k, c) in enumerate(seq):
            if c == 0:
                layer.reset()
            nk = seq[i + 1][1] if i + 1 < len(seq) else None
            nxt = integ.stage_packed(hx, hc, offs[nk]) if nk is not None else None
            a, b = calls[c]
            integ.integrate_staged(slot, poses[a:b])
            slot = nxt

    def synchronous():
        for _ in range(args.steps):
            step(False)

    for _ in range(2):
        step(False)
    e2e_sync_ms = timed(synchronous)
    e2e_ms = timed(streamed)
    h2d = P * 12 + (P * 3 if rgb is not None else 0) + 8 * (F + len(calls)) + 48 * F
    d2h = 24 * F
    # in-run H2D bandwidth of the same pinned inputs (plain copy, outside the timed regions)
    bw_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    bw_ev[0].record(stream)
    d_xyz.copy_(h_xyz, non_blocking=True)
    if h_rgb is not None:
        d_rgb.copy_(h_rgb, non_blocking=True)
    bw_ev[1].record(stream)
    torch.cuda.synchronize()
    h2d_gbs = (P * 12 + (P * 3 if rgb is not None else 0)) / (bw_ev[0].elapsed_time(bw_ev[1]) / 1e3) / 1e9

    # ---- per-scan latency (F = 1 per call, host input, each call completed
    # before the next, as the reference's CLI inserts one scan at a time)
    lat = None
    if not args.no_latency and world == 1:
        nl = min(F, 100)
        per = []
        layer.reset()
        layer.flush()
        for f in range(nl):
            o = np.array([off[f], off[f + 1]], dtype=np.uint64)
            torch.cuda.synchronize()
            t_a = time.perf_counter()
            integ.integrate_packed(hx, hc, o, poses[f:f + 1], False)
            layer.flush()
            torch.cuda.synchronize()  # vxg_flush only orders the handle's stream behind the fold: wait on the host
            per.append(time.perf_counter() - t_a)
        per_ms = sorted(1e3 * x for x in per)
        lat = {"frames": nl, "median_ms": statistics.median(per_ms),
               "p90_ms": per_ms[min(len(per_ms) - 1, int(0.9 * len(per_ms)))], "mean_ms": statistics.mean(per_ms),
               "api": "vxg_integrate_packed with F=1 from pinned host memory + vxg_flush + a host wait for the "
                      "device (the layer is final in HBM when the clock stops); host steady clock per call, like "
                      "cli.cpp:171-174"}

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
            prof = json.load(f).get(wc.name, {})
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
    roof_apply = roof("apply", "k_fold_all (long-run producer/consumer pairs + short runs, one grid)",
                      16.0 * n_upd + 24.0 * n_vox,
                      "16 B/update + 24 B/distinct voxel (SURVEY.md 8d); bound in practice by the longest "
                      "per-voxel chain (work.longest_fold_chain sequential steps)")
    roofline = roof_sort if stages["record_sort"][0] >= stages["apply"][0] else roof_apply

    # ---- CPU baseline (the reference, rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        core = pin_one_core()
        res = cpu_reference_run(wc, packed, F, budget_s=args.cpu_budget)
        try:
            os.sched_setaffinity(0, set(range(os.cpu_count() or 1)))
        except Exception:
            pass
        if res is not None:
            u, dt, per_f = res
            nf = len(per_f)
            cpu = {"value": u / dt, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": (f"{'all' if nf == F else 'first'} {nf} of {F} frames of {wc.name} into a fresh layer; "
                              f"unmodified reference sources (Eigen shim), g++ -O3, 1 thread pinned to core {core} "
                              f"of {os.cpu_count()}; steady_clock around integrate(), {dt:.2f} s"
                              + ("" if nf == F else "; the remaining frames are not timed (rate extrapolated)")),
                   "median_insert_ms": 1e3 * statistics.median(per_f), "frames": nf, "nproc": os.cpu_count()}

    api_streamed = ("vxg_stage_packed + vxg_integrate_staged (pinned host input, the next batch staged before this "
                    "one is integrated)")
    api_sync = "vxg_integrate_packed (pinned host input, H2D then compute)"
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_frame": ms_step / F,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic (seeded analytic scenes, workload.c; EuRoC/KITTI/Cow absent)",
            "config": common_config(wc, F),
            "parallelism": ((f"map sharded by block owner over {world} ranks, replicated traversal (no record "
                             f"exchange)" if args.replicated else
                             f"map sharded by block owner over {world} ranks, NCCL all-to-all of update records")
                            if world > 1 else ("1 GPU, sharded path over a 1-rank NCCL communicator"
                                               if args.sharded_nccl else "1 GPU")),
            "work": {"points_per_step": P, "updates_per_step": n_upd, "frames_per_call": FC,
                     "records_per_step": n_rec, "n_vox_per_step": n_vox, "longest_fold_chain": info["max_chain"],
                     "blocks": info["blocks"], "sort_passes": passes},
            # both host-input entry points are timed with their H2D copies inside the region; the headline is
            # the faster one ON THIS BOX (the streamed path depends on how well the box overlaps DMA with compute)
            "e2e": {"value": total_updates / (min(e2e_ms, e2e_sync_ms) / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": min(e2e_ms, e2e_sync_ms),
                    "api": api_streamed if e2e_ms <= e2e_sync_ms else api_sync,
                    "h2d_gbs_in_run": h2d_gbs,
                    "streamed": {"value": total_updates / (e2e_ms / 1e3), "ms_per_step": e2e_ms, "api": api_streamed},
                    "sync_one_call": {"value": total_updates / (e2e_sync_ms / 1e3), "ms_per_step": e2e_sync_ms,
                                      "api": api_sync}},
            "latency_f1": lat,
            "ms_per_frame_f1": lat["median_ms"] if lat else None,
            "roofline": roofline,
            "roofline_stages": {"record_sort": roof_sort, "apply": roof_apply},
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
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

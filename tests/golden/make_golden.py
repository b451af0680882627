#!/usr/bin/env python3
"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the
unmodified /root/reference sources compiled against oracle/eigen_shim).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Each fixture stores the inputs (per-frame xyz / rgb / pose), the TsdfConfig,
the layer geometry, the reference's per-frame integrate() counters and the
reference's VXBLX bytes (zlib-compressed inside the npz). The GPU and oracle
tests replay the inputs and must reproduce the bytes exactly.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bindings import RefLayer, ref_available  # noqa: E402
from paper_1611_03631_b200 import workload as W  # noqa: E402
from paper_1611_03631_b200.tsdf import MergeMode, TsdfConfig, WeightMode  # noqa: E402


def plane_scan(wall_x, rays_y, rays_z, spread):
    """The reference tests' plane_scan (test_tsdf_integrator.cpp:122-133)."""
    pts = []
    for iy in range(rays_y):
        for iz in range(rays_z):
            y = np.float32(spread) * (np.float32(2.0) * np.float32(iy) / np.float32(rays_y - 1) - np.float32(1.0))
            z = np.float32(spread) * (np.float32(2.0) * np.float32(iz) / np.float32(rays_z - 1) - np.float32(1.0))
            pts.append((wall_x, y, z))
    return np.array(pts, dtype=np.float32)


def pole_scene():
    """Pole in front of a wall (test_tsdf_integrator.cpp:366-383)."""
    pts = [(2.05, 0.05, 0.025 * iz + 0.01) for iz in range(8)]
    pts += [(4.0, -1.0 + 0.04 * iy, 0.05 * iz - 0.5) for iy in range(60) for iz in range(30)]
    return np.array(pts, dtype=np.float32)


def test_config(v, merge, weight):  # test_tsdf_integrator.cpp:113-120
    c = TsdfConfig.for_voxel_size(v)
    c.merge_mode, c.weight_mode = merge, weight
    c.min_ray_length, c.max_ray_length = 0.05, 20.0
    return c


IDENT = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], np.float32)


def cases():
    out = []
    for cfg_id, nf, scale in [(0, 1, 0.1), (1, 2, 0.07), (2, 2, 0.07), (3, 1, 0.05)]:
        wc = W.CONFIGS[cfg_id]
        frames = [W.frame(cfg_id, f * 9, scale, wc.frames) for f in range(nf)]
        out.append((f"cfg{cfg_id}_scale{scale}", W.tsdf_config(wc), wc.voxel_size, wc.vps, frames))
    rng = np.random.default_rng(7)
    for merge in MergeMode:
        for weight in WeightMode:
            fr = [(plane_scan(np.float32(3.0), 20, 20, 0.5), rng.integers(0, 256, (400, 3), dtype=np.uint8), IDENT)]
            out.append((f"plane_{merge.name}_{weight.name}", test_config(0.2, merge, weight), 0.2, 16, fr))
    for merge in (MergeMode.kGroupedRaycast, MergeMode.kGroupedAntiGraze):
        out.append((f"pole_{merge.name}", test_config(0.2, merge, WeightMode.kConstant), 0.2, 16,
                    [(pole_scene(), None, IDENT)]))
    single = np.array([[1.0, 0.0, 0.0]], np.float32)
    out.append(("single_point_simple", test_config(0.1, MergeMode.kSimpleRaycast, WeightMode.kConstant), 0.1, 16,
                [(single, None, IDENT)]))
    out.append(("two_points_simple", test_config(0.1, MergeMode.kSimpleRaycast, WeightMode.kConstant), 0.1, 16,
                [(np.repeat(single, 2, axis=0), None, IDENT)]))
    rays = rng.normal(size=(300, 3)).astype(np.float32)
    rays *= (rng.uniform(0.3, 3.0, (300, 1)) / np.linalg.norm(rays, axis=1, keepdims=True)).astype(np.float32)
    pose = np.array([0.36, -0.48, 0.8, 1.5, 0.8, 0.6, 0.0, -2.25, -0.48, 0.64, 0.6, 0.75], np.float32)
    out.append(("random_posed_grouped_dropoff",
                test_config(0.07, MergeMode.kGroupedRaycast, WeightMode.kInverseZ2Dropoff), 0.07, 8,
                [(rays, rng.integers(0, 256, (300, 3), dtype=np.uint8), pose), (rays[::-1].copy(), None, IDENT)]))
    bounded = test_config(0.1, MergeMode.kSimpleRaycast, WeightMode.kConstant)
    bounded.min_ray_length, bounded.max_ray_length = 0.5, 2.0
    out.append(("out_of_range_skips", bounded, 0.1, 16,
                [(np.array([[0.2, 0, 0], [5.0, 0, 0], [1.0, 0, 0]], np.float32), None, IDENT)]))
    out.append(("empty_scan", test_config(0.1, MergeMode.kGroupedRaycast, WeightMode.kInverseZ2), 0.1, 16,
                [(np.zeros((0, 3), np.float32), None, IDENT)]))
    return out


def main():
    if not ref_available():
        sys.exit("oracle/_ref/libvxfref.so missing: build it in the container with /root/reference (make -C oracle)")
    for name, cfg, v, vps, frames in cases():
        ref = RefLayer(cfg, v, vps)
        stats = [ref.integrate(x, c, p) for (x, c, p) in frames]
        blob = ref.save_bytes()
        arrays = {"vxblx": np.frombuffer(blob, dtype=np.uint8)}
        for i, (x, c, p) in enumerate(frames):
            arrays[f"xyz{i}"] = x
            arrays[f"pose{i}"] = np.asarray(p, np.float32).reshape(12)
            if c is not None:
                arrays[f"rgb{i}"] = c
        meta = {"name": name, "voxel_size": v, "vps": vps, "frames": len(frames), "stats": stats,
                "config": {"truncation": cfg.truncation, "dropoff_epsilon": cfg.dropoff_epsilon,
                           "max_weight": cfg.max_weight, "weight_mode": int(cfg.weight_mode),
                           "merge_mode": int(cfg.merge_mode), "min_ray_length": cfg.min_ray_length,
                           "max_ray_length": cfg.max_ray_length},
                "generator": "oracle/_ref (unmodified reference sources + eigen_shim)"}
        arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        print(f"{name}: stats={stats} vxblx={len(blob)} bytes")


if __name__ == "__main__":
    main()

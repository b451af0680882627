"""Seeded synthetic workloads for BASELINE.json configs[0..4].

BENCH / TEST INPUT GENERATION ONLY (not the measured path). The paper's
datasets are absent; analytic scenes rendered by workload.c stand in for them
with BASELINE.json's shapes, sizes and noise models. `scale` shrinks the image
(intrinsics scaled alike) for parity tests that must finish in seconds on the
CPU oracle.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libworkload.so")

SEED = 1  # scene=1 (+2 trajectory, +3 noise, +4 colour, +5 invalidation inside workload.c)


class Prim(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("up", ctypes.c_int32), ("a", ctypes.c_double * 6)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make workload`")
        L = ctypes.CDLL(LIB_PATH)
        L.wl_make_scene.restype = ctypes.c_int
        L.wl_make_scene.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(Prim), ctypes.c_int]
        L.wl_pose.restype = None
        L.wl_pose.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_float)]
        L.wl_render_pinhole.restype = ctypes.c_int64
        L.wl_render_pinhole.argtypes = [ctypes.POINTER(Prim), ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                        ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.wl_render_lidar.restype = ctypes.c_int64
        L.wl_render_lidar.argtypes = [ctypes.POINTER(Prim), ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                      ctypes.POINTER(Prim)]
        _lib = L
    return _lib


@dataclass(frozen=True)
class WorkloadConfig:
    """One BASELINE.json config: sensor model + TsdfConfig."""
    cfg: int
    name: str
    frames: int
    sensor: str  # "pinhole" | "lidar"
    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    noise_k: float = 0.0      # sigma = noise_k * z^2 (pinhole)
    drop_prob: float = 0.0
    rgb: bool = True
    beams: int = 0
    elev_lo: float = 0.0
    elev_hi: float = 0.0
    az_step: float = 0.0
    range_sigma: float = 0.0
    lidar_range: float = 0.0
    # TsdfConfig
    voxel_size: float = 0.05
    truncation: float = 0.1
    dropoff_epsilon: float = 0.05
    max_weight: float = 1e4
    weight_mode: int = 2
    merge_mode: int = 1
    min_ray: float = 0.05
    max_ray: float = 5.0
    vps: int = 16


CONFIGS = {
    0: WorkloadConfig(0, "cfg0_rgbd_simple_640x480", 1, "pinhole", 640, 480, 525.0, 525.0, 319.5, 239.5, 0.005, 0.0,
                      True, voxel_size=0.05, truncation=0.10, dropoff_epsilon=0.05, weight_mode=0, merge_mode=0,
                      min_ray=0.05, max_ray=5.0),
    1: WorkloadConfig(1, "cfg1_rgbd_merged_640x480_x100", 100, "pinhole", 640, 480, 525.0, 525.0, 319.5, 239.5, 0.005,
                      0.0, True, voxel_size=0.05, truncation=0.10, dropoff_epsilon=0.05, weight_mode=2, merge_mode=1,
                      min_ray=0.05, max_ray=5.0),
    2: WorkloadConfig(2, "cfg2_stereo_merged_752x480_x200", 200, "pinhole", 752, 480, 470.0, 470.0, 375.5, 239.5,
                      0.02, 0.10, True, voxel_size=0.10, truncation=0.30, dropoff_epsilon=0.10, weight_mode=2,
                      merge_mode=1, min_ray=0.05, max_ray=8.0),
    3: WorkloadConfig(3, "cfg3_lidar64_merged_x500", 500, "lidar", rgb=False, beams=64, elev_lo=-24.8, elev_hi=2.0,
                      az_step=0.17, range_sigma=0.02, lidar_range=80.0, voxel_size=0.20, truncation=0.60,
                      dropoff_epsilon=0.20, weight_mode=2, merge_mode=1, min_ray=0.05, max_ray=80.0),
    4: WorkloadConfig(4, "cfg4_rgbd_merged_2048x2048_x300", 300, "pinhole", 2048, 2048, 1500.0, 1500.0, 1023.5,
                      1023.5, 0.005, 0.0, True, voxel_size=0.02, truncation=0.06, dropoff_epsilon=0.02, weight_mode=2,
                      merge_mode=1, min_ray=0.05, max_ray=10.0),
}


def tsdf_config(wc: WorkloadConfig, merge_mode: Optional[int] = None, weight_mode: Optional[int] = None):
    from ..tsdf import MergeMode, TsdfConfig, WeightMode
    return TsdfConfig(truncation=wc.truncation, dropoff_epsilon=wc.dropoff_epsilon, max_weight=wc.max_weight,
                      weight_mode=WeightMode(wc.weight_mode if weight_mode is None else weight_mode),
                      merge_mode=MergeMode(wc.merge_mode if merge_mode is None else merge_mode),
                      min_ray_length=wc.min_ray, max_ray_length=wc.max_ray)


_scene_cache = {}


def scene(cfg: int):
    if cfg not in _scene_cache:
        buf = (Prim * 4096)()
        n = lib().wl_make_scene(cfg, SEED, buf, 4096)
        _scene_cache[cfg] = (buf, min(n, 4096))
    return _scene_cache[cfg]


def pose(cfg: int, frame: int, n_frames: Optional[int] = None) -> np.ndarray:
    wc = CONFIGS[cfg]
    out = np.zeros(12, dtype=np.float32)
    lib().wl_pose(cfg, frame, n_frames or wc.frames, SEED + 1, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    return out


def frame(cfg: int, f: int, scale: float = 1.0, n_frames: Optional[int] = None
          ) -> Tuple[np.ndarray, Optional[np.ndarray], np.ndarray]:
    """(xyz [N,3] float32 sensor frame, rgb [N,3] uint8 or None, pose [12] float32).

    scale < 1 renders a smaller image with proportionally scaled intrinsics
    (pinhole) or a coarser azimuth step (LiDAR)."""
    wc = CONFIGS[cfg]
    prims, n = scene(cfg)
    P = pose(cfg, f, n_frames)
    pp = P.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    if wc.sensor == "pinhole":
        W = max(2, int(round(wc.width * scale)))
        H = max(2, int(round(wc.height * scale)))
        sx, sy = W / wc.width, H / wc.height
        xyz = np.zeros((W * H, 3), dtype=np.float32)
        rgb = np.zeros((W * H, 3), dtype=np.uint8) if wc.rgb else None
        k = lib().wl_render_pinhole(prims, n, pp, W, H, wc.fx * sx, wc.fy * sy, (wc.cx + 0.5) * sx - 0.5,
                                    (wc.cy + 0.5) * sy - 0.5, 1e30, wc.noise_k, wc.drop_prob, SEED, f,
                                    xyz.ctypes.data_as(ctypes.c_void_p),
                                    rgb.ctypes.data_as(ctypes.c_void_p) if rgb is not None else None)
        return xyz[:k].copy(), (rgb[:k].copy() if rgb is not None else None), P
    az = wc.az_step / scale
    steps = int(np.ceil(360.0 / az - 1e-9))
    xyz = np.zeros((steps * wc.beams, 3), dtype=np.float32)
    scratch = (Prim * 4096)()
    k = lib().wl_render_lidar(prims, n, pp, wc.beams, wc.elev_lo, wc.elev_hi, az, wc.lidar_range, wc.range_sigma,
                              SEED, f, xyz.ctypes.data_as(ctypes.c_void_p), scratch)
    return xyz[:k].copy(), None, P


def frames(cfg: int, count: Optional[int] = None, scale: float = 1.0, start: int = 0,
           n_frames: Optional[int] = None) -> List[Tuple[np.ndarray, Optional[np.ndarray], np.ndarray]]:
    wc = CONFIGS[cfg]
    count = wc.frames if count is None else count
    return [frame(cfg, start + i, scale, n_frames) for i in range(count)]


def pack(frames_list) -> Tuple[np.ndarray, Optional[np.ndarray], np.ndarray, np.ndarray]:
    """Packs frames into (xyz [P,3], rgb [P,3] | None, offsets [F+1] uint64, poses [F,12])."""
    xyz = np.concatenate([f[0] for f in frames_list]).astype(np.float32, copy=False)
    has_rgb = all(f[1] is not None for f in frames_list)
    rgb = np.concatenate([f[1] for f in frames_list]) if has_rgb else None
    offsets = np.zeros(len(frames_list) + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum([len(f[0]) for f in frames_list])
    poses = np.stack([f[2] for f in frames_list]).astype(np.float32)
    return np.ascontiguousarray(xyz), rgb, offsets, poses

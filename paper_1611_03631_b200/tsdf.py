"""Python mirror of the reference integrator interface, backed by the B200 C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/vxf/tsdf_integrator.h, layer.h, scan.h,
serialization.h), so parity tests read like the reference's own tests:

    layer = TsdfLayer(0.1, 16)
    integrator = TsdfIntegrator(TsdfConfig.for_voxel_size(0.1), layer)
    updates = integrator.integrate(Scan(points, colors, pose))
    integrator.raycasts_last_scan(); layer.voxel_ptr((gx, gy, gz))

std::invalid_argument -> ValueError (same message text); vxf::ParseError ->
ParseError. Everything runs on the GPU through libvxg.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from ._capi import (ParseError, VXG_INPUT_DEVICE, VXG_INPUT_HOST, VxgEsdfConfig, VxgFrame, VxgMcTables, VxgStats,
                    VxgTsdfConfig, VxgVoxel,
                    check, lib)

VOXEL_DTYPE = np.dtype([("distance", "<f4"), ("weight", "<f4"), ("r", "u1"), ("g", "u1"), ("b", "u1"),
                        ("pad", "u1")])
K_TSDF_OBSERVED_WEIGHT = np.float32(1e-4)  # core.h:32


class WeightMode(enum.IntEnum):  # tsdf_integrator.h:11-15
    kConstant = 0
    kInverseZ2 = 1
    kInverseZ2Dropoff = 2


class MergeMode(enum.IntEnum):  # tsdf_integrator.h:17-21
    kSimpleRaycast = 0
    kGroupedRaycast = 1
    kGroupedAntiGraze = 2


@dataclass
class TsdfConfig:  # tsdf_integrator.h:23-41
    truncation: float = 0.4
    dropoff_epsilon: float = 0.1
    max_weight: float = 1e4
    weight_mode: WeightMode = WeightMode.kInverseZ2Dropoff
    merge_mode: MergeMode = MergeMode.kGroupedRaycast
    min_ray_length: float = 0.05
    max_ray_length: float = 10.0

    @staticmethod
    def for_voxel_size(v: float) -> "TsdfConfig":
        v32 = float(np.float32(v))
        return TsdfConfig(truncation=float(np.float32(4.0) * np.float32(v32)), dropoff_epsilon=v32)

    def to_c(self) -> VxgTsdfConfig:
        return VxgTsdfConfig(self.truncation, self.dropoff_epsilon, self.max_weight, int(self.weight_mode),
                             int(self.merge_mode), self.min_ray_length, self.max_ray_length)

    def validate(self) -> None:  # tsdf_integrator.cpp:10-20 (same messages)
        f = np.float32
        if not (f(self.dropoff_epsilon) > 0) or not (f(self.dropoff_epsilon) < f(self.truncation)):
            raise ValueError("tsdf config requires 0 < dropoff_epsilon < truncation")
        if not (f(self.min_ray_length) >= 0) or not (f(self.min_ray_length) < f(self.max_ray_length)):
            raise ValueError("tsdf config requires 0 <= min_ray_length < max_ray_length")
        if not (f(self.max_weight) > 0):
            raise ValueError("tsdf config requires max_weight > 0")


def pose_3x4(pose) -> np.ndarray:
    """Accepts None (identity), a 3x4 [R|t], a 4x4 homogeneous matrix or 12 floats."""
    if pose is None:
        return np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], dtype=np.float32)
    a = np.asarray(pose, dtype=np.float32)
    if a.shape == (4, 4):
        a = a[:3, :]
    return np.ascontiguousarray(a.reshape(12), dtype=np.float32)


@dataclass
class Scan:  # scan.h:13-20
    points: np.ndarray
    colors: Optional[np.ndarray] = None
    pose: np.ndarray = field(default_factory=lambda: pose_3x4(None))

    def __post_init__(self):
        self.points = np.ascontiguousarray(np.asarray(self.points, dtype=np.float32).reshape(-1, 3))
        if self.colors is not None:
            c = np.asarray(self.colors)
            self.colors = None if c.size == 0 else np.ascontiguousarray(c.astype(np.uint8).reshape(-1, 3))
        self.pose = pose_3x4(self.pose)

    def has_colors(self) -> bool:
        return self.colors is not None

    def origin(self) -> np.ndarray:
        return self.pose.reshape(3, 4)[:, 3].copy()


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class TsdfLayer:
    """Device-resident block-hashed TSDF layer (layer.h:56-164) on one B200.

    The layer owns the device handle (slab + block hash + stream); integrators
    attach their config to it for the duration of each integrate call.
    """

    def __init__(self, voxel_size: float, voxels_per_side: int = 16, device: int = 0, block_capacity: int = 0,
                 _config: Optional[TsdfConfig] = None):
        if not (np.float32(voxel_size) > 0) or voxels_per_side < 1:
            raise ValueError("layer requires voxel_size > 0 and voxels_per_side >= 1")
        self._voxel_size = float(np.float32(voxel_size))
        self._vps = int(voxels_per_side)
        self._device = int(device)
        self._h = ctypes.c_void_p()
        cfg = (_config or TsdfConfig.for_voxel_size(self._voxel_size)).to_c()
        check(lib().vxg_create(ctypes.byref(cfg), self._voxel_size, self._vps, self._device, int(block_capacity),
                               ctypes.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().vxg_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- geometry (layer.h:69-72)
    def voxel_size(self) -> float:
        return self._voxel_size

    def voxels_per_side(self) -> int:
        return self._vps

    def block_size(self) -> float:
        return float(np.float32(self._voxel_size) * np.float32(self._vps))

    def block_count(self) -> int:
        n = ctypes.c_uint64()
        check(lib().vxg_block_count(self._h, ctypes.byref(n)))
        return int(n.value)

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # ---- export / query
    def export_blocks(self) -> Tuple[np.ndarray, np.ndarray]:
        """Blocks in save_layer order (x,y,z-sorted): (idx [B,3] int32, voxels [B, vps^3] VOXEL_DTYPE)."""
        nb = self.block_count()
        nv = self._vps ** 3
        idx = np.zeros((nb, 3), dtype=np.int32)
        vox = np.zeros((nb, nv), dtype=VOXEL_DTYPE)
        n = ctypes.c_uint64()
        check(lib().vxg_export_blocks(self._h, _ptr(idx), _ptr(vox), nb, ctypes.byref(n)))
        return idx[: n.value], vox[: n.value]

    def blocks(self) -> Dict[Tuple[int, int, int], np.ndarray]:
        idx, vox = self.export_blocks()
        return {tuple(int(v) for v in i): vox[k] for k, i in enumerate(idx)}

    def import_blocks(self, idx: np.ndarray, voxels: np.ndarray) -> None:
        idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, 3)
        voxels = np.ascontiguousarray(voxels).view(VOXEL_DTYPE).reshape(len(idx), -1)
        check(lib().vxg_import_blocks(self._h, _ptr(idx), _ptr(voxels), len(idx)))

    def query(self, g: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """voxel_ptr for many global indices: (voxels, found)."""
        g = np.ascontiguousarray(g, dtype=np.int32).reshape(-1, 3)
        out = np.zeros(len(g), dtype=VOXEL_DTYPE)
        found = np.zeros(len(g), dtype=np.uint8)
        if len(g):
            check(lib().vxg_query_voxels(self._h, _ptr(g), len(g), _ptr(out), _ptr(found)))
        return out, found.astype(bool)

    def interpolate_distance(self, points: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """interpolate_distance (interpolation.h:28-60) for many world points:
        (distance, found); found is False where the reference returns nullopt."""
        p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        d = np.zeros(len(p), dtype=np.float32)
        found = np.zeros(len(p), dtype=np.uint8)
        if len(p):
            check(lib().vxg_interpolate_distance(self._h, _ptr(p), len(p), _ptr(d), _ptr(found), 0))
        return d, found.astype(bool)

    def surface_error(self, ground_truth_points: np.ndarray, truncation: float) -> Dict[str, float]:
        """surface_error (analysis.cpp:41-59): ErrorStats as a dict
        (rms, mean, max, count, unknown_fraction)."""
        p = np.ascontiguousarray(ground_truth_points, dtype=np.float32).reshape(-1, 3)
        out = np.zeros(5, dtype=np.float64)
        check(lib().vxg_surface_error(self._h, _ptr(p), len(p), float(truncation), _ptr(out)))
        return {"rms": float(out[0]), "mean": float(out[1]), "max": float(out[2]), "count": int(out[3]),
                "unknown_fraction": float(out[4])}

    def voxel_ptr(self, g) -> Optional[np.void]:
        """Layer::voxel_ptr (layer.h:99-112): None when the block is unallocated."""
        out, found = self.query(np.asarray(g, dtype=np.int32).reshape(1, 3))
        return out[0] if found[0] else None

    # ---- serialization (serialization.h)
    def save_bytes(self) -> bytes:
        need = ctypes.c_uint64()
        check(lib().vxg_serialize_vxblx(self._h, None, 0, ctypes.byref(need)))
        buf = np.zeros(need.value, dtype=np.uint8)
        check(lib().vxg_serialize_vxblx(self._h, _ptr(buf), need.value, ctypes.byref(need)))
        return buf.tobytes()

    def save_file(self, path: str) -> None:
        check(lib().vxg_save_vxblx(self._h, path.encode()))

    def load_bytes(self, data: bytes) -> None:
        buf = np.frombuffer(data, dtype=np.uint8)
        check(lib().vxg_load_vxblx(self._h, buf.ctypes.data_as(ctypes.c_void_p), len(buf)))
        hdr_v = np.frombuffer(data[10:18], dtype="<f8")[0] if len(data) >= 18 else self._voxel_size
        self._voxel_size = float(np.float32(hdr_v))
        if len(data) >= 22:
            self._vps = int(np.frombuffer(data[18:22], dtype="<u4")[0])

    def reset(self) -> None:
        check(lib().vxg_reset(self._h))

    def flush(self) -> None:
        """Order the handle's stream after the last batch's fold (no host sync):
        an event recorded afterwards covers the whole integration."""
        check(lib().vxg_flush(self._h))

    # ---- updated-block consumers (layer.h:124-148)
    def register_consumer(self, name: str) -> None:
        check(lib().vxg_register_consumer(self._h, name.encode()))

    def drain_updated(self, name: str) -> set:
        n = ctypes.c_uint64()
        check(lib().vxg_drain_updated(self._h, name.encode(), None, 0, ctypes.byref(n)))
        idx = np.zeros((max(n.value, 1), 3), dtype=np.int32)
        check(lib().vxg_drain_updated(self._h, name.encode(), _ptr(idx), n.value, ctypes.byref(n)))
        return {tuple(int(v) for v in i) for i in idx[: n.value]}

    # ---- stage profiling
    def profile(self, enable: bool = True) -> None:
        check(lib().vxg_profile(self._h, 1 if enable else 0))

    def stage_times(self, reset: bool = True) -> Dict[str, Tuple[float, int, int]]:
        n = lib().vxg_stage_count()
        ms = (ctypes.c_double * n)()
        la = (ctypes.c_uint64 * n)()
        un = (ctypes.c_uint64 * n)()
        check(lib().vxg_stage_times(self._h, ms, la, un, 1 if reset else 0))
        return {lib().vxg_stage_name(i).decode(): (ms[i], la[i], un[i]) for i in range(n)}

    def kernel_launches(self, reset: bool = True) -> int:
        n = ctypes.c_uint64()
        check(lib().vxg_kernel_launches(self._h, ctypes.byref(n), 1 if reset else 0))
        return int(n.value)

    def batch_info(self, reset: bool = True) -> Dict[str, int]:
        """records emitted, distinct voxels folded (N_vox), longest fold chain, blocks, record-sort passes."""
        out = (ctypes.c_uint64 * 5)()
        check(lib().vxg_batch_info(self._h, out, 1 if reset else 0))
        return {"records": int(out[0]), "n_vox": int(out[1]), "max_chain": int(out[2]), "blocks": int(out[3]),
                "sort_passes": int(out[4])}

    def shard_init(self, rank: int, world: int, nccl_id: bytes = b"", replicated: bool = False) -> None:
        """Makes this layer shard `rank` of `world` (one process per GPU, NCCL
        all-to-all of update records between shards).
        replicated=True: every rank walks all rays and keeps its own blocks'
        records (no record exchange). world=1 with an id runs the sharded path
        through a 1-rank NCCL communicator (self send/recv)."""
        if nccl_id:
            _nccl_preload()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id.ljust(128, b"\0")[:128]) if nccl_id else None
        check(lib().vxg_shard_init(self._h, int(rank), int(world), buf))
        check(lib().vxg_shard_set_replicated(self._h, 1 if replicated else 0))

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        check(lib().vxg_set_stream(self._h, ctypes.c_void_p(stream_ptr) if stream_ptr else None))


class TsdfIntegrator:
    """vxf::TsdfIntegrator (tsdf_integrator.h:75-112) on the B200 path."""

    def __init__(self, config: TsdfConfig, layer: TsdfLayer):
        config.validate()
        self._config = config
        self._layer = layer
        self._raycasts = 0
        self._skipped = 0

    def config(self) -> TsdfConfig:
        return self._config

    def raycasts_last_scan(self) -> int:
        return self._raycasts

    def skipped_points_last_scan(self) -> int:
        return self._skipped

    def _bind(self) -> None:
        c = self._config.to_c()
        check(lib().vxg_set_config(self._layer.handle, ctypes.byref(c)))

    def integrate(self, scan: Scan) -> int:
        """size_t integrate(const Scan&) (tsdf_integrator.cpp:111-127)."""
        if scan.colors is not None and len(scan.colors) != len(scan.points):
            raise ValueError("scan colors must parallel points")
        self._bind()
        st = VxgStats()
        pose = (ctypes.c_float * 12)(*scan.pose.tolist())
        check(lib().vxg_integrate(self._layer.handle, _ptr(scan.points), _ptr(scan.colors), len(scan.points), pose,
                                  ctypes.byref(st)))
        self._raycasts, self._skipped = int(st.raycasts), int(st.skipped)
        return int(st.updates)

    def integrate_batch(self, scans: Sequence[Scan]) -> np.ndarray:
        """Integrates scans in order (identical to sequential integrate calls);
        returns per-scan [updates, raycasts, skipped] as an (F, 3) uint64 array."""
        F = len(scans)
        for s in scans:
            if s.colors is not None and len(s.colors) != len(s.points):
                raise ValueError("scan colors must parallel points")
        self._bind()
        frames = (VxgFrame * max(F, 1))()
        for i, s in enumerate(scans):
            frames[i].xyz = s.points.ctypes.data
            frames[i].rgb = s.colors.ctypes.data if s.colors is not None else None
            frames[i].n = len(s.points)
            frames[i].pose[:] = s.pose.tolist()
        stats = (VxgStats * max(F, 1))()
        check(lib().vxg_integrate_batch(self._layer.handle, frames, F, VXG_INPUT_HOST, stats))
        out = np.array([[s.updates, s.raycasts, s.skipped] for s in stats[:F]], dtype=np.uint64).reshape(F, 3)
        if F:
            self._raycasts, self._skipped = int(out[-1, 1]), int(out[-1, 2])
        return out

    def integrate_packed(self, xyz_ptr: int, rgb_ptr: Optional[int], offsets: np.ndarray, poses: np.ndarray,
                         device_input: bool) -> np.ndarray:
        """Packed batch over raw pointers (device or pinned host memory)."""
        self._bind()
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        poses = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
        F = len(poses)
        stats = (VxgStats * max(F, 1))()
        check(lib().vxg_integrate_packed(
            self._layer.handle, ctypes.c_void_p(xyz_ptr), ctypes.c_void_p(rgb_ptr) if rgb_ptr else None,
            offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            poses.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), F,
            VXG_INPUT_DEVICE if device_input else VXG_INPUT_HOST, stats))
        out = np.array([[s.updates, s.raycasts, s.skipped] for s in stats[:F]], dtype=np.uint64).reshape(F, 3)
        if F:
            self._raycasts, self._skipped = int(out[-1, 1]), int(out[-1, 2])
        return out

    def stage_packed(self, xyz_ptr: int, rgb_ptr: Optional[int], offsets: np.ndarray) -> int:
        """Streaming ingestion: start the asynchronous H2D copy of a packed batch
        (pinned host pointers) into a staging slot; returns the slot id. The
        host buffers must stay valid until integrate_staged(slot) returns."""
        self._bind()
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        slot = ctypes.c_int()
        check(lib().vxg_stage_packed(
            self._layer.handle, ctypes.c_void_p(xyz_ptr), ctypes.c_void_p(rgb_ptr) if rgb_ptr else None,
            offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(offsets) - 1, ctypes.byref(slot)))
        return slot.value

    def integrate_staged(self, slot: int, poses: np.ndarray) -> np.ndarray:
        """Integrate a batch staged by stage_packed (same results as integrate_packed)."""
        self._bind()
        poses = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
        F = len(poses)
        stats = (VxgStats * max(F, 1))()
        check(lib().vxg_integrate_staged(self._layer.handle, int(slot),
                                         poses.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), stats))
        out = np.array([[s.updates, s.raycasts, s.skipped] for s in stats[:F]], dtype=np.uint64).reshape(F, 3)
        if F:
            self._raycasts, self._skipped = int(out[-1, 1]), int(out[-1, 2])
        return out



# ---------------------------------------------------------------- ESDF
ESDF_VOXEL_DTYPE = np.dtype([("distance", "<f4"), ("flags", "u1"), ("parent", "i1", (3,))])  # serialization.cpp:116-122


class FixedBandMode(enum.IntEnum):  # esdf_integrator.h:12-15
    kOneVoxel = 0
    kHalfTruncation = 1


class DistanceMetric(enum.IntEnum):  # esdf_integrator.h:17-20
    kQuasiEuclidean = 0
    kEuclidean = 1


class QueueMode(enum.IntEnum):  # esdf_integrator.h:22-26
    kFifo = 0
    kPrioritySingleInsert = 1
    kPriorityMultiInsert = 2


@dataclass
class EsdfConfig:  # esdf_integrator.h:28-41 (same defaults)
    d_max: float = 4.0
    band_mode: FixedBandMode = FixedBandMode.kOneVoxel
    truncation: float = 0.4
    metric: DistanceMetric = DistanceMetric.kQuasiEuclidean
    queue_mode: QueueMode = QueueMode.kPrioritySingleInsert
    bucket_width: float = 0.0

    def band_radius(self, voxel_size: float) -> float:
        return float(np.float32(voxel_size) if self.band_mode == FixedBandMode.kOneVoxel
                     else np.float32(0.5) * np.float32(self.truncation))

    def to_c(self) -> VxgEsdfConfig:
        return VxgEsdfConfig(self.d_max, int(self.band_mode), self.truncation, int(self.metric),
                             int(self.queue_mode), self.bucket_width)


class EsdfLayer:
    """An ESDF layer produced on the device (vxf::EsdfLayer, layer.h:167): the
    serialized VXBLX bytes (save_layer) plus a block view decoded from them."""

    def __init__(self, data: bytes):
        self._data = data
        self.voxel_size = float(np.float32(np.frombuffer(data[10:18], dtype="<f8")[0]))
        self.vps = int(np.frombuffer(data[18:22], dtype="<u4")[0])
        self._count = int(np.frombuffer(data[23:31], dtype="<u8")[0])
        self.rounds = 0

    def voxels_per_side(self) -> int:
        return self.vps

    def block_count(self) -> int:
        return self._count

    def save_bytes(self) -> bytes:
        return self._data

    def blocks(self) -> Dict[Tuple[int, int, int], np.ndarray]:
        nv = self.vps ** 3
        rec = np.dtype([("idx", "<i8", (3,)), ("vox", ESDF_VOXEL_DTYPE, (nv,))])
        arr = np.frombuffer(self._data, dtype=rec, count=self._count, offset=31)
        return {tuple(int(x) for x in r["idx"]): r["vox"] for r in arr}


class EsdfIntegrator:
    """vxf::EsdfIntegrator's batch entry points that run on the device."""

    @staticmethod
    def build_from_occupancy(tsdf: "TsdfLayer", config: EsdfConfig) -> EsdfLayer:
        """EsdfIntegrator::build_from_occupancy (esdf_integrator.cpp:303-330): every
        observed voxel with negative TSDF distance seeds at 0; distances lower
        outward (quasi-Euclidean). ValueError with the reference's validate()
        text; ValueError for the Euclidean metric (order-dependent, not offered)."""
        rounds = ctypes.c_uint64()
        check(lib().vxg_esdf_build_occupancy(tsdf.handle, ctypes.byref(config.to_c()), ctypes.byref(rounds)))
        need = ctypes.c_uint64()
        check(lib().vxg_esdf_serialize_vxblx(tsdf.handle, None, 0, ctypes.byref(need)))
        buf = np.zeros(need.value, dtype=np.uint8)
        check(lib().vxg_esdf_serialize_vxblx(tsdf.handle, _ptr(buf), need.value, ctypes.byref(need)))
        out = EsdfLayer(buf.tobytes())
        out.rounds = int(rounds.value)
        return out


@dataclass
class Mesh:
    """vxf::Mesh (mesh.h:13-33): triangle soup, 3 vertices per triangle in
    emission order, per-vertex normals and optional colours."""
    vertices: np.ndarray  # [V, 3] float32
    normals: np.ndarray   # [V, 3] float32
    colors: np.ndarray    # [V, 3] uint8 (empty without colours)
    triangles: np.ndarray  # [T, 3] uint32

    def empty(self) -> bool:
        return len(self.triangles) == 0

    def has_colors(self) -> bool:
        return len(self.colors) > 0


class MeshExtractor:
    """vxf::MeshExtractor (mesh_extractor.h:13-35) on the device slab:
    extract_blocks / extract_all replace the fragments of the blocks they
    touch; fragments() maps block index -> Mesh; combined() concatenates the
    fragments in (x, y, z) block order. The marching-cubes case tables are the
    caller's (the reference build's mc_tables), as a VxgMcTables."""

    def __init__(self, layer: TsdfLayer, tables, with_colors: bool = True):
        self._layer = layer
        self._tables = tables
        self._with_colors = bool(with_colors)
        self._fragments: Dict[Tuple[int, int, int], Mesh] = {}

    def _run(self, blocks: Optional[np.ndarray]) -> None:
        h = self._layer.handle
        nf, nt = ctypes.c_uint64(), ctypes.c_uint64()
        b = None if blocks is None else np.ascontiguousarray(blocks, dtype=np.int32).reshape(-1, 3)
        check(lib().vxg_mesh_extract(h, ctypes.byref(self._tables), None if b is None else b.ctypes.data,
                                     0 if b is None else len(b), int(self._with_colors), ctypes.byref(nf),
                                     ctypes.byref(nt)))
        B, T = nf.value, nt.value
        bidx = np.zeros((B, 3), np.int32)
        frag = np.zeros(B + 1, np.uint64)
        v = np.zeros((3 * T, 3), np.float32)
        n = np.zeros((3 * T, 3), np.float32)
        c = np.zeros((3 * T, 3), np.uint8) if self._with_colors else np.zeros((0, 3), np.uint8)
        check(lib().vxg_mesh_fetch(h, bidx.ctypes.data, frag.ctypes.data, v.ctypes.data, n.ctypes.data,
                                   c.ctypes.data if self._with_colors else None))
        for j in range(B):
            t0, t1 = int(frag[j]), int(frag[j + 1])
            k = t1 - t0
            tri = np.arange(3 * k, dtype=np.uint32).reshape(k, 3)
            self._fragments[tuple(int(x) for x in bidx[j])] = Mesh(
                v[3 * t0:3 * t1].copy(), n[3 * t0:3 * t1].copy(),
                c[3 * t0:3 * t1].copy() if self._with_colors else np.zeros((0, 3), np.uint8), tri)

    def extract_blocks(self, blocks) -> None:
        self._run(np.asarray(list(blocks), dtype=np.int32).reshape(-1, 3))

    def extract_all(self) -> None:
        self._run(None)

    def fragments(self) -> Dict[Tuple[int, int, int], Mesh]:
        return self._fragments

    def combined(self) -> Mesh:
        vs, ns, cs, ts = [], [], [], []
        base = 0
        for k in sorted(self._fragments):
            m = self._fragments[k]
            vs.append(m.vertices)
            ns.append(m.normals)
            cs.append(m.colors)
            ts.append(m.triangles + base)
            base += len(m.vertices)
        cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros((0, 3), dt)  # noqa: E731
        return Mesh(cat(vs, np.float32), cat(ns, np.float32),
                    cat(cs, np.uint8) if self._with_colors else np.zeros((0, 3), np.uint8), cat(ts, np.uint32))


def extract_mesh(layer: TsdfLayer, tables, with_colors: bool = True) -> Mesh:
    """One-shot extraction over the whole layer (mesh_extractor.cpp:153-157)."""
    ex = MeshExtractor(layer, tables, with_colors)
    ex.extract_all()
    return ex.combined()

def _check_io(rc: int) -> None:
    """Scan I/O errors are std::runtime_error in the reference (scan.cpp)."""
    if rc in (1,):  # VXG_EINVAL: bad arguments on our side
        check(rc)
    if rc != 0:
        raise RuntimeError(lib().vxg_last_error().decode())


def load_ply_points(path: str, device: Optional[int] = None) -> Scan:
    """vxf::load_ply_points (scan.cpp:70-180). A binary payload is decoded on the
    GPU. device=None: a Scan with numpy arrays in host memory (identity pose);
    device=k: (xyz, rgb-or-None) torch CUDA tensors on device k, ready for
    integrate_packed(..., device_input=True)."""
    n, hc = ctypes.c_uint64(), ctypes.c_int()
    bp = path.encode()
    _check_io(lib().vxg_ply_load(bp, 0 if device is None else device, None, None, 0, VXG_INPUT_HOST,
                                 ctypes.byref(n), ctypes.byref(hc)))
    N = n.value
    if device is None:
        xyz = np.zeros((N, 3), np.float32)
        rgb = np.zeros((N, 3), np.uint8) if hc.value else None
        _check_io(lib().vxg_ply_load(bp, 0, xyz.ctypes.data, None if rgb is None else rgb.ctypes.data, N,
                                     VXG_INPUT_HOST, ctypes.byref(n), ctypes.byref(hc)))
        return Scan(xyz, rgb)
    import torch
    xyz = torch.empty((N, 3), dtype=torch.float32, device=f"cuda:{device}")
    rgb = torch.empty((N, 3), dtype=torch.uint8, device=f"cuda:{device}") if hc.value else None
    _check_io(lib().vxg_ply_load(bp, device, xyz.data_ptr(), None if rgb is None else rgb.data_ptr(), N,
                                 VXG_INPUT_DEVICE, ctypes.byref(n), ctypes.byref(hc)))
    return xyz, rgb


@dataclass
class TimedPose:
    """vxf::TimedPose (scan.h:22-25)."""
    timestamp: float
    pose: np.ndarray  # 3x4 [R | t]


def load_tum_trajectory(path: str) -> list:
    """vxf::load_tum_trajectory (scan.cpp:182-211)."""
    n = ctypes.c_uint64()
    bp = path.encode()
    _check_io(lib().vxg_tum_load(bp, None, None, 0, ctypes.byref(n)))
    ts = np.zeros(n.value, np.float64)
    ps = np.zeros((n.value, 3, 4), np.float32)
    _check_io(lib().vxg_tum_load(bp, ts.ctypes.data, ps.ctypes.data, n.value, ctypes.byref(n)))
    return [TimedPose(float(ts[i]), ps[i]) for i in range(n.value)]


def save_ply_mesh(mesh: "Mesh", path: str) -> None:
    """vxf::save_ply_mesh (scan.cpp:213-240)."""
    v = np.ascontiguousarray(mesh.vertices, np.float32)
    nr = np.ascontiguousarray(mesh.normals, np.float32)
    c = np.ascontiguousarray(mesh.colors, np.uint8) if mesh.has_colors() else None
    t = np.ascontiguousarray(mesh.triangles, np.uint32)
    _check_io(lib().vxg_save_ply_mesh(path.encode(), v.ctypes.data, nr.ctypes.data,
                                      None if c is None else c.ctypes.data, len(v), t.ctypes.data, len(t)))

def _nccl_preload() -> None:
    """libvxg dlopens libnccl.so.2 by soname. Import torch first when it is
    installed, so that the soname resolves to torch's bundled NCCL (the one
    torch.distributed uses) instead of pinning an older system copy that
    libtorch_cuda could not load against afterwards."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for vxg_shard_init (rank 0 makes it, the caller broadcasts it)."""
    _nccl_preload()
    buf = (ctypes.c_uint8 * 128)()
    check(lib().vxg_nccl_unique_id(buf))
    return bytes(buf)


class ShardGroup:
    """`world` map shards on ONE device exchanging update records in-process
    (the sharded kernels with device-to-device copies in place of NVLink) —
    the single-GPU test vehicle of the multi-GPU path (vxg_group_*)."""

    def __init__(self, config: TsdfConfig, voxel_size: float, voxels_per_side: int = 16, world: int = 2,
                 device: int = 0, block_capacity: int = 0, replicated: bool = False):
        config.validate()
        self._voxel_size = float(np.float32(voxel_size))
        self._vps = int(voxels_per_side)
        self._g = ctypes.c_void_p()
        c = config.to_c()
        check(lib().vxg_group_create(ctypes.byref(c), self._voxel_size, self._vps, int(device), int(world),
                                     int(block_capacity), ctypes.byref(self._g)))
        check(lib().vxg_group_set_replicated(self._g, 1 if replicated else 0))
        self.world = int(world)

    def __del__(self):
        g = getattr(self, "_g", None)
        if g is not None and g.value:
            try:
                lib().vxg_group_destroy(g)
            except Exception:
                pass
            self._g = None

    def shard_block_counts(self):
        out = []
        for i in range(self.world):
            h = ctypes.c_void_p()
            check(lib().vxg_group_shard(self._g, i, ctypes.byref(h)))
            n = ctypes.c_uint64()
            check(lib().vxg_block_count(h, ctypes.byref(n)))
            out.append(int(n.value))
        return out

    def integrate_batch(self, scans: Sequence[Scan]) -> np.ndarray:
        F = len(scans)
        xyz = np.ascontiguousarray(np.concatenate([s.points for s in scans]) if F else np.zeros((0, 3), np.float32))
        has = all(s.colors is not None for s in scans)
        if not has and any(s.colors is not None for s in scans):
            raise ValueError("ShardGroup.integrate_batch needs colours on all scans or none")
        rgb = np.ascontiguousarray(np.concatenate([s.colors for s in scans])) if (has and F) else None
        offsets = np.zeros(F + 1, dtype=np.uint64)
        offsets[1:] = np.cumsum([len(s.points) for s in scans])
        poses = np.ascontiguousarray(np.stack([s.pose for s in scans]).astype(np.float32)) if F else np.zeros((0, 12), np.float32)
        stats = (VxgStats * max(F, 1))()
        check(lib().vxg_group_integrate_packed(self._g, _ptr(xyz), _ptr(rgb),
                                               offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                               poses.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), F,
                                               VXG_INPUT_HOST, stats))
        return np.array([[s.updates, s.raycasts, s.skipped] for s in stats[:F]], dtype=np.uint64).reshape(F, 3)

    def save_bytes(self) -> bytes:
        need = ctypes.c_uint64()
        check(lib().vxg_group_serialize_vxblx(self._g, None, 0, ctypes.byref(need)))
        buf = np.zeros(need.value, dtype=np.uint8)
        check(lib().vxg_group_serialize_vxblx(self._g, _ptr(buf), need.value, ctypes.byref(need)))
        return buf.tobytes()


# ---- the reference's public free functions, evaluated on the device (batched)
def projective_distance(x, p, s, device: int = 0) -> np.ndarray:
    """tsdf_integrator.cpp:22-27 for n (x, p, s) triples."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, 3)
    p = np.ascontiguousarray(p, dtype=np.float32).reshape(-1, 3)
    s = np.ascontiguousarray(s, dtype=np.float32).reshape(-1, 3)
    out = np.zeros(len(x), dtype=np.float32)
    check(lib().vxg_eval_projective_distance(device, _ptr(x), _ptr(p), _ptr(s), len(x), _ptr(out)))
    return out


def measurement_weight(mode: WeightMode, z, d, truncation: float, dropoff_epsilon: float,
                       device: int = 0) -> np.ndarray:
    """tsdf_integrator.cpp:29-44, elementwise."""
    z = np.ascontiguousarray(np.atleast_1d(z), dtype=np.float32)
    d = np.ascontiguousarray(np.broadcast_to(np.atleast_1d(d), z.shape), dtype=np.float32)
    out = np.zeros(len(z), dtype=np.float32)
    check(lib().vxg_eval_measurement_weight(device, int(mode), _ptr(z), _ptr(d), len(z), truncation,
                                            dropoff_epsilon, _ptr(out)))
    return out


def update_tsdf_voxels(voxels: np.ndarray, starts: np.ndarray, d, w, truncation: float, max_weight: float,
                       rgb: Optional[np.ndarray] = None, device: int = 0) -> np.ndarray:
    """update_tsdf_voxel (tsdf_integrator.cpp:46-67) folded sequentially per voxel:
    voxel i folds records starts[i]..starts[i+1] in order. Returns the new voxels."""
    v = np.ascontiguousarray(voxels.copy()).view(VOXEL_DTYPE).reshape(-1)
    starts = np.ascontiguousarray(starts, dtype=np.uint64)
    d = np.ascontiguousarray(d, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    rgb = None if rgb is None else np.ascontiguousarray(rgb, dtype=np.uint8).reshape(-1, 3)
    check(lib().vxg_eval_update_voxels(device, _ptr(v), len(v), _ptr(starts), _ptr(d), _ptr(w), _ptr(rgb),
                                       truncation, max_weight))
    return v


def raycast(start, end, voxel_size: float, device: int = 0):
    """RayCaster walks (tsdf_integrator.cpp:69-104) for n segments: list of (k,3) int32 arrays."""
    start = np.ascontiguousarray(start, dtype=np.float32).reshape(-1, 3)
    end = np.ascontiguousarray(end, dtype=np.float32).reshape(-1, 3)
    n = len(start)
    counts = np.zeros(max(n, 1), dtype=np.uint32)
    check(lib().vxg_eval_raycast(device, _ptr(start), _ptr(end), n, voxel_size, _ptr(counts), None, None))
    offsets = np.zeros(max(n, 1), dtype=np.uint64)
    if n > 1:
        offsets[1:n] = np.cumsum(counts[: n - 1], dtype=np.uint64)
    total = int(offsets[n - 1] + counts[n - 1]) if n else 0
    out = np.zeros((max(total, 1), 3), dtype=np.int32)
    check(lib().vxg_eval_raycast(device, _ptr(start), _ptr(end), n, voxel_size, _ptr(counts), _ptr(offsets),
                                 _ptr(out)))
    return [out[int(offsets[i]): int(offsets[i]) + int(counts[i])] for i in range(n)]


__all__ = ["WeightMode", "MergeMode", "TsdfConfig", "Scan", "TsdfLayer", "TsdfIntegrator", "ParseError",
           "ShardGroup", "nccl_unique_id",
           "projective_distance", "measurement_weight", "update_tsdf_voxels", "raycast", "VOXEL_DTYPE",
           "K_TSDF_OBSERVED_WEIGHT", "pose_3x4"]

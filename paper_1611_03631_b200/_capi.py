"""ctypes binding of the vxg C ABI (include/vxg.h) — the product's Python surface.

The shared library ``libvxg.so`` (CUDA kernels for sm_100a + C ABI) is built
in-tree by ``make lib`` (``__graft_entry__.build()``). There is deliberately no
CPU fallback: if the library is missing or no sm_100 device is present, every
call raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_uint8, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvxg.so")

VXG_OK, VXG_EINVAL, VXG_ENOMEM, VXG_ECUDA, VXG_ERANGE, VXG_EPARSE, VXG_EIO = range(7)
VXG_INPUT_HOST, VXG_INPUT_DEVICE = 0, 1


class VxgTsdfConfig(ctypes.Structure):
    _fields_ = [
        ("truncation", c_float),
        ("dropoff_epsilon", c_float),
        ("max_weight", c_float),
        ("weight_mode", c_int32),
        ("merge_mode", c_int32),
        ("min_ray_length", c_float),
        ("max_ray_length", c_float),
    ]


class VxgStats(ctypes.Structure):
    _fields_ = [("updates", c_uint64), ("raycasts", c_uint64), ("skipped", c_uint64)]


class VxgVoxel(ctypes.Structure):
    _fields_ = [("distance", c_float), ("weight", c_float), ("r", c_uint8), ("g", c_uint8), ("b", c_uint8),
                ("pad", c_uint8)]


class VxgFrame(ctypes.Structure):
    _fields_ = [("xyz", c_void_p), ("rgb", c_void_p), ("n", c_uint64), ("pose", c_float * 12)]


class VxgMcTables(ctypes.Structure):
    _fields_ = [("corner_offsets", (c_int32 * 3) * 8), ("edge_corners", (c_int32 * 2) * 12),
                ("edge_table", ctypes.c_uint16 * 256), ("tri_table", (ctypes.c_int8 * 16) * 256)]


class VxgEsdfConfig(ctypes.Structure):
    _fields_ = [("d_max", c_float), ("band_mode", c_int32), ("truncation", c_float), ("metric", c_int32),
                ("queue_mode", c_int32), ("bucket_width", c_float)]


# (name, restype, argtypes) for every symbol include/vxg.h declares.
SIGNATURES = [
    ("vxg_last_error", c_char_p, []),
    ("vxg_device_info", c_int, [c_int, c_char_p, ctypes.c_size_t]),
    ("vxg_create", c_int, [POINTER(VxgTsdfConfig), c_float, c_int, c_int, c_uint64, POINTER(c_void_p)]),
    ("vxg_destroy", c_int, [c_void_p]),
    ("vxg_get_config", c_int, [c_void_p, POINTER(VxgTsdfConfig)]),
    ("vxg_set_config", c_int, [c_void_p, POINTER(VxgTsdfConfig)]),
    ("vxg_set_stream", c_int, [c_void_p, c_void_p]),
    ("vxg_integrate", c_int, [c_void_p, c_void_p, c_void_p, c_uint64, POINTER(c_float), POINTER(VxgStats)]),
    ("vxg_integrate_batch", c_int, [c_void_p, POINTER(VxgFrame), c_uint64, c_int, POINTER(VxgStats)]),
    ("vxg_integrate_packed", c_int,
     [c_void_p, c_void_p, c_void_p, POINTER(c_uint64), POINTER(c_float), c_uint64, c_int, POINTER(VxgStats)]),
    ("vxg_stage_packed", c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_uint64), c_uint64, POINTER(c_int)]),
    ("vxg_integrate_staged", c_int, [c_void_p, c_int, POINTER(c_float), POINTER(VxgStats)]),
    ("vxg_mesh_extract", c_int,
     [c_void_p, POINTER(VxgMcTables), c_void_p, c_uint64, c_int, POINTER(c_uint64), POINTER(c_uint64)]),
    ("vxg_mesh_fetch", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("vxg_ply_load", c_int,
     [c_char_p, c_int, c_void_p, c_void_p, c_uint64, c_int, POINTER(c_uint64), POINTER(c_int)]),
    ("vxg_tum_load", c_int, [c_char_p, c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_save_ply_mesh", c_int, [c_char_p, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p, c_uint64]),
    ("vxg_block_count", c_int, [c_void_p, POINTER(c_uint64)]),
    ("vxg_export_blocks", c_int, [c_void_p, c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_import_blocks", c_int, [c_void_p, c_void_p, c_void_p, c_uint64]),
    ("vxg_fetch_blocks", c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]),
    ("vxg_query_voxels", c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]),
    ("vxg_interpolate_distance", c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_int]),
    ("vxg_surface_error", c_int, [c_void_p, c_void_p, c_uint64, c_float, c_void_p]),
    ("vxg_serialize_vxblx", c_int, [c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_esdf_build_occupancy", c_int, [c_void_p, POINTER(VxgEsdfConfig), POINTER(c_uint64)]),
    ("vxg_esdf_serialize_vxblx", c_int, [c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_save_vxblx", c_int, [c_void_p, c_char_p]),
    ("vxg_load_vxblx", c_int, [c_void_p, c_void_p, c_uint64]),
    ("vxg_reset", c_int, [c_void_p]),
    ("vxg_flush", c_int, [c_void_p]),
    ("vxg_register_consumer", c_int, [c_void_p, c_char_p]),
    ("vxg_drain_updated", c_int, [c_void_p, c_char_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_profile", c_int, [c_void_p, c_int]),
    ("vxg_stage_count", c_int, []),
    ("vxg_stage_name", c_char_p, [c_int]),
    ("vxg_stage_times", c_int, [c_void_p, POINTER(c_double), POINTER(c_uint64), POINTER(c_uint64), c_int]),
    ("vxg_batch_info", c_int, [c_void_p, POINTER(c_uint64), c_int]),
    ("vxg_kernel_launches", c_int, [c_void_p, POINTER(c_uint64), c_int]),
    ("vxg_nccl_unique_id", c_int, [c_void_p]),
    ("vxg_shard_init", c_int, [c_void_p, c_int, c_int, c_void_p]),
    ("vxg_shard_set_replicated", c_int, [c_void_p, c_int]),
    ("vxg_group_set_replicated", c_int, [c_void_p, c_int]),
    ("vxg_group_create", c_int, [POINTER(VxgTsdfConfig), c_float, c_int, c_int, c_int, c_uint64, POINTER(c_void_p)]),
    ("vxg_group_destroy", c_int, [c_void_p]),
    ("vxg_group_shard", c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    ("vxg_group_set_config", c_int, [c_void_p, POINTER(VxgTsdfConfig)]),
    ("vxg_group_integrate_packed", c_int,
     [c_void_p, c_void_p, c_void_p, POINTER(c_uint64), POINTER(c_float), c_uint64, c_int, POINTER(VxgStats)]),
    ("vxg_group_serialize_vxblx", c_int, [c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    ("vxg_selftest_fold", c_int, [c_int, c_uint64, c_uint64, c_uint32, c_uint64, POINTER(c_uint64)]),
    ("vxg_selftest_prims", c_int, [c_void_p, c_uint64, c_int, c_int, c_uint64, POINTER(c_uint64)]),
    ("vxg_debug_top_runs", c_int, [c_void_p, POINTER(c_uint32), POINTER(c_uint32), c_uint32]),
    ("vxg_eval_projective_distance", c_int, [c_int, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p]),
    ("vxg_eval_measurement_weight", c_int, [c_int, c_int, c_void_p, c_void_p, c_uint64, c_float, c_float, c_void_p]),
    ("vxg_eval_update_voxels", c_int,
     [c_int, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_float]),
    ("vxg_eval_raycast", c_int, [c_int, c_void_p, c_void_p, c_uint64, c_float, c_void_p, c_void_p, c_void_p]),
]

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libvxg.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first (`make lib` or __graft_entry__.build()); "
                "there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


class ParseError(RuntimeError):
    """vxf::ParseError (serialization.h:12-16): malformed VXBLX stream."""


def check(rc: int) -> None:
    if rc == VXG_OK:
        return
    msg = lib().vxg_last_error().decode()
    if rc == VXG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    if rc == VXG_EPARSE:
        raise ParseError(msg)
    if rc == VXG_ENOMEM:
        raise MemoryError(msg)
    if rc == VXG_ERANGE:
        raise OverflowError(msg)
    if rc == VXG_EIO:
        raise OSError(msg)
    raise RuntimeError(f"vxg error {rc}: {msg}")

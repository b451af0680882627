"""ctypes bindings for the CPU checker — TEST INFRASTRUCTURE ONLY.

* OracleLayer: oracle/liboracle.so, the restatement (oracle/vxf_oracle.cpp).
* RefLayer:    oracle/_ref/libvxfref.so, the UNMODIFIED reference sources
               compiled against oracle/eigen_shim (oracle/ref_capi.cpp).
Both expose integrate(points, colors, pose) -> (updates, raycasts, skipped) and
save_bytes() -> VXBLX bytes, so every parity test compares like with like.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_size_t, c_uint64, c_void_p

import numpy as np

from paper_1611_03631_b200._capi import VxgEsdfConfig, VxgMcTables, VxgStats, VxgTsdfConfig, VxgVoxel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libvxfref.so")
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "unit_tests_ref")

_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        L = ctypes.CDLL(ORACLE_SO)
        L.vxo_config_validate.argtypes = [POINTER(VxgTsdfConfig), c_char_p, c_size_t]
        L.vxo_layer_create.restype = c_void_p
        L.vxo_layer_create.argtypes = [c_float, c_int]
        L.vxo_layer_destroy.argtypes = [c_void_p]
        L.vxo_block_count.restype = c_size_t
        L.vxo_block_count.argtypes = [c_void_p]
        L.vxo_integrate.argtypes = [c_void_p, POINTER(VxgTsdfConfig), c_void_p, c_void_p, c_size_t,
                                    POINTER(c_float), POINTER(VxgStats)]
        L.vxo_export_blocks.restype = c_size_t
        L.vxo_export_blocks.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.vxo_voxel.argtypes = [c_void_p, c_int32, c_int32, c_int32, POINTER(VxgVoxel)]
        L.vxo_set_block.argtypes = [c_void_p, c_void_p, c_void_p]
        L.vxo_save_vxblx.restype = c_size_t
        L.vxo_save_vxblx.argtypes = [c_void_p, c_void_p, c_size_t]
        L.vxo_projective_distance.restype = c_float
        L.vxo_projective_distance.argtypes = [POINTER(c_float)] * 3
        L.vxo_measurement_weight.restype = c_float
        L.vxo_measurement_weight.argtypes = [c_int, c_float, c_float, c_float, c_float]
        L.vxo_update_voxel.argtypes = [POINTER(VxgVoxel), c_float, c_float, c_float, c_float, c_void_p]
        L.vxo_raycast.restype = c_size_t
        L.vxo_raycast.argtypes = [POINTER(c_float), POINTER(c_float), c_float, c_void_p, c_size_t]
        L.vxo_global_index.argtypes = [POINTER(c_float), c_float, c_void_p]
        L.vxo_index_hash.restype = c_uint64
        L.vxo_index_hash.argtypes = [c_int32, c_int32, c_int32]
        L.vxo_grouped_ray_order.restype = c_size_t
        L.vxo_grouped_ray_order.argtypes = [POINTER(VxgTsdfConfig), c_float, c_void_p, c_size_t, POINTER(c_float),
                                            c_void_p, c_size_t]
        L.vxo_interpolate.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]
        L.vxo_surface_error.argtypes = [c_void_p, c_void_p, c_size_t, c_float, c_void_p]
        L.vxo_mesh_extract.restype = c_size_t
        L.vxo_mesh_extract.argtypes = [c_void_p, POINTER(VxgMcTables), c_int, c_void_p, c_size_t] + [c_void_p] * 5 + \
            [c_size_t, c_size_t, POINTER(c_uint64)]
        L.vxo_esdf_occupancy.restype = c_size_t
        L.vxo_esdf_occupancy.argtypes = [c_void_p, POINTER(VxgEsdfConfig), c_void_p, c_size_t, c_char_p, c_size_t]
        L.vxo_bucket_schedule.restype = c_size_t
        L.vxo_bucket_schedule.argtypes = [c_size_t, c_size_t, c_void_p, c_size_t]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        L = ctypes.CDLL(REF_SO)
        L.vxr_last_error.restype = c_char_p
        L.vxr_create.restype = c_void_p
        L.vxr_create.argtypes = [POINTER(VxgTsdfConfig), c_float, c_int]
        L.vxr_destroy.argtypes = [c_void_p]
        L.vxr_integrate.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t, POINTER(c_float), POINTER(VxgStats)]
        L.vxr_block_count.restype = c_size_t
        L.vxr_block_count.argtypes = [c_void_p]
        L.vxr_save_vxblx.restype = c_size_t
        L.vxr_save_vxblx.argtypes = [c_void_p, c_void_p, c_size_t]
        L.vxr_config_validate.argtypes = [POINTER(VxgTsdfConfig), c_char_p, c_size_t]
        L.vxr_projective_distance.restype = c_float
        L.vxr_projective_distance.argtypes = [POINTER(c_float)] * 3
        L.vxr_measurement_weight.restype = c_float
        L.vxr_measurement_weight.argtypes = [c_int, c_float, c_float, c_float, c_float]
        L.vxr_update_voxel.argtypes = [POINTER(VxgVoxel), c_float, c_float, c_float, c_float, c_void_p]
        L.vxr_raycast.restype = c_size_t
        L.vxr_raycast.argtypes = [POINTER(c_float), POINTER(c_float), c_float, c_void_p, c_size_t]
        L.vxr_index_hash.restype = c_uint64
        L.vxr_index_hash.argtypes = [c_int32, c_int32, c_int32]
        L.vxr_interpolate.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]
        L.vxr_surface_error.argtypes = [c_void_p, c_void_p, c_size_t, c_float, c_void_p]
        L.vxr_set_block.argtypes = [c_void_p, c_void_p, c_void_p]
        L.vxr_mc_tables.argtypes = [POINTER(VxgMcTables)]
        L.vxr_load_ply.argtypes = [c_char_p, c_void_p, c_void_p, POINTER(c_uint64), POINTER(c_int)]
        L.vxr_load_tum.argtypes = [c_char_p, c_void_p, c_void_p, POINTER(c_uint64)]
        L.vxr_save_ply_mesh.argtypes = [c_char_p, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p, c_uint64]
        L.vxr_esdf_occupancy.restype = c_size_t
        L.vxr_esdf_occupancy.argtypes = [c_void_p, POINTER(VxgEsdfConfig), c_void_p, c_size_t]
        L.vxr_mesh_extract.restype = c_size_t
        L.vxr_mesh_extract.argtypes = [c_void_p, c_int, c_void_p, c_size_t] + [c_void_p] * 5 + \
            [c_size_t, c_size_t, POINTER(c_uint64)]
        L.vxr_last_integrate_seconds.restype = ctypes.c_double
        L.vxr_last_integrate_seconds.argtypes = []
        L.vxr_load_resave.restype = c_size_t
        L.vxr_load_resave.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t]
        _ref = L
    return _ref


def ref_load_resave(data: bytes) -> bytes:
    """vxf::load_tsdf_layer then vxf::save_layer (the reference's own code)."""
    L = ref_lib()
    n = L.vxr_load_resave(data, len(data), None, 0)
    if n == 0:
        raise ValueError(L.vxr_last_error().decode())
    buf = ctypes.create_string_buffer(n)
    L.vxr_load_resave(data, len(data), buf, n)
    return buf.raw


def _pose_arr(pose):
    p = np.ascontiguousarray(np.asarray(pose, dtype=np.float32).reshape(12))
    return p, p.ctypes.data_as(POINTER(c_float))


def _vp(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


class OracleLayer:
    def __init__(self, config, voxel_size: float, vps: int = 16):
        self.L = oracle_lib()
        self.cfg = config.to_c() if hasattr(config, "to_c") else config
        self.h = self.L.vxo_layer_create(voxel_size, vps)
        self.vps = vps
        assert self.h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.vxo_layer_destroy(self.h)
            self.h = None

    def integrate(self, points, colors=None, pose=None):
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        cols = None if colors is None else np.ascontiguousarray(colors, dtype=np.uint8).reshape(-1, 3)
        if pose is None:
            pose = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
        _keep, pp = _pose_arr(pose)
        st = VxgStats()
        rc = self.L.vxo_integrate(self.h, ctypes.byref(self.cfg), _vp(pts), _vp(cols), len(pts), pp,
                                  ctypes.byref(st))
        if rc != 0:
            raise ValueError("oracle rejected the config")
        return int(st.updates), int(st.raycasts), int(st.skipped)

    def interpolate_distance(self, points):
        return _interp(self.L.vxo_interpolate, self.h, points)

    def esdf_occupancy_bytes(self, esdf_config) -> bytes:
        """build_from_occupancy (restated) -> ESDF VXBLX bytes; ValueError(text) if invalid."""
        c = esdf_config.to_c() if hasattr(esdf_config, "to_c") else esdf_config
        err = ctypes.create_string_buffer(256)
        need = self.L.vxo_esdf_occupancy(self.h, ctypes.byref(c), None, 0, err, 256)
        if need == 0:
            raise ValueError(err.value.decode())
        buf = np.zeros(need, dtype=np.uint8)
        self.L.vxo_esdf_occupancy(self.h, ctypes.byref(c), _vp(buf), need, err, 256)
        return buf.tobytes()

    def surface_error(self, points, truncation):
        return _surface_error(self.L.vxo_surface_error, self.h, points, truncation)

    def block_count(self):
        return int(self.L.vxo_block_count(self.h))

    def save_bytes(self) -> bytes:
        need = self.L.vxo_save_vxblx(self.h, None, 0)
        buf = np.zeros(need, dtype=np.uint8)
        self.L.vxo_save_vxblx(self.h, _vp(buf), need)
        return buf.tobytes()

    def export_blocks(self):
        nb = self.block_count()
        idx = np.zeros((nb, 3), dtype=np.int32)
        from paper_1611_03631_b200.tsdf import VOXEL_DTYPE
        vox = np.zeros((nb, self.vps ** 3), dtype=VOXEL_DTYPE)
        self.L.vxo_export_blocks(self.h, _vp(idx), _vp(vox), nb)
        return idx, vox

    def set_block(self, idx, voxels):
        i = np.ascontiguousarray(idx, dtype=np.int32)
        v = np.ascontiguousarray(voxels)
        self.L.vxo_set_block(self.h, _vp(i), _vp(v))

    def mesh_fragments(self, tables, with_colors=True, blocks=None):
        b = None if blocks is None else np.ascontiguousarray(blocks, dtype=np.int32).reshape(-1, 3)
        return _mesh(lambda *a: self.L.vxo_mesh_extract(self.h, ctypes.byref(tables), int(with_colors), _vp(b),
                                                        0 if b is None else len(b), *a), with_colors)


def mc_tables() -> VxgMcTables:
    """The reference build's marching-cubes case tables (oracle/_ref)."""
    t = VxgMcTables()
    ref_lib().vxr_mc_tables(ctypes.byref(t))
    return t


def ref_load_ply(path):
    """(xyz, rgb or None) from the reference's load_ply_points, or raises RuntimeError(text)."""
    L = ref_lib()
    n, hc = c_uint64(), c_int()
    if L.vxr_load_ply(path.encode(), None, None, ctypes.byref(n), ctypes.byref(hc)):
        raise RuntimeError(L.vxr_last_error().decode())
    xyz = np.zeros((n.value, 3), np.float32)
    rgb = np.zeros((n.value, 3), np.uint8) if hc.value else None
    L.vxr_load_ply(path.encode(), _vp(xyz), _vp(rgb), ctypes.byref(n), ctypes.byref(hc))
    return xyz, rgb


def ref_load_tum(path):
    L = ref_lib()
    n = c_uint64()
    if L.vxr_load_tum(path.encode(), None, None, ctypes.byref(n)):
        raise RuntimeError(L.vxr_last_error().decode())
    ts = np.zeros(n.value, np.float64)
    ps = np.zeros((n.value, 3, 4), np.float32)
    L.vxr_load_tum(path.encode(), _vp(ts), _vp(ps), ctypes.byref(n))
    return ts, ps


def ref_save_ply_mesh(path, v, n, c, tri):
    L = ref_lib()
    v, n, tri = (np.ascontiguousarray(a) for a in (v, n, tri))
    c = None if c is None else np.ascontiguousarray(c)
    if L.vxr_save_ply_mesh(path.encode(), _vp(v), _vp(n), _vp(c), len(v), _vp(tri), len(tri)):
        raise RuntimeError(L.vxr_last_error().decode())


def _mesh(call, with_colors):
    """Run a two-call mesh extraction; returns {block: (verts[3T,3], normals, colors)}."""
    nt = c_uint64()
    nf = call(None, None, None, None, None, 0, 0, ctypes.byref(nt))
    T = nt.value
    bidx = np.zeros((nf, 3), np.int32)
    frag = np.zeros(nf + 1, np.uint64)
    v = np.zeros((3 * T, 3), np.float32)
    n = np.zeros((3 * T, 3), np.float32)
    c = np.zeros((3 * T, 3), np.uint8)
    r = call(_vp(bidx), _vp(frag), _vp(v), _vp(n), _vp(c) if with_colors else None, nf, T, ctypes.byref(nt))
    assert r == nf, "reference fragment triangles are not sequential"
    out = {}
    for j in range(nf):
        a, b = 3 * int(frag[j]), 3 * int(frag[j + 1])
        out[tuple(int(x) for x in bidx[j])] = (v[a:b], n[a:b], c[a:b] if with_colors else np.zeros((0, 3), np.uint8))
    return out


def _interp(fn, h, points):
    p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
    d = np.zeros(len(p), dtype=np.float32)
    f = np.zeros(len(p), dtype=np.uint8)
    fn(h, _vp(p), len(p), _vp(d), _vp(f))
    return d, f.astype(bool)


def _surface_error(fn, h, points, truncation):
    p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
    out = np.zeros(5, dtype=np.float64)
    fn(h, _vp(p), len(p), float(truncation), _vp(out))
    return {"rms": float(out[0]), "mean": float(out[1]), "max": float(out[2]), "count": int(out[3]),
            "unknown_fraction": float(out[4])}


class RefLayer:
    def __init__(self, config, voxel_size: float, vps: int = 16):
        self.L = ref_lib()
        self.cfg = config.to_c() if hasattr(config, "to_c") else config
        self.h = self.L.vxr_create(ctypes.byref(self.cfg), voxel_size, vps)
        if not self.h:
            raise ValueError(self.L.vxr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.vxr_destroy(self.h)
            self.h = None

    def integrate(self, points, colors=None, pose=None):
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        cols = None if colors is None else np.ascontiguousarray(colors, dtype=np.uint8).reshape(-1, 3)
        if pose is None:
            pose = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
        _keep, pp = _pose_arr(pose)
        st = VxgStats()
        rc = self.L.vxr_integrate(self.h, _vp(pts), _vp(cols), len(pts), pp, ctypes.byref(st))
        if rc != 0:
            raise ValueError(self.L.vxr_last_error().decode())
        return int(st.updates), int(st.raycasts), int(st.skipped)

    def last_integrate_seconds(self) -> float:
        """steady_clock time of the last integrate() alone (benchmark.cpp:93-95)."""
        return float(self.L.vxr_last_integrate_seconds())

    def esdf_occupancy_bytes(self, esdf_config) -> bytes:
        """The reference's EsdfIntegrator::build_from_occupancy -> save_layer bytes."""
        c = esdf_config.to_c() if hasattr(esdf_config, "to_c") else esdf_config
        need = self.L.vxr_esdf_occupancy(self.h, ctypes.byref(c), None, 0)
        if need == 0:
            raise ValueError(self.L.vxr_last_error().decode())
        buf = np.zeros(need, dtype=np.uint8)
        self.L.vxr_esdf_occupancy(self.h, ctypes.byref(c), _vp(buf), need)
        return buf.tobytes()

    def interpolate_distance(self, points):
        return _interp(self.L.vxr_interpolate, self.h, points)

    def surface_error(self, points, truncation):
        return _surface_error(self.L.vxr_surface_error, self.h, points, truncation)

    def block_count(self):
        return int(self.L.vxr_block_count(self.h))

    def set_block(self, idx, voxels):
        i = np.ascontiguousarray(idx, dtype=np.int32)
        v = np.ascontiguousarray(voxels)
        self.L.vxr_set_block(self.h, _vp(i), _vp(v))

    def mesh_fragments(self, with_colors=True, blocks=None):
        b = None if blocks is None else np.ascontiguousarray(blocks, dtype=np.int32).reshape(-1, 3)
        return _mesh(lambda *a: self.L.vxr_mesh_extract(self.h, int(with_colors), _vp(b),
                                                        0 if b is None else len(b), *a), with_colors)

    def save_bytes(self) -> bytes:
        need = self.L.vxr_save_vxblx(self.h, None, 0)
        buf = np.zeros(need, dtype=np.uint8)
        self.L.vxr_save_vxblx(self.h, _vp(buf), need)
        return buf.tobytes()


def parse_vxblx(data: bytes):
    """(voxel_size, vps, idx [B,3] int64, voxels [B, vps^3] VOXEL_DTYPE) from VXBLX bytes."""
    from paper_1611_03631_b200.tsdf import VOXEL_DTYPE
    assert data[:6] == b"VXBLX\0"
    vs = np.frombuffer(data[10:18], dtype="<f8")[0]
    vps = int(np.frombuffer(data[18:22], dtype="<u4")[0])
    nb = int(np.frombuffer(data[23:31], dtype="<u8")[0])
    nv = vps ** 3
    rec = np.dtype([("idx", "<i8", 3), ("vox", VOXEL_DTYPE, nv)])
    body = np.frombuffer(data[31:], dtype=rec, count=nb)
    return vs, vps, body["idx"].copy(), body["vox"].copy()

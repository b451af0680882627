"""Meshing on the device slab (vxg_mesh_extract) vs the CPU oracle and the
reference's own MeshExtractor (oracle/_ref), fragment by fragment, bitwise:
vertices, per-vertex normals (central differences of interpolate_distance)
and colours."""
import numpy as np
import pytest

from mesh_helpers import random_layer, sphere_layer
from oracle_bindings import OracleLayer, RefLayer, mc_tables, ref_available
from paper_1611_03631_b200 import MeshExtractor, Scan, TsdfConfig, TsdfIntegrator, TsdfLayer, extract_mesh
from paper_1611_03631_b200 import workload as W

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def _gpu_frags(layer, with_colors=True, blocks=None):
    ex = MeshExtractor(layer, mc_tables(), with_colors)
    if blocks is None:
        ex.extract_all()
    else:
        ex.extract_blocks(blocks)
    return {k: (m.vertices, m.normals, m.colors) for k, m in ex.fragments().items()}


def _same(a, b):
    assert a.keys() == b.keys()
    for k in a:
        for x, y, what in zip(a[k], b[k], ("vertices", "normals", "colors")):
            assert x.shape == y.shape, (k, what, x.shape, y.shape)
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), (k, what)


def _layers(v, vps, blocks):
    cfg = TsdfConfig.for_voxel_size(v)
    g = TsdfLayer(v, vps)
    idx, vox = blocks
    g.import_blocks(idx, vox)
    o = OracleLayer(cfg, v, vps)
    for i in range(len(idx)):
        o.set_block(idx[i], vox[i])
    return g, o


def test_sphere_field(gpu):
    g, o = _layers(0.05, 8, sphere_layer())
    a = _gpu_frags(g)
    assert sum(len(f[0]) for f in a.values()) > 300
    _same(a, o.mesh_fragments(mc_tables()))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("with_colors", [True, False])
def test_random_fields_with_holes(gpu, seed, with_colors):
    g, o = _layers(0.1, 8, random_layer(seed))
    a = _gpu_frags(g, with_colors)
    assert sum(len(f[0]) for f in a.values()) > 1000
    _same(a, o.mesh_fragments(mc_tables(), with_colors))
    req = np.array([[0, 0, 0], [-1, 0, -1], [1, 1, 0], [50, 50, 50], [0, 0, 0]], np.int32)
    _same(_gpu_frags(g, with_colors, req), o.mesh_fragments(mc_tables(), with_colors, blocks=req))


def test_integrated_cfg1_frames_vs_reference(gpu):
    """Ten full-size merged cfg1 frames integrated on the GPU, meshed on the GPU;
    the reference integrates and meshes the same frames on the CPU."""
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    layer = TsdfLayer(wc.voxel_size, wc.vps)
    integ = TsdfIntegrator(cfg, layer)
    ref = RefLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in W.frames(1, count=10, start=0):
        assert integ.integrate(Scan(x, c, p)) == ref.integrate(x, c, p)[0]
    a = _gpu_frags(layer)
    assert sum(len(f[0]) for f in a.values()) > 10000
    _same(a, ref.mesh_fragments())


def test_reextraction_replaces_fragments_and_empty_field(gpu):
    g, _ = _layers(0.05, 8, sphere_layer())
    ex = MeshExtractor(g, mc_tables())
    ex.extract_all()
    once = len(ex.combined().triangles)
    idx, _ = g.export_blocks()
    ex.extract_blocks(idx)
    assert len(ex.combined().triangles) == once
    # uniform positive field -> empty mesh (test_mesh_extractor.cpp:49-61)
    e = TsdfLayer(0.1, 8)
    idx = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 1]], np.int32)
    from paper_1611_03631_b200 import VOXEL_DTYPE
    vox = np.zeros((3, 512), VOXEL_DTYPE)
    vox["distance"] = 0.7
    vox["weight"] = 1.0
    e.import_blocks(idx, vox)
    assert extract_mesh(e, mc_tables()).empty()

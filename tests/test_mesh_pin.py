"""Meshing oracle pinned to the reference (CPU): the restatement's marching
cubes (oracle/vxf_oracle.cpp vxo_mesh_extract) against the UNMODIFIED
mesh_extractor.cpp compiled in oracle/_ref, fragment by fragment, bitwise —
vertices, normals, colours — on integrated scans, analytic fields and random
fields with holes, extract_all and extract_blocks."""
import numpy as np
import pytest

from oracle_bindings import OracleLayer, RefLayer, mc_tables, ref_available
from mesh_helpers import random_layer, sphere_layer
from paper_1611_03631_b200 import TsdfConfig
from paper_1611_03631_b200 import workload as W

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _same(a, b):
    assert a.keys() == b.keys()
    for k in a:
        for x, y, what in zip(a[k], b[k], ("vertices", "normals", "colors")):
            assert x.shape == y.shape, (k, what, x.shape, y.shape)
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), (k, what)


def _pair(v, vps, blocks):
    cfg = TsdfConfig.for_voxel_size(v)
    o, r = OracleLayer(cfg, v, vps), RefLayer(cfg, v, vps)
    idx, vox = blocks
    for i in range(len(idx)):
        o.set_block(idx[i], vox[i])
        r.set_block(idx[i], vox[i])
    return o, r


@pytest.mark.parametrize("with_colors", [True, False])
def test_integrated_scans(with_colors):
    wc = W.CONFIGS[1]
    cfg = W.tsdf_config(wc)
    o, r = OracleLayer(cfg, wc.voxel_size, wc.vps), RefLayer(cfg, wc.voxel_size, wc.vps)
    for x, c, p in W.frames(1, count=2, scale=0.3, start=3):
        assert o.integrate(x, c, p) == r.integrate(x, c, p)
    t = mc_tables()
    a, b = o.mesh_fragments(t, with_colors), r.mesh_fragments(with_colors)
    assert sum(len(f[0]) for f in a.values()) > 300
    _same(a, b)


def test_sphere_field():
    o, r = _pair(0.05, 8, sphere_layer())
    a, b = o.mesh_fragments(mc_tables()), r.mesh_fragments()
    assert sum(len(f[0]) for f in a.values()) > 300
    _same(a, b)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_fields_with_holes(seed):
    o, r = _pair(0.1, 8, random_layer(seed))
    t = mc_tables()
    _same(o.mesh_fragments(t), r.mesh_fragments())
    req = np.array([[0, 0, 0], [-1, 0, -1], [1, 1, 0], [50, 50, 50], [0, 0, 0]], np.int32)  # absent + duplicate
    _same(o.mesh_fragments(t, blocks=req), r.mesh_fragments(blocks=req))

"""Meshing (MeshExtractor::extract_all, mesh_extractor.cpp:48-52) on the device
slab vs the reference's own MeshExtractor (oracle/_ref, 1 thread) on the SAME
layer: the map after integrating the 100-frame cfg1 trajectory. Prints one JSON
line. GPU time = vxg_mesh_extract (count, scan, emit; the layer is resident)
plus vxg_mesh_fetch (D2H of the mesh), wall clock around the synchronous calls,
median of 10 after 2 warm-ups."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bindings import RefLayer, mc_tables  # noqa: E402  (checker / CPU baseline only)
from paper_1611_03631_b200 import MeshExtractor, TsdfIntegrator, TsdfLayer  # noqa: E402
from paper_1611_03631_b200 import workload as W  # noqa: E402

wc = W.CONFIGS[1]
cfg = W.tsdf_config(wc)
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1024)
integ = TsdfIntegrator(cfg, layer)
dx, dc = torch.from_numpy(xyz).cuda(), torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
torch.cuda.synchronize()
tables = mc_tables()
times = []
for i in range(12):
    ex = MeshExtractor(layer, tables, True)
    t0 = time.perf_counter()
    ex.extract_all()
    times.append(time.perf_counter() - t0)
gpu_s = statistics.median(times[2:])
frags = ex.fragments()
T = sum(len(m.triangles) for m in frags.values())
# the reference on the same layer content
idx, vox = layer.export_blocks()
ref = RefLayer(cfg, wc.voxel_size, wc.vps)
for i in range(len(idx)):
    ref.set_block(idx[i], vox[i])
t0 = time.perf_counter()
rf = ref.mesh_fragments(True)
cpu_s = time.perf_counter() - t0
same = rf.keys() == frags.keys() and all(
    np.array_equal(rf[k][0].view(np.uint32), frags[k].vertices.view(np.uint32)) and
    np.array_equal(rf[k][1].view(np.uint32), frags[k].normals.view(np.uint32)) and
    np.array_equal(rf[k][2], frags[k].colors) for k in frags)
cubes = len(idx) * wc.vps ** 3
print(json.dumps({"metric": "mesh_extract_all", "workload": "cfg1 map after 100 frames", "blocks": int(len(idx)),
                  "cubes": cubes, "triangles": int(T), "gpu_ms": gpu_s * 1e3, "gpu_cubes_per_s": cubes / gpu_s,
                  "cpu_reference_ms": cpu_s * 1e3, "cpu_cores": 1, "speedup": cpu_s / gpu_s,
                  "bit_exact_vs_reference": bool(same)}))

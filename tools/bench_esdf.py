"""ESDF occupancy baseline (EsdfIntegrator::build_from_occupancy,
esdf_integrator.cpp:303-330) on the device slab vs the reference's own
EsdfIntegrator (oracle/_ref, 1 thread) on the SAME layer: the map after
integrating the 100-frame cfg1 trajectory, d_max 4 m, quasi-Euclidean,
priority single-insert queue (the reference defaults). Prints one JSON line.
GPU time = vxg_esdf_build_occupancy (neighbour table, seeding, relaxation
rounds, parents; the layer is resident), wall clock around the synchronous
call, median of 10 after 2 warm-ups; plus the full Python call (build + D2H
serialisation)."""
import ctypes
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from esdf_helpers import same_distances_and_flags  # noqa: E402
from oracle_bindings import RefLayer  # noqa: E402  (checker / CPU baseline only)
from paper_1611_03631_b200 import EsdfConfig, EsdfIntegrator, TsdfIntegrator, TsdfLayer  # noqa: E402
from paper_1611_03631_b200 import _capi  # noqa: E402
from paper_1611_03631_b200 import workload as W  # noqa: E402

wc = W.CONFIGS[1]
cfg = W.tsdf_config(wc)
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1024)
integ = TsdfIntegrator(cfg, layer)
dx, dc = torch.from_numpy(xyz).cuda(), torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
torch.cuda.synchronize()
ec = EsdfConfig(d_max=4.0, truncation=wc.truncation)
c = ec.to_c()
rounds = ctypes.c_uint64()
times = []
for i in range(12):
    t0 = time.perf_counter()
    _capi.check(_capi.lib().vxg_esdf_build_occupancy(layer.handle, ctypes.byref(c), ctypes.byref(rounds)))
    times.append(time.perf_counter() - t0)
gpu_s = statistics.median(times[2:])
t0 = time.perf_counter()
g = EsdfIntegrator.build_from_occupancy(layer, ec).save_bytes()
full_s = time.perf_counter() - t0
idx, vox = layer.export_blocks()
ref = RefLayer(cfg, wc.voxel_size, wc.vps)
for i in range(len(idx)):
    ref.set_block(idx[i], vox[i])
t0 = time.perf_counter()
r = ref.esdf_occupancy_bytes(ec)
cpu_s = time.perf_counter() - t0
try:
    same_distances_and_flags(g, r)
    same = True
except AssertionError:
    same = False
voxels = len(idx) * wc.vps ** 3
print(json.dumps({"metric": "esdf_build_from_occupancy", "workload": "cfg1 map after 100 frames, d_max 4",
                  "blocks": int(len(idx)), "voxels": voxels, "relax_rounds": int(rounds.value),
                  "gpu_ms": gpu_s * 1e3, "gpu_ms_with_serialize": full_s * 1e3,
                  "gpu_voxels_per_s": voxels / gpu_s, "cpu_reference_ms": cpu_s * 1e3, "cpu_cores": 1,
                  "speedup": cpu_s / gpu_s, "bit_exact_distances_flags_vs_reference": same}))

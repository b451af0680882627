"""Dev probe: host-clock latency of one F=1 integrate call (+flush) of a config, fresh layer each time."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prof = len(sys.argv) <= 3 or sys.argv[3] != 'noprof'
wc = W.CONFIGS[cfg]
xyz, rgb, off, poses = W.pack(W.frames(cfg, count=1))
layer = TsdfLayer(wc.voxel_size, wc.vps, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
hx = torch.from_numpy(xyz).pin_memory(); hc = torch.from_numpy(rgb).pin_memory() if rgb is not None else None
o = np.array([off[0], off[1]], dtype=np.uint64)
for r in range(reps):
    layer.reset(); layer.flush(); torch.cuda.synchronize()
    if prof:
        layer.profile(True); layer.stage_times(True)
    t = time.perf_counter()
    st = integ.integrate_packed(hx.data_ptr(), hc.data_ptr() if hc is not None else None, o, poses[0:1], False)
    layer.flush(); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f'rep {r}: {1e3*dt:.3f} ms updates {int(st[0,0])}', {k: round(v[0], 3) for k, v in layer.stage_times(True).items()} if prof else '')
    layer.profile(False)

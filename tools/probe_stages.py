"""Dev probe: per-stage ms / launches / units of one device-resident cfg1 step."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
layer.reset()
layer.profile(True); layer.stage_times(True); layer.batch_info(True)
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
torch.cuda.synchronize()
for k, v in layer.stage_times(True).items():
    print(f"{k:12s} {v[0]:8.3f} ms  launches {v[1]:4d}  units {v[2]}")
print(layer.batch_info(True))
print("config", W.tsdf_config(wc))

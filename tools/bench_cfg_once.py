"""Dev probe: one device-resident batch of a config (for ncu captures): cfg, frames, reps."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
cfg = int(sys.argv[1]); n = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wc = W.CONFIGS[cfg]
xyz, rgb, off, poses = W.pack(W.frames(cfg, count=n))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=16384)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda() if rgb is not None else None
for _ in range(reps):
    layer.reset()
    integ.integrate_packed(dx.data_ptr(), dc.data_ptr() if dc is not None else None, off, poses, True)
torch.cuda.synchronize()
print(layer.batch_info())

"""Dev probe: one device-resident cfg1 step (for ncu launch lists / captures)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=n))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda()
for _ in range(reps):
    layer.reset()
    integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
torch.cuda.synchronize()
print(layer.batch_info())

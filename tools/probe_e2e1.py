"""Dev probe: one host-input integrate_packed (VXG_H2D_PARTS) for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
hx = torch.from_numpy(xyz).pin_memory(); hc = torch.from_numpy(rgb).pin_memory()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    layer.reset(); integ.integrate_packed(hx.data_ptr(), hc.data_ptr(), off, poses, False)
torch.cuda.synchronize()

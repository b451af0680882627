import ctypes, sys, numpy as np, time
sys.path.insert(0, '.')
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from paper_1611_03631_b200._capi import lib
wc = W.CONFIGS[1]
fr = W.frames(1, count=100)
xyz, rgb, off, poses = W.pack(fr)
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
import torch
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
print(layer.batch_info())
n = 40
L = (ctypes.c_uint32 * n)(); K = (ctypes.c_uint32 * n)()
lib().vxg_debug_top_runs(layer.handle, L, K, n)
idx, vox = layer.export_blocks()
# map keys: slot -> need block index: use query by exporting... print raw
print('top run lengths', list(L)[:40])
print('top keys', list(K)[:10])
# run length of per-frame sensor voxel for comparison
for name in ['rays/frame']:
    pass

"""Dev probe: fold-chain (run length) distribution of one batch of a config."""
import ctypes, sys, numpy as np
sys.path.insert(0, '.')
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from paper_1611_03631_b200._capi import lib
import torch
cfg = int(sys.argv[1]); nf = int(sys.argv[2])
wc = W.CONFIGS[cfg]
xyz, rgb, off, poses = W.pack(W.frames(cfg, count=nf))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=16384)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda() if rgb is not None else None
integ.integrate_packed(dx.data_ptr(), dc.data_ptr() if dc is not None else None, off, poses, True)
info = layer.batch_info()
print(info)
n = info['n_vox'] + 1
L = (ctypes.c_uint32 * n)(); K = (ctypes.c_uint32 * n)()
lib().vxg_debug_top_runs(layer.handle, L, K, n)
l = np.array(L, dtype=np.int64); k = np.array(K, dtype=np.int64)
l = l[k != 0xFFFFFFFF]
tot = l.sum()
print('runs', len(l), 'records', tot, 'mean', tot / len(l))
for t in [64, 256, 1024, 4096, 16384, 65536, 262144]:
    m = l >= t
    print(f'len>={t:7d}: runs {m.sum():9d} records {l[m].sum():12d} ({100*l[m].sum()/tot:5.1f}%)')

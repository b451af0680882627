"""Dev probe: fold-chain (run length) distribution of the cfg1 100-frame batch."""
import ctypes, sys, numpy as np
sys.path.insert(0, '.')
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from paper_1611_03631_b200._capi import lib
import torch
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
info = layer.batch_info()
print(info)
if len(sys.argv) > 1:
    n = info['n_vox'] + 1
    L = (ctypes.c_uint32 * n)(); K = (ctypes.c_uint32 * n)()
    lib().vxg_debug_top_runs(layer.handle, L, K, n)
    l = np.array(L, dtype=np.int64); k = np.array(K, dtype=np.int64)
    l = l[k != 0xFFFFFFFF]
    tot = l.sum()
    print('runs', len(l), 'records', tot, 'mean', tot / len(l))
    for t in [64, 256, 1024, 2048, 4096, 8192, 16384, 32768]:
        m = l >= t
        print(f'len>={t:6d}: runs {m.sum():7d} records {l[m].sum():11d} ({100*l[m].sum()/tot:5.1f}%)')
    print('quantiles', np.percentile(l, [50, 90, 99, 99.9]))

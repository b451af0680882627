"""Dev probe: globaltimer trace of the fold kernel on the cfg1 100-frame batch."""
import ctypes, sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
from paper_1611_03631_b200._capi import lib
L = lib()
L.vxg_debug_fold.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
dx = torch.from_numpy(xyz).cuda(); dc = torch.from_numpy(rgb).cuda()
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
layer.reset()
L.vxg_debug_fold(layer.handle, 1, None, 0, None)
layer.profile(True); layer.stage_times(True)
integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
print('apply ms', layer.stage_times(True)['apply'][0])
n = ctypes.c_uint64()
L.vxg_debug_fold(layer.handle, 0, None, 0, ctypes.byref(n))
buf = np.zeros(4 * n.value + 20, np.uint64)
L.vxg_debug_fold(layer.handle, 0, buf.ctypes.data, len(buf), ctypes.byref(n))
d = buf[:4 * n.value].reshape(-1, 4).astype(np.int64)
spec = d[:, 3] >> 32
nfail = (d[:, 2] >> 32) & 0xFFFF
nskip = (d[:, 2] >> 48) & 0xFFFF
d[:, 2] &= 0xFFFFFFFF
d[:, 3] &= 0xFFFFFFFF
cw, cb, pw, pb, pwe, psc, cvo, cch = [int(x) for x in buf[4 * n.value + 2:4 * n.value + 10]]
csp, nsp, cse, nse = [int(x) for x in buf[4 * n.value + 10:4 * n.value + 14]]
print(f'spec chunks {nsp} at {csp/max(nsp,1):.0f} cycles; other chunks {nse} at {cse/max(nse,1):.0f} cycles')
nrec = int(d[d[:, 1] > 0][:, 2].sum())
ptop, ppre, pstore = [int(x) for x in buf[4 * n.value + 14:4 * n.value + 17]]
print(f'producer per record: top {ptop/nrec:.1f} prerec {ppre/nrec:.1f} store {pstore/nrec:.1f}')
print(f'per record (cycles, summed over pairs): consumer busy {cb/nrec:.1f} wait {cw/nrec:.1f} vote {cvo/nrec:.1f} chain {cch/nrec:.1f}; producer busy {pb/nrec:.1f} wait {pw/nrec:.1f} weigh {pwe/nrec:.1f} scan {psc/nrec:.1f}')
print(f'consumer wait {cw / max(cb, 1):.3f} of busy; producer wait {pw / max(pb, 1):.3f} of busy')
long_ = d[d[:, 1] > 0]
t0 = long_[:, 0].min()
print('long runs', len(long_), 'first start', 0, 'last long end (us)', (long_[:, 1].max() - t0) / 1e3)

dur = (long_[:, 1] - long_[:, 0])
for i in np.argsort(-long_[:, 2])[:8]:
    print(f'len {long_[i,2]:6d} sat {long_[i,3]:6d} spec {spec[d[:, 1] > 0][i]:6d} failchunks {nfail[d[:, 1] > 0][i]:4d} skipchunks {nskip[d[:, 1] > 0][i]:4d} start {(long_[i,0]-t0)/1e3:8.1f}us dur {dur[i]/1e3:8.1f}us  ns/step {dur[i]/long_[i,2]:.1f}')
print('median ns/step over long runs', np.median(dur / long_[:, 2]), 'sat fraction', long_[:, 3].sum() / long_[:, 2].sum(), 'spec fraction', spec[d[:, 1] > 0].sum() / long_[:, 2].sum())

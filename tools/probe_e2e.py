"""Dev probe: host-input integrate_packed timing (VXG_H2D_PARTS), stage times."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
hx = torch.from_numpy(xyz).pin_memory(); hc = torch.from_numpy(rgb).pin_memory()
for _ in range(3):
    layer.reset(); integ.integrate_packed(hx.data_ptr(), hc.data_ptr(), off, poses, False)
torch.cuda.synchronize()
layer.profile(True); layer.stage_times(True)
ts = []
for _ in range(3):
    t = time.perf_counter()
    layer.reset(); integ.integrate_packed(hx.data_ptr(), hc.data_ptr(), off, poses, False)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
st = layer.stage_times(True)
print("wall ms", [round(x, 2) for x in ts], "stages", {k: round(v[0] / 3, 3) for k, v in st.items()})

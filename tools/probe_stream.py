"""Dev probe: marginal per-step cost of the streamed e2e path (stage_packed +
integrate_staged) vs the device-resident path, K = 10 and 30 steps."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
wc = W.CONFIGS[1]
xyz, rgb, off, poses = W.pack(W.frames(1, count=100))
stream = torch.cuda.current_stream()
layer = TsdfLayer(wc.voxel_size, 16, block_capacity=1024)
layer.set_stream(stream.cuda_stream)
integ = TsdfIntegrator(W.tsdf_config(wc), layer)
hx = torch.from_numpy(xyz).pin_memory(); hc = torch.from_numpy(rgb).pin_memory()
dx = hx.cuda(); dc = hc.cuda()

def streamed(K):
    slot = integ.stage_packed(hx.data_ptr(), hc.data_ptr(), off)
    for k in range(K):
        layer.reset()
        nxt = integ.stage_packed(hx.data_ptr(), hc.data_ptr(), off) if k + 1 < K else None
        integ.integrate_staged(slot, poses)
        slot = nxt

def device(K):
    for k in range(K):
        layer.reset()
        integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)

def device_with_copy(K):
    side = torch.cuda.Stream()
    buf = torch.empty_like(hx, device='cuda'); bufc = torch.empty_like(hc, device='cuda')
    for k in range(K):
        with torch.cuda.stream(side):
            buf.copy_(hx, non_blocking=True); bufc.copy_(hc, non_blocking=True)
        layer.reset()
        integ.integrate_packed(dx.data_ptr(), dc.data_ptr(), off, poses, True)
    torch.cuda.synchronize()

def t(fn, K):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); fn(K); layer.flush(); e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1)

for fn in (device, streamed, device_with_copy):
    fn(3)
    a, b = t(fn, 10), t(fn, 30)
    print(f"{fn.__name__:18s} K=10 {a/10:.3f} ms/step  K=30 {b/30:.3f} ms/step  marginal {(b-a)/20:.3f}", flush=True)

"""Dev probe: pinned H2D bandwidth of a 460 MB buffer, 10 copies, with the
process on all CPUs and on the GPU's local CPUs (NUMA)."""
import os, sys, time
import torch

def local_cpus(dev=0):
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    return bus

def run(tag):
    n = 460_805_608
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(tag, "ms", [round(t, 2) for t in ts], "GB/s median", round(n / sorted(ts)[5] / 1e6, 1), flush=True)

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
p = torch.cuda.get_device_properties(0)
print("props", [a for a in dir(p) if "pci" in a.lower() or "bus" in a.lower()])
os.system("nvidia-smi topo -m | head -5; ls /sys/bus/pci/devices | head -3; lscpu | grep -i numa")
run("all-cpus")

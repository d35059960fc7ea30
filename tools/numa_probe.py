"""H2D bandwidth from pinned host memory with the process bound to each NUMA
node's CPUs (is the GPU-local node faster?)."""
import glob
import os
import sys

import numpy as np
import torch

def node_cpus():
    out = {}
    for d in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        with open(os.path.join(d, "cpulist")) as f:
            spec = f.read().strip()
        cpus = []
        for part in spec.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus += list(range(int(a), int(b) + 1))
            elif part:
                cpus.append(int(part))
        out[int(d.split("node")[-1])] = cpus
    return out

dev = torch.device("cuda", 0)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("nodes:", {k: (min(v), max(v), len(v)) for k, v in node_cpus().items()})
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    pci = pynvml.nvmlDeviceGetPciInfo(h).busId
    pci = pci.decode() if isinstance(pci, bytes) else pci
    path = f"/sys/bus/pci/devices/{pci.lower()[4:] if len(pci) > 12 else pci.lower()}"
    print("gpu pci", pci, "numa_node:", open(os.path.join(path, "numa_node")).read().strip() if os.path.exists(path) else "?")
    aff = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
    cpus = [i for i in range(os.cpu_count()) if (aff[i // 64] >> (i % 64)) & 1]
    print("nvml cpu affinity:", cpus[:8], "...", len(cpus))
except Exception as e:
    print("nvml:", e)
a = np.random.default_rng(0).normal(size=(262144 * 3 * 4,))
for node, cpus in node_cpus().items():
    os.sched_setaffinity(0, cpus)
    t = torch.from_numpy(a.copy()).pin_memory()
    for _ in range(2):
        d = t.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d = t.to(dev, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"bound to node {node}: H2D {t.numel() * 8 / ms / 1e6:.1f} GB/s")

"""Round 2: D2H bandwidth into pinned host buffers allocated while the
allocating thread runs on each NUMA node (first-touch placement), against
the GPU's local node (sysfs local_cpulist of its PCI device)."""
import glob
import json
import os
import time

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
node_cpus = {os.path.basename(n): cpulist(open(n + "/cpulist").read()) for n in nodes}
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
try:
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
except Exception as e:  # noqa: BLE001
    print("nvml", e)
gpu_node = None
if bus:
    p = "/sys/bus/pci/devices/" + bus.lower()[-12:]
    for cand in (p, "/sys/bus/pci/devices/" + bus.lower()):
        if os.path.exists(cand + "/numa_node"):
            gpu_node = int(open(cand + "/numa_node").read())
            break
print(json.dumps({"nodes": {k: (v[0], v[-1], len(v)) for k, v in node_cpus.items()}, "gpu_bus": bus,
                  "gpu_numa_node": gpu_node, "cpus": os.cpu_count()}), flush=True)
N = 4 << 30
dev = torch.empty(N // 8, dtype=torch.int64, device="cuda")
dev.fill_(1)
orig = os.sched_getaffinity(0)
for name, cpus in node_cpus.items():
    os.sched_setaffinity(0, cpus)
    host = torch.empty(N // 8, dtype=torch.int64, pin_memory=True)
    os.sched_setaffinity(0, orig)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"alloc_node": name, "d2h_GBps": round(N / best / 1e9, 2)}), flush=True)
    del host

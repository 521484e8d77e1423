"""Host->device copy bandwidth from pinned memory, with the process on all CPUs and then bound
to the CPUs local to the GPU (sysfs local_cpulist; pinned pages first-touched there)."""
import os
import sys
import time

import torch


def local_cpus():
    bus = getattr(torch.cuda.get_device_properties(0), "pci_bus_id", None)
    if not isinstance(bus, str):   # some torch versions expose the bus number only
        import subprocess
        bus = subprocess.check_output(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader",
                                       "-i", "0"]).decode().strip()
    bus = bus.lower()
    if bus.count(":") == 2 and len(bus.split(":")[0]) == 8:
        bus = bus[4:]
    path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
    s = open(path).read().strip()
    cpus = set()
    for part in s.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return path, s, cpus


def h2d(gb=4.0, reps=3):
    n = int(gb * (1 << 30))
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    del h, d
    return best


torch.cuda.init()
print("all cpus:", len(os.sched_getaffinity(0)), "H2D GB/s", round(h2d(), 1), flush=True)
try:
    path, s, cpus = local_cpus()
    print("local_cpulist", path, s)
    os.sched_setaffinity(0, cpus)
    print("bound:", len(os.sched_getaffinity(0)), "H2D GB/s", round(h2d(), 1), flush=True)
except Exception as ex:  # noqa: BLE001
    print("no local cpu list:", ex)
sys.exit(0)

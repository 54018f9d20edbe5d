"""Host topology of the GPU box and the PCIe copy rate from pinned buffers placed on each NUMA
node (the calling thread bound to the node's CPUs while the buffer is allocated and first
touched), one direction at a time and both at once: does host-buffer placement move the e2e
path's copy rate?

    python tools/numa_probe.py
"""
import glob
import os
import time

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


dev = torch.device("cuda:0")
p = torch.cuda.get_device_properties(0)
bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
try:
    gnode = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read())
except OSError:
    gnode = None
nodes = sorted(int(n.rsplit("node", 1)[1]) for n in glob.glob("/sys/devices/system/node/node[0-9]*"))
print(f"gpu {bus} numa_node {gnode}; nodes {nodes}; cpus {os.cpu_count()}; affinity {len(os.sched_getaffinity(0))}")
for n in nodes:
    print(f"  node {n}: cpus {open(f'/sys/devices/system/node/node{n}/cpulist').read().strip()}")

nbytes = 403 * 1000 * 1000
d = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
d2 = torch.empty_like(d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
orig = os.sched_getaffinity(0)
for n in nodes + [None]:
    cpus = cpulist(open(f"/sys/devices/system/node/node{n}/cpulist").read()) if n is not None else sorted(orig)
    os.sched_setaffinity(0, cpus)
    h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    h.fill_(1.0)
    h2 = torch.empty_like(h).pin_memory()
    h2.fill_(1.0)
    res = {}
    for name in ("h2d", "d2h", "both"):
        best = 0.0
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = max(best, nbytes * (2 if name == "both" else 1) / dt / 1e9)
        res[name] = round(best, 1)
    print(f"buffers on node {n if n is not None else 'default'}: GB/s {res}", flush=True)
    del h, h2
os.sched_setaffinity(0, orig)

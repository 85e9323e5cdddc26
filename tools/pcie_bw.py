"""Host<->device copy bandwidth of the GPU box (pinned host memory), one direction at a time
and both at once, with the process on all CPUs and then pinned to the GPU's NUMA node
(first-touch puts the pinned pages there).  Explains the e2e leg of bench.py.
usage: python tools/pcie_bw.py [MiB]"""
import os
import sys

import torch

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = mib << 20


def gpu_numa():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
    bus = bus.lower()[-12:]
    base = f"/sys/bus/pci/devices/{bus}"
    node = int(open(f"{base}/numa_node").read().strip())
    cpus = open(f"{base}/local_cpulist").read().strip()
    return bus, node, cpus


def parse_list(s):
    out = set()
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def run(tag):
    h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_up.fill_(1)
    h_dn.fill_(2)
    d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_up.copy_(h_up, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dn.copy_(d_dn, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_up = timed(lambda: d_up.copy_(h_up, non_blocking=True))
    t_dn = timed(lambda: h_dn.copy_(d_dn, non_blocking=True))
    t_bo = timed(both)
    print(f"{tag}: H2D {n / t_up / 1e9:6.1f} GB/s  D2H {n / t_dn / 1e9:6.1f} GB/s  "
          f"both at once {2 * n / t_bo / 1e9:6.1f} GB/s total", flush=True)


torch.cuda.init()
try:
    bus, node, cpus = gpu_numa()
    print(f"GPU {bus}: NUMA node {node}, local CPUs {cpus}; process CPUs {len(os.sched_getaffinity(0))}; "
          f"nodes {sorted(os.listdir('/sys/devices/system/node'))}", flush=True)
except Exception as e:  # noqa: BLE001
    print("no NUMA info:", e)
    cpus = None
run("all CPUs")
if cpus:
    os.sched_setaffinity(0, parse_list(cpus))
    run(f"pinned to {cpus}")

"""PCIe throughput vs the NUMA node the pinned host buffers live on: for
every node, pin this process to the node's CPUs, allocate (first touch)
pinned buffers there, time H2D, D2H and both at once.  GB/s per direction."""

from __future__ import annotations

import glob
import json
import os

import torch


def cpulist(s: str) -> set[int]:
    out = set()
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out |= set(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def gbps(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def main():
    torch.cuda.init()
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    info = {"gpu_pci": bus}
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    info["nodes"] = {os.path.basename(n): open(f"{n}/cpulist").read().strip() for n in nodes}
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        pci = pynvml.nvmlDeviceGetPciInfo(h).busId
        pci = pci.decode() if isinstance(pci, bytes) else pci
        dom = pci.lower()[-12:]
        for cand in glob.glob("/sys/bus/pci/devices/*"):
            if cand.lower().endswith(dom):
                info["gpu_numa_node"] = open(f"{cand}/numa_node").read().strip()
        info["gpu_busid"] = pci
    except Exception as e:  # noqa: BLE001
        info["nvml"] = str(e)
    print(json.dumps(info), flush=True)
    n = 334_430_208 // 8
    dev_a = torch.empty(n, dtype=torch.float64, device="cuda")
    dev_b = torch.empty(n, dtype=torch.float64, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    for node in nodes:
        cpus = cpulist(open(f"{node}/cpulist").read())
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        h_in = torch.zeros(n, dtype=torch.float64).pin_memory()
        h_out = torch.zeros(n, dtype=torch.float64).pin_memory()

        def h2d():
            with torch.cuda.stream(up):
                dev_a.copy_(h_in, non_blocking=True)
            torch.cuda.current_stream().wait_stream(up)

        def d2h():
            with torch.cuda.stream(down):
                h_out.copy_(dev_b, non_blocking=True)
            torch.cuda.current_stream().wait_stream(down)

        def both():
            up.wait_stream(torch.cuda.current_stream())
            down.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(up):
                dev_a.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(down):
                h_out.copy_(dev_b, non_blocking=True)
            torch.cuda.current_stream().wait_stream(up)
            torch.cuda.current_stream().wait_stream(down)

        r = {"node": os.path.basename(node), "h2d": gbps(h2d, n * 8), "d2h": gbps(d2h, n * 8),
             "both_each": gbps(both, n * 8)}
        print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
        del h_in, h_out


if __name__ == "__main__":
    main()

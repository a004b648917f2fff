"""PCIe ceiling of this box: H2D / D2H bandwidth between pinned host memory and the GPU,
one vs several concurrent streams, several transfer sizes, and with the pinned buffer first-
touched from a CPU on the GPU's NUMA node vs elsewhere.  Bounds the e2e (host-buffer) numbers
of bench.py."""
import json
import os
import sys

import torch


def numa_of_gpu(idx=0):
    try:
        import pynvml  # nvidia_ml_py
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        bus = bus.lower()[-12:]
        for cand in (bus, "0000" + bus[-8:]):
            p = "/sys/bus/pci/devices/%s/numa_node" % cand
            if os.path.exists(p):
                return int(open(p).read()), bus
        return None, bus
    except Exception as e:  # noqa: BLE001
        return None, str(e)


def bw(nbytes, nstreams, direction, reps=10, pinned=None):
    dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    host = pinned if pinned is not None else torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    n = nbytes // 8
    parts = [(i * n // nstreams, (i + 1) * n // nstreams) for i in range(nstreams)]

    def once():
        for s, (a, b) in zip(streams, parts):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                if direction == "d2h":
                    host[a:b].copy_(dev[a:b], non_blocking=True)
                else:
                    dev[a:b].copy_(host[a:b], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)

    once()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return nbytes / (ms * 1e-3) / 1e9


def main():
    torch.cuda.set_device(0)
    node, bus = numa_of_gpu(0)
    out = {"gpu_numa_node": node, "bus": bus, "cpus": os.cpu_count(),
           "affinity": sorted(os.sched_getaffinity(0))[:4] + ["..."]}
    res = []
    for size in (8 << 20, 80_000_000, 256 << 20):
        for ns in (1, 2, 4):
            for d in ("d2h", "h2d"):
                res.append({"bytes": size, "streams": ns, "dir": d, "GBps": round(bw(size, ns, d), 2)})
    out["default"] = res
    # both directions at once (separate copy engines): the ceiling of the elementwise e2e path,
    # which streams its input up while the results of earlier chunks come back
    n = 256 << 20
    a_d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
    b_d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
    a_h = torch.empty(n // 8, dtype=torch.float64).pin_memory()
    b_h = torch.empty(n // 8, dtype=torch.float64).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            a_d.copy_(a_h, non_blocking=True)
        with torch.cuda.stream(s2):
            b_h.copy_(b_d, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    both()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        both()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out["bidirectional_256MB_each"] = {"ms": round(ms, 3),
                                       "GBps_per_direction": round(n / (ms * 1e-3) / 1e9, 2),
                                       "GBps_total": round(2 * n / (ms * 1e-3) / 1e9, 2)}
    # pin from a CPU on the GPU's NUMA node (first touch decides the page's node)
    if node is not None and node >= 0:
        try:
            cpus = [int(x) for x in open("/sys/devices/system/node/node%d/cpulist" % node).read()
                    .strip().replace("-", ",").split(",")[:1]]
            lst = open("/sys/devices/system/node/node%d/cpulist" % node).read().strip()
            first = []
            for part in lst.split(","):
                a, _, b = part.partition("-")
                first += list(range(int(a), int(b or a) + 1))
            os.sched_setaffinity(0, first)
            h = torch.zeros(80_000_000 // 8, dtype=torch.float64).pin_memory()
            out["numa_local"] = {"cpulist": lst,
                                 "d2h_1s": round(bw(80_000_000, 1, "d2h", pinned=h), 2),
                                 "d2h_2s": round(bw(80_000_000, 2, "d2h", pinned=h), 2),
                                 "h2d_1s": round(bw(80_000_000, 1, "h2d", pinned=h), 2)}
            del cpus
        except Exception as e:  # noqa: BLE001
            out["numa_local"] = str(e)
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()

"""Pinned-buffer H2D/D2H rate by the NUMA node the buffer was allocated from
(process affinity set to that node's CPUs before cudaHostAlloc), next to the
GPU-local CPU set NVML reports. One JSON line; see profiles/r01_e2e.md."""
import glob
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def cpulist(path):
    out = set()
    for part in open(path).read().strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out |= set(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def timed(fn, reps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    torch.cuda.set_device(0)
    n = 4096 * 64 * 5
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    res = {"bytes": n * 8, "nvml_local_cpus": sorted(bench._gpu_local_cpus(0) or [])[:4] + ["..."]}
    allc = os.sched_getaffinity(0)
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    for node in nodes:
        cpus = cpulist(node + "/cpulist") & allc
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        h = torch.empty(n, dtype=torch.float64).pin_memory()
        h.fill_(1.0)
        name = os.path.basename(node)
        res[name + "_cpus"] = len(cpus)
        res[name + "_h2d_ms"] = timed(lambda: dev.copy_(h, non_blocking=True))
        res[name + "_d2h_ms"] = timed(lambda: h.copy_(dev, non_blocking=True))
        del h
    os.sched_setaffinity(0, allc)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

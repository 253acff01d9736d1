"""Benchmark of the flux-differencing volume integral (BASELINE.json metric:
volume-integral DOF updates/s = 1/PID, fp64).

Workload (BASELINE.json configs[1]): 3D compressible Euler, N=3 (4^3 LGL nodes),
16^3 periodic Cartesian hexes on [-1,1]^3, Ranocha EC flux, density-wave state
(rho = 1 + 0.98 sin(pi(x+y+z)), v = (0.1,0.2,0.3), p = 20); one step = one
volume-integral pass over the mesh (262,144 nodes). The FAST kernels with
per-node log tables (precompute="primitives_and_logs", the paper's
technique). The input (10.5 MB) fits in L2, so the steps rotate over replicas
of (u, VOL) whose total exceeds 3x L2 (every step reads its input from HBM);
the K timed steps run as one CUDA graph bracketed by CUDA events. A secondary
figure times each launch alone with L2 flushed before it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): the volume integral has no exchange step; every rank
owns one cfg2-sized slab (weak scaling), value = all nodes / max-rank time.
--impl reference times the CPU oracle (C restatement of the reference's
scalar path, bitwise equal to it; all host threads) on the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "volume-integral DOF updates/s (1/PID), fp64"
UNIT = "DOF/s"
BYTES_PER_NODE = 80.0  # u read once + VOL written once, 5 doubles each
FLOP_PER_NODE = 428.5  # Ranocha Cartesian 3D N=3, prim+logs, log branch
CONFIG_NAME = "cfg2: 3D Euler N=3, 16^3 Cartesian hexes, Ranocha EC, volume integral"
L2_BYTES = 126 * 1024 * 1024  # B200 L2


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = (
        "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
        "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.QUERY, "--format=csv,noheader,nounits",
                 "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def n_samples(self):
        return len(self.rows)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for name, val in zip(names, r[5:9]):
                    if val.lower() == "active":
                        reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
            "window": "from the first timed launch through a <=3 s continuation of the same launch sequence",
        }


def cpu_baseline(setup, u, steps=3):
    """The oracle (reference arithmetic, bitwise) on the host cores."""
    from oracle import oracle

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    mesh = oracle.mesh_from_setup(setup)
    oracle.volume(u, mesh, "ranocha", "primitives_and_logs", nthreads=threads)  # warm-up
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.volume(u, mesh, "ranocha", "primitives_and_logs", nthreads=threads)
        times.append(time.perf_counter() - t0)
    nodes = u.shape[0] * u.shape[1]
    return {
        "value": nodes / statistics.mean(times),
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": "full cfg2 mesh (4096 elements, 262144 nodes), oracle/fdg_oracle.c volume_fluxdiff order, "
                  "precompute=primitives_and_logs, %d timed passes after 1 warm-up, mean" % steps,
        "cpu_model": _cpu_model(),
    }


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the same workload (rank 0 only)."""
    if rank != 0:
        return 0
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(2)
    from oracle import oracle

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    mesh = oracle.mesh_from_setup(setup)
    for _ in range(args.warmup):
        oracle.volume(u, mesh, "ranocha", "primitives_and_logs", nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.volume(u, mesh, "ranocha", "primitives_and_logs", nthreads=threads)
        times.append(time.perf_counter() - t0)
    nodes = u.shape[0] * u.shape[1]
    ms = 1e3 * statistics.mean(times)
    value = nodes / (ms * 1e-3)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAME, "nodes": nodes, "elements": u.shape[0]},
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": threads,
            "kind": "port",
            "sample": "each step: full cfg2 volume integral (262144 nodes) through oracle/fdg_oracle.c "
                      "(C restatement of the reference's scalar path, bitwise equal to it), pthreads",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _gpu_local_cpus(index):
    """Host CPUs NVML reports as local to GPU `index` (its NUMA node), or None."""
    try:
        import pynvml

        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            n = os.cpu_count() or 64
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        finally:
            pynvml.nvmlShutdown()
        cpus = {64 * w + b for w, mask in enumerate(words) for b in range(64) if (int(mask) >> b) & 1}
        return cpus or None
    except Exception:
        return None


def _traffic_from_profile():
    """dram bytes per launch of the volume kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "vol_cfg2_ncu_summary.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def run_sharded(args, rank, world, local, dist):
    """Full RHS (or SSPRK43 step) of cfg4 / cfg5, slab-partitioned over the
    ranks with the NCCL face-trace halo every RHS (strong scaling)."""
    import torch

    from paper_2112_10517_b200 import _native as N
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DeviceMesh
    from paper_2112_10517_b200.parallel import HaloExchange, slab_partition
    from paper_2112_10517_b200.timeint import SSPRK43, DeviceStepper

    cfg = {"rhs4": 4, "rhs5": 5, "step4": 4}[args.workload]
    setup, u_host, config = workloads.build(cfg, kernel="batched")
    part = slab_partition(setup, rank, world)
    dm = DeviceMesh(setup, partition=part)
    lo, hi = part["lo"], part["hi"]
    u = torch.as_tensor(np.ascontiguousarray(u_host[lo:hi]), device="cuda")
    nodes_total = u_host.shape[0] * u_host.shape[1]
    del u_host
    halo = HaloExchange(part, setup.d, setup.op.degree + 1, torch, dist, device="cuda", pack=dm.pack_faces) \
        if world > 1 else None
    scheme = config.scheme()
    out = dm.empty()
    stepper = None
    if args.workload == "step4":
        stepper = DeviceStepper(dm, config, SSPRK43, exchange=halo)
        dt = 1e-4

    def step():
        if stepper is not None:
            return stepper.step(u, dt, check=False)
        ghost = halo(u) if halo is not None else None
        return dm.rhs(u, scheme, out=out, ghost_u=ghost)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    stream = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    launches0 = N.launch_count()
    with ClockSampler(local) as clocks:
        a.record(stream)
        for _ in range(args.steps):
            step()
        b.record(stream)
        torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    ms = a.elapsed_time(b) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rhs_per_step = 4 if stepper is not None else 1
    value = nodes_total * rhs_per_step / (ms * 1e-3)
    line = {
        "metric": "full-RHS DOF updates/s (1/PID), fp64",
        "value": value,
        "unit": "DOF/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": "cfg%d %s: %s" % (cfg, args.workload, workloads.CONFIGS[cfg]),
            "nodes_total": nodes_total,
            "partition": "x-slabs of the element index, NCCL grouped send/recv of face traces per RHS",
            "l2": "inputs larger than L2 (%.0f MB state)" % (nodes_total * 5 * 8 / 1e6),
            "rhs_per_step": rhs_per_step,
        },
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="vol2", choices=["vol2", "rhs4", "rhs5", "step4"],
                    help="vol2: the headline (BASELINE configs[1]); rhs4/rhs5: sharded full RHS of cfg4/cfg5 "
                         "(strong scaling, NCCL face-trace halo); step4: sharded SSPRK43 step of cfg4")
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload != "vol2":
        return run_sharded(args, rank, world, local, dist)

    from paper_2112_10517_b200 import _native as N
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import device_mesh_for
    from paper_2112_10517_b200.discretization import mesh_fluxdiff_volume

    setup, u_host, config = workloads.build(2, kernel="batched")
    nodes = u_host.shape[0] * u_host.shape[1]
    dm = device_mesh_for(setup)
    scheme = config.scheme()
    stream = torch.cuda.current_stream()
    # Rotating replicas: step i reads u[i % R] and writes vol[i % R]; R copies
    # of (u, VOL) span > 3x the 126 MB L2, so every step's input comes from
    # HBM (by the time a replica is reused, > 3x L2 of other data has passed).
    step_bytes = 2 * u_host.nbytes
    n_rep = max(2, -(-3 * L2_BYTES // step_bytes))
    u0 = torch.as_tensor(u_host, device="cuda")
    us = [u0.clone() for _ in range(n_rep)]
    vols = [dm.empty() for _ in range(n_rep)]
    del u0

    def step(i):
        dm.volume(us[i % n_rep], scheme, out=vols[i % n_rep])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # the K timed steps are one CUDA graph (kernel after kernel, no host launch
    # gaps): the measured time per step is what a solver loop pays per volume
    # integral, launch-to-launch
    graph = torch.cuda.CUDAGraph()
    launches0 = N.launch_count()
    with torch.cuda.graph(graph):
        for i in range(args.steps):
            step(i)
    launches = N.launch_count() - launches0  # kernel nodes in the graph (one per step)
    graph.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        a.record(stream)
        graph.replay()
        b.record(stream)
        torch.cuda.synchronize()
        # the timed region lasts well under nvidia-smi's sampling period: keep the
        # same launch sequence running until the sampler has seen the load
        t_end = time.time() + 3.0
        while time.time() < t_end and clocks.n_samples() < 8:
            for _ in range(20):
                graph.replay()
            torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = a.elapsed_time(b) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * nodes / (ms * 1e-3)

    # secondary: each launch alone, L2 flushed before it (event pair per launch)
    flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.sum()
        starts[i].record(stream)
        step(0)
        ends[i].record(stream)
    torch.cuda.synchronize()
    per_launch_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    del flush, graph

    # ---- end to end through the public API with pinned host buffers
    # The pinned buffers are allocated (pages placed) and the e2e loop runs on
    # the GPU's NUMA-local CPUs (NVML CPU affinity): a remote-socket buffer
    # halves the H2D rate on some hosts. The affinity is restored afterwards
    # (the CPU baseline below uses every host thread).
    cpus_all = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    cpus_near = _gpu_local_cpus(local)
    if cpus_near and cpus_all:
        cpus_near &= cpus_all
        if cpus_near:
            os.sched_setaffinity(0, cpus_near)
    try:
        # page-locked by cudaHostAlloc (libfdg fdg_host_alloc): caching-allocator
        # pinned blocks ran H2D at 0.20-0.74 ms for the same 10.5 MB on one box
        u_pin = N.pinned_empty(u_host.shape)
        np.copyto(u_pin.numpy(), u_host)
        out_pin = N.pinned_empty(u_host.shape)
        for _ in range(max(args.warmup, 3)):
            mesh_fluxdiff_volume(u_pin, setup, config, out=out_pin)
        e2e_ms = []
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mesh_fluxdiff_volume(u_pin, setup, config, out=out_pin)
            b.record(stream)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
    finally:
        if cpus_near and cpus_all:
            os.sched_setaffinity(0, cpus_all)
    e2e = statistics.mean(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    hbm, peak_src = _peaks()
    achieved = BYTES_PER_NODE * nodes / (ms * 1e-3) / 1e9
    fp64_peak = N.fp64_peak_tflops()
    traffic = _traffic_from_profile()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": CONFIG_NAME,
            "elements_per_gpu": u_host.shape[0],
            "nodes_per_gpu": nodes,
            "kernel": "batched (FAST), precompute=primitives_and_logs",
            "l2": "inputs larger than L2: %d rotating replicas of (u, VOL), %.0f MB > 3x the 126 MB L2" % (
                n_rep, n_rep * step_bytes / 1e6),
            "timing": "K steps captured in one CUDA graph, CUDA events around the replay, ms_per_step = total / K",
            "parallelism": "replicas per GPU (element-local, no exchange)" if world > 1 else "single GPU",
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": hbm,
            "unit": "GB/s",
            "frac": achieved / hbm,
            "traffic": traffic,
            "peak_source": peak_src + " (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic_bytes_per_node": BYTES_PER_NODE,
        },
        "fp64": {
            "achieved_tflops": FLOP_PER_NODE * nodes / (ms * 1e-3) / 1e12,
            "peak_tflops_probe": fp64_peak,
            "frac": FLOP_PER_NODE * nodes / (ms * 1e-3) / 1e12 / fp64_peak if fp64_peak else None,
            "algorithmic_flop_per_node": FLOP_PER_NODE,
        },
        "e2e": {
            "value": world * nodes / (e2e * 1e-3),
            "unit": UNIT,
            "ms_per_step": e2e,
            "h2d_bytes_per_step": int(u_host.nbytes),
            "d2h_bytes_per_step": int(u_host.nbytes),
            "host_cpus": "GPU-local (NVML affinity, %d CPUs) for the pinned buffers and the loop" % len(cpus_near)
            if cpus_near else "process default",
            "ms_min": min(e2e_ms),
            "ms_median": statistics.median(e2e_ms),
            "path": "paper_2112_10517_b200.mesh_fluxdiff_volume(pinned CPU tensor, out=pinned) -> libfdg.so "
            "fdg_volume_host (chunked H2D / kernel / D2H pipeline)",
        },
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "isolated_launch_ms": {
            "mean": statistics.mean(per_launch_ms), "min": min(per_launch_ms), "max": max(per_launch_ms),
            "how": "each launch alone between its own event pair, L2 flushed (256 MB read) before it",
        },
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(setup, u_host)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

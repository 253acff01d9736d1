"""Benchmark of the flux-differencing volume integral (BASELINE.json metric:
volume-integral DOF updates/s = 1/PID, fp64).

Headline workload (BASELINE.json configs[4], the largest configuration and
the one that fits a single B200): 3D compressible Euler, N=3 (4^3 LGL
nodes), 128^3 periodic Cartesian hexes on [-1,1]^3 (134,217,728 nodes, 5.4 GB
state), Ranocha EC flux, the seeded perturbed density wave (rho = 1 + 0.98
sin(pi(x+y+z)) + 0.01 clip(N(0,1), -1, 1), v = (0.1,0.2,0.3), p = 20; the
clip is SURVEY.md 9 item 4); one step = one volume-integral pass over the
mesh, FAST kernels with per-node log tables (precompute="primitives_and_logs",
the paper's technique). Geometry and state are built on the device
(workloads.build_device), so no 22 GB host setup happens. The state (5.4 GB)
is 43x the 126 MB L2: every step reads its input from HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload vol5|vol3|vol2|rhs5|rhs4|step4] [--quick]

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL). The elements
are split into contiguous slabs of the C-ordered element index (strong
scaling: total work fixed); the volume integral has no exchange step, so the
only collectives are the barriers and the MAX of the per-rank device times.
value = all nodes / max-rank time per step.

Secondary lines (``secondary``, skipped by --quick): the other volume-integral
configs (cfg5 Shima, cfg3 N=7 Chandrashekar -- FP64-bound --, cfg2) and the
sharded full RHS of cfg5, cfg4 and one cfg4 SSPRK43 step, slab-partitioned
with the NCCL face-trace halo at N > 1.

--impl reference times the reference's scalar path on the host cores (the C
restatement oracle/fdg_oracle.c, bitwise equal to the reference; all host
threads) on a bounded sample of the same workload: the first 8 element planes
of the 128^3 mesh (131,072 elements, 8.4 M nodes; VOL is element-local, so
the per-node rate is the whole mesh's).
"""

import argparse
import hashlib
import json
import os
import socket
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
L2_BYTES = 126 * 1024 * 1024  # B200 L2
SAMPLE_PLANES = 8  # CPU sample: the first 8 planes of 128^2 elements

# per workload: BASELINE config, volume flux, algorithmic bytes / flops per node
VOL_WORKLOADS = {
    "vol5": dict(cfg=5, flux="ranocha", bytes=80.0, flop=428.5,
                 name="cfg5: 3D Euler N=3, 128^3 Cartesian hexes, Ranocha EC, noisy density wave, volume integral"),
    "vol5_shima": dict(cfg=5, flux="shima", bytes=80.0, flop=287.0,
                       name="cfg5: 3D Euler N=3, 128^3 Cartesian hexes, Shima KEP, noisy density wave, volume integral"),
    "vol3": dict(cfg=3, flux="chandrashekar", bytes=80.0, flop=1058.5,
                 name="cfg3: 3D Euler N=7, 32^3 Cartesian hexes, Chandrashekar EC, seeded random state, volume integral"),
    "vol2": dict(cfg=2, flux="ranocha", bytes=80.0, flop=428.5,
                 name="cfg2: 3D Euler N=3, 16^3 Cartesian hexes, Ranocha EC, density wave, volume integral"),
}


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
        return float(p.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _config_dict(workload, world):
    """The config object both arms print (identical keys and values)."""
    w = VOL_WORKLOADS[workload]
    from paper_2112_10517_b200 import workloads

    c = workloads.CONFIGS[w["cfg"]]
    n_elem = int(np.prod(c["dims"]))
    nodes = n_elem * (c["p"] + 1) ** len(c["dims"])
    return {
        "workload": w["name"],
        "elements": n_elem,
        "nodes": nodes,
        "dofs": nodes * (len(c["dims"]) + 2),
        "volume_flux": w["flux"],
        "precompute": "primitives_and_logs" if w["flux"] in ("ranocha", "chandrashekar") else "none",
        "l2": "input larger than L2 (%.0f MB state > 126 MB)" % (nodes * (len(c["dims"]) + 2) * 8 / 1e6)
        if nodes * (len(c["dims"]) + 2) * 8 > 3 * L2_BYTES else "rotating replicas > 3x L2",
        "parallelism": "element slabs over %d ranks, no exchange (strong scaling)" % world if world > 1
        else "single GPU",
    }


# ----------------------------------------------------------------- clocks


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


# ------------------------------------------------------------ CPU (oracle)


def _host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _oracle_sample(workload):
    """(oracle mesh, host state) of the bounded CPU sample of ``workload``."""
    from types import SimpleNamespace

    from oracle import oracle
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.operators import build_dsplit, lgl_operator

    w = VOL_WORKLOADS[workload]
    c = workloads.CONFIGS[w["cfg"]]
    plane = int(np.prod(c["dims"][1:]))
    n_s = min(SAMPLE_PLANES, c["dims"][0]) * plane
    u, areas, jac = workloads.cartesian_sample(w["cfg"], n_s)
    op = lgl_operator(c["p"])
    d = len(c["dims"])
    setup = SimpleNamespace(
        d=d, op=op, dsplit=build_dsplit(op), gas=workloads.GAS,
        metrics=SimpleNamespace(cartesian=True, areas=tuple(areas), jac_const=jac),
        plus_neighbor=tuple(np.arange(n_s) for _ in range(d)),
    )
    return oracle.mesh_from_setup(setup), u


def _sample_desc(workload, u):
    return ("first %d element planes of the mesh (%d elements, %d nodes) through oracle/fdg_oracle.c "
            "(C restatement of the reference's scalar volume_fluxdiff, bitwise equal to it), "
            "precompute=%s, pthreads" % (SAMPLE_PLANES, u.shape[0], u.shape[0] * u.shape[1],
                                         _config_dict(workload, 1)["precompute"]))


def cpu_baseline(workload, passes=5):
    """The oracle on the host cores on the bounded sample (rank 0, N=1)."""
    from oracle import oracle

    w = VOL_WORKLOADS[workload]
    pre = _config_dict(workload, 1)["precompute"]
    mesh, u = _oracle_sample(workload)
    threads = _host_threads()
    oracle.volume(u, mesh, w["flux"], pre, nthreads=threads)  # warm-up
    times = []
    for _ in range(passes):
        t0 = time.perf_counter()
        oracle.volume(u, mesh, w["flux"], pre, nthreads=threads)
        times.append(time.perf_counter() - t0)
    nodes = u.shape[0] * u.shape[1]
    return {
        "value": nodes / statistics.mean(times),
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": _sample_desc(workload, u) + "; %d timed passes after 1 warm-up, mean" % passes,
        "cpu_model": _cpu_model(),
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's scalar path (C restatement) on the
    host cores, same workload, config, metric (rank 0 only)."""
    if rank != 0:
        return 0
    from oracle import oracle

    workload = args.workload if args.workload in VOL_WORKLOADS else "vol5"
    w = VOL_WORKLOADS[workload]
    pre = _config_dict(workload, 1)["precompute"]
    mesh, u = _oracle_sample(workload)
    threads = _host_threads()
    for _ in range(args.warmup):
        oracle.volume(u, mesh, w["flux"], pre, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.volume(u, mesh, w["flux"], pre, nthreads=threads)
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
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": _config_dict(workload, world),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": threads,
            "kind": "port",
            "sample": _sample_desc(workload, u) + "; each step one pass",
            "cpu_model": _cpu_model(),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- helpers


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


def _lib_digest():
    """sha256 (16 hex) of the kernel SOURCES libfdg.so is built from
    (csrc/*.cu, *.cuh, *.h, units/, Makefile, include/fdg.h): identifies the
    build across rebuilds of the same sources."""
    csrc = os.path.join(ROOT, "paper_2112_10517_b200", "csrc")
    files = []
    for base, dirs, names in os.walk(csrc):
        dirs[:] = sorted(d for d in dirs if not d.startswith("obj"))
        files += [os.path.join(base, n) for n in names
                  if n.endswith((".cu", ".cuh", ".h")) or n == "Makefile"]
    files.append(os.path.join(ROOT, "include", "fdg.h"))
    h = hashlib.sha256()
    for f in sorted(files):
        h.update(os.path.relpath(f, ROOT).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _traffic_from_profile(workload):
    """DRAM bytes per launch of the timed kernel, from the ncu capture of the
    same libfdg.so build committed under profiles/ (matched by the library's
    sha256; null when the library was rebuilt since)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None, "no committed capture"
    with open(path) as f:
        rec = json.load(f)
    ent = rec.get(workload)
    if not ent:
        return None, "no capture of this workload"
    if ent.get("src_sha16") != _lib_digest():
        return None, "capture %s is of another kernel-source revision" % ent.get("capture")
    return ent.get("dram_bytes_per_launch"), ent.get("capture")


def _max_over_ranks(x, dist):
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _slab_setup(setup, lo, hi):
    """A Cartesian setup restricted to elements [lo, hi) for the element-local
    volume integral (no neighbours are read)."""
    from types import SimpleNamespace

    d = setup.d
    return SimpleNamespace(
        d=d, op=setup.op, dsplit=setup.dsplit, gas=setup.gas, metrics=setup.metrics,
        plus_neighbor=tuple(np.arange(hi - lo) for _ in range(d)), n_elements=hi - lo,
    )


def _slab_range(n_planes, plane, rank, world):
    p_lo, p_hi = n_planes * rank // world, n_planes * (rank + 1) // world
    return p_lo * plane, p_hi * plane


def _time_launches(step, steps, stream, dist, local, sample_clocks=True):
    """K launches of ``step`` between two events on ``stream`` (barrier and
    synchronize on both sides); max over ranks. Returns (ms/step, clocks)."""
    import torch

    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    clocks = None
    if sample_clocks:
        with ClockSampler(local) as cs:
            a.record(stream)
            for i in range(steps):
                step(i)
            b.record(stream)
            torch.cuda.synchronize()
            t_end = time.time() + 3.0
            while time.time() < t_end and cs.n_samples() < 8:
                for i in range(steps):
                    step(i)
                torch.cuda.synchronize()
        clocks = cs.summary()
    else:
        a.record(stream)
        for i in range(steps):
            step(i)
        b.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = _max_over_ranks(a.elapsed_time(b) / steps, dist)
    return ms, clocks


# --------------------------------------------------------------- GPU arms


def measure_volume(workload, args, rank, world, local, dist, headline):
    """One volume-integral workload, elements split into slabs over ranks."""
    import torch

    from paper_2112_10517_b200 import _native as N
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import device_mesh_for

    w = VOL_WORKLOADS[workload]
    setup, u_full, config = workloads.build_device(w["cfg"], kernel="batched", volume_flux=w["flux"])
    c = workloads.CONFIGS[w["cfg"]]
    plane = int(np.prod(c["dims"][1:]))
    lo, hi = _slab_range(c["dims"][0], plane, rank, world)
    u = u_full[lo:hi].clone() if world > 1 else u_full
    del u_full
    nodes_total = setup.n_elements * setup.n_nodes
    nodes_local = u.shape[0] * u.shape[1]
    slab = _slab_setup(setup, lo, hi)
    dm = device_mesh_for(slab)
    scheme = config.scheme()
    stream = torch.cuda.current_stream()
    step_bytes = 2 * u.numel() * 8
    n_rep = 1 if step_bytes > 3 * L2_BYTES else max(2, -(-3 * L2_BYTES // step_bytes))
    us = [u] + [u.clone() for _ in range(n_rep - 1)]
    vols = [dm.empty() for _ in range(n_rep)]

    def step(i):
        dm.volume(us[i % n_rep], scheme, out=vols[i % n_rep])

    for i in range(args.warmup):
        step(i)
    graph = None
    if n_rep > 1:
        # short launches: the K steps as one CUDA graph (no host launch gaps)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(args.steps):
                step(i)
        graph.replay()
        torch.cuda.synchronize()
    if graph is not None:
        # the whole K-step graph is replayed in call 0: elapsed / K = per step
        ms, clocks = _time_launches(lambda i: graph.replay() if i == 0 else None, args.steps, stream, dist, local,
                                    sample_clocks=headline)
    else:
        ms, clocks = _time_launches(step, args.steps, stream, dist, local, sample_clocks=headline)
    launches = args.steps  # one element-kernel launch per step
    value = nodes_total / (ms * 1e-3)
    hbm, peak_src = _peaks()
    achieved = w["bytes"] * nodes_total / world / (ms * 1e-3) / 1e9  # per GPU
    fp64_peak = N.fp64_peak_tflops()
    tflops = w["flop"] * nodes_total / world / (ms * 1e-3) / 1e12
    res = {
        "value": value,
        "ms_per_step": ms,
        "nodes": nodes_total,
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": hbm,
            "unit": "GB/s",
            "frac": achieved / hbm,
            "peak_source": peak_src,
            "algorithmic_bytes_per_node": w["bytes"],
            "per": "GPU (each rank's slab / the max-rank time)",
        },
        "fp64": {
            "achieved_tflops": tflops,
            "peak_tflops_probe": fp64_peak,
            "frac": tflops / fp64_peak if fp64_peak else None,
            "algorithmic_flop_per_node": w["flop"],
        },
        "timing": ("K steps in one CUDA graph over %d rotating replicas of (u, VOL) (> 3x L2)" % n_rep)
        if graph is not None else "K launches between two CUDA events; the input is > 3x L2",
        "gpu_launches": launches,
    }
    # the binding roofline side: the slower of HBM bytes and FP64 flops
    t_hbm = w["bytes"] / (hbm * 1e9)
    t_fp = w["flop"] / (fp64_peak * 1e12) if fp64_peak else 0.0
    res["roofline_bound"] = "fp64" if t_fp > t_hbm else "hbm"
    res["roofline_frac_binding"] = (max(t_hbm, t_fp) * nodes_total / world) / (ms * 1e-3)
    if headline:
        res["clocks"] = clocks
        traffic, src = _traffic_from_profile(workload)
        res["roofline"]["traffic"] = traffic
        res["roofline"]["traffic_source"] = src
        res["_e2e"] = _e2e_volume(args, slab, u, config, local, dist, nodes_total, world)
    return res


def _e2e_volume(args, slab, u_dev, config, local, dist, nodes_total, world):
    """The same metric through the public API with HOST buffers: pinned host
    state in, pinned host VOL out, every step's H2D and D2H inside the timed
    region (mesh_fluxdiff_volume -> fdg_volume_host, chunked pipeline)."""
    import torch

    from paper_2112_10517_b200 import _native as N
    from paper_2112_10517_b200.discretization import mesh_fluxdiff_volume

    stream = torch.cuda.current_stream()
    cpus_all = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    cpus_near = _gpu_local_cpus(local)
    if cpus_near and cpus_all:
        cpus_near &= cpus_all
        if cpus_near:
            os.sched_setaffinity(0, cpus_near)
    try:
        u_pin = N.pinned_empty(tuple(u_dev.shape))
        u_pin.copy_(u_dev)
        out_pin = N.pinned_empty(tuple(u_dev.shape))
        steps = max(3, min(args.steps, 10))
        for _ in range(2):
            mesh_fluxdiff_volume(u_pin, slab, config, out=out_pin)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e2e_ms = []
        for _ in range(steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mesh_fluxdiff_volume(u_pin, slab, config, out=out_pin)
            b.record(stream)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        # the numpy-in / numpy-out call the reference's callers make
        u_np = u_pin.numpy().copy()
        np_ms = []
        for _ in range(2):
            t0 = time.perf_counter()
            mesh_fluxdiff_volume(u_np, slab, config)
            np_ms.append(1e3 * (time.perf_counter() - t0))
        del u_np
    finally:
        if cpus_near and cpus_all:
            os.sched_setaffinity(0, cpus_all)
    e2e = _max_over_ranks(statistics.mean(e2e_ms), dist)
    np_ms_max = _max_over_ranks(min(np_ms), dist)
    nbytes = int(u_dev.numel() * 8)
    return {
        "value": nodes_total / (e2e * 1e-3),
        "unit": UNIT,
        "ms_per_step": e2e,
        "h2d_bytes_per_step": nbytes * world,
        "d2h_bytes_per_step": nbytes * world,
        "steps": steps,
        "host_cpus": "GPU-local (NVML affinity, %d CPUs) for the pinned buffers and the loop" % len(cpus_near)
        if cpus_near else "process default",
        "ms_min": min(e2e_ms),
        "path": "paper_2112_10517_b200.mesh_fluxdiff_volume(pinned CPU tensor, out=pinned) -> libfdg.so "
                "fdg_volume_host (chunked H2D / kernel / D2H pipeline); CUDA events on the caller's stream",
        "numpy_path": {
            "value": nodes_total / (np_ms_max * 1e-3),
            "ms_per_step": np_ms_max,
            "how": "mesh_fluxdiff_volume(numpy array) -> new numpy array (multi-threaded host copy into pinned staging, "
                   "the same chunked pipeline, multi-threaded copy out); wall clock, best of 2",
        },
    }


def measure_sharded(kind, args, rank, world, local, dist):
    """Full RHS (rhs5, rhs4) or one SSPRK43 step (step4), slab-partitioned
    with the face-trace halo (NCCL at N > 1), strong scaling."""
    import torch

    from paper_2112_10517_b200 import _native as N
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DeviceMesh
    from paper_2112_10517_b200.parallel import HALO_RESERVE_SMS, HaloExchange, slab_partition, split_launch
    from paper_2112_10517_b200.timeint import SSPRK43, DeviceStepper

    cfg = {"rhs4": 4, "rhs5": 5, "step4": 4}[kind]
    setup, u_full, config = workloads.build_device(cfg, kernel="batched")
    part = slab_partition(setup, rank, world)
    dm = DeviceMesh(setup, partition=part)
    u = u_full[part["lo"] : part["hi"]].clone() if world > 1 else u_full
    del u_full
    nodes_total = setup.n_elements * setup.n_nodes
    halo = HaloExchange(part, setup.d, setup.op.degree + 1, torch, dist, device="cuda", pack=dm.pack_faces) \
        if world > 1 else None
    if halo is not None:
        dm.reserve_sms(HALO_RESERVE_SMS)  # the exchange's kernels run beside the interior launch
    scheme = config.scheme()
    out = dm.empty()
    stepper = None
    if kind == "step4":
        stepper = DeviceStepper(dm, config, SSPRK43, exchange=halo)
        dt = 1e-4

    def launch(ranges, ghost):
        dm.rhs(u, scheme, out=out, ghost_u=ghost, ranges=ranges)

    def step(i):
        if stepper is not None:
            return stepper.step(u, dt, check=False)
        # interior elements while the face traces are in flight, then the two boundary planes
        split_launch(halo, u, dm.n_elem, launch, dm.nn)

    for i in range(args.warmup):
        step(i)
    launches0 = N.launch_count()
    steps = max(3, min(args.steps, 10))
    ms, _ = _time_launches(step, steps, torch.cuda.current_stream(), dist, local, sample_clocks=False)
    launches = (N.launch_count() - launches0) // steps
    rhs_per_step = 4 if stepper is not None else 1
    return {
        "metric": "full-RHS DOF updates/s (1/PID), fp64" if stepper is None
        else "full-RHS DOF updates/s inside SSPRK43 steps (4 RHS per step), fp64",
        "value": nodes_total * rhs_per_step / (ms * 1e-3),
        "ms_per_step": ms,
        "steps": steps,
        "workload": "cfg%d %s: %s" % (cfg, kind, workloads.CONFIGS[cfg]),
        "nodes": nodes_total,
        "rhs_per_step": rhs_per_step,
        "partition": "x-slabs of the element index; NCCL grouped send/recv of the face traces per RHS, "
                     "overlapped with the interior elements (boundary planes after the exchange)"
        if world > 1 else "single GPU",
        "scaling": "strong",
        "launches_per_step": launches,
        "hbm_frac_80B_per_node_rhs": 80.0 * nodes_total * rhs_per_step / world / (ms * 1e-3) / 1e9 / _peaks()[0],
    }


def measure_pid(args):
    """The paper's own PID protocol (harness.measure_pid):
    3D isentropic vortex, N=3, 8^3 elements on [-5,5]^3, Ranocha volume and
    surface flux, RK54 with the CFL step of the initial state, 90 steps = 450
    RHS evaluations, 5 repeats; FAST fused stage kernels, the 90 steps as one
    CUDA graph. Also the C oracle's single-thread PID of one RHS (the
    reference is single-threaded by design, harness.py:449-451)."""
    from oracle import oracle
    from paper_2112_10517_b200.pid import build_pid_run, measure_pid_device

    setup, u0, cfg = build_pid_run(d=3, p=3, elements=8, volume_flux="ranocha", surface_flux="ranocha",
                                   kernel="batched")
    r = measure_pid_device(setup, u0, cfg, n_steps=90, repeats=5)
    mesh = oracle.mesh_from_setup(setup)
    oracle.rhs(u0, mesh, "ranocha", "ranocha", nthreads=1)
    t0 = time.perf_counter()
    n_cpu = 3
    for _ in range(n_cpu):
        oracle.rhs(u0, mesh, "ranocha", "ranocha", nthreads=1)
    cpu_pid = (time.perf_counter() - t0) / n_cpu / r["dofs"]
    return {
        "metric": "PID (s per RHS evaluation per DOF), lower is better",
        "value": r["mean_pid"], "std": r["std_pid"], "n_rhs": r["n_rhs"], "dofs": r["dofs"], "dt": r["dt"],
        "workload": "3D isentropic vortex (eps=20), N=3, 8^3 elements, Ranocha/Ranocha, RK54 CFL 0.5, 90 steps",
        "how": r["how"],
        "cpu_oracle_pid_1_thread": cpu_pid,
        "cpu_oracle_note": "oracle/fdg_oracle.c rhs (the reference's scalar arithmetic) on 1 host thread, 3 RHS",
    }


def measure_gauss(args):
    """RHS of the Gauss-node family: 3D, N=3 on Gauss nodes,
    32^3 curved elements (the cfg4 warp), gauss_fluxdiff, Ranocha + llf:
    projection kernel + hybridized volume/interface kernel per RHS."""
    import torch

    from paper_2112_10517_b200 import RhsConfig, build_mesh, build_setup, gauss_operator
    from paper_2112_10517_b200.device import gauss_mesh_for
    from paper_2112_10517_b200.workloads import GAS, _prim2cons_torch

    mesh = build_mesh((32, 32, 32), bounds=(-1.0, 1.0), amplitude=-0.1)
    setup = build_setup(mesh, gauss_operator(3), GAS, device="cuda")
    x = setup.coords
    q = torch.empty(x.shape[:-1] + (5,), dtype=torch.float64, device="cuda")
    q[..., 0] = 1.0 + 0.5 * torch.sin(torch.pi * x.sum(-1))
    q[..., 1], q[..., 2], q[..., 3], q[..., 4] = 0.1, 0.2, 0.3, 2.0
    u = _prim2cons_torch(q, GAS.inv_gamma_minus_one)
    cfg = RhsConfig(volume_scheme="gauss_fluxdiff", volume_flux="ranocha", surface_flux="llf")
    gm = gauss_mesh_for(setup, cfg.volume_scheme)
    scheme = cfg.scheme()
    out = gm.empty()
    proj, nrm = gm.project(u)

    def step(i):
        gm.project(u, proj, nrm)
        gm.rhs(u, scheme, out=out, proj=proj, nrm=nrm)

    for i in range(3):
        step(i)
    ms, _ = _time_launches(step, 10, torch.cuda.current_stream(), None, 0, sample_clocks=False)
    nodes = setup.n_elements * setup.n_nodes
    return {
        "metric": "full-RHS DOF updates/s (1/PID), fp64", "value": nodes / (ms * 1e-3), "ms_per_step": ms,
        "nodes": nodes,
        "workload": "Gauss nodes N=3, 32^3 curved hexes (cfg4 warp), gauss_fluxdiff Ranocha + llf, density wave",
        "launches_per_step": 2,
    }


def run_ours(args, rank, world, local, dist):
    import torch

    headline = args.workload if args.workload in VOL_WORKLOADS else None
    if headline is None:
        res = measure_sharded(args.workload, args, rank, world, local, dist)
        if rank == 0:
            print(json.dumps(res), flush=True)
        return 0
    t_start = time.time()
    r = measure_volume(headline, args, rank, world, local, dist, headline=True)
    torch.cuda.empty_cache()
    e2e = r.pop("_e2e")
    line = {
        "metric": METRIC,
        "value": r["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE generators, workloads.build_device)",
        "config": _config_dict(headline, world),
        "kernel": "FAST element kernel (kernel='batched'), libfdg.so kernel-source sha256 %s" % _lib_digest(),
        "timing": r["timing"],
        "roofline": r["roofline"],
        "fp64": r["fp64"],
        "roofline_binding": {"bound": r["roofline_bound"], "frac": r["roofline_frac_binding"],
                             "rule": "slower of flop count at the FP64 probe peak and bytes at HBM bandwidth"},
        "e2e": e2e,
        "gpu_launches": r["gpu_launches"],
        "clocks": r["clocks"],
    }
    if not args.quick:
        sec = {}
        for wl in ("vol5_shima", "vol3", "vol2"):
            if wl == headline:
                continue
            try:
                s = measure_volume(wl, args, rank, world, local, dist, headline=False)
                sec[wl] = {k: s[k] for k in ("value", "ms_per_step", "nodes", "roofline", "fp64", "roofline_bound",
                                            "roofline_frac_binding", "timing")}
                sec[wl]["workload"] = VOL_WORKLOADS[wl]["name"]
            except Exception as err:  # a secondary failure never hides the headline
                sec[wl] = {"error": repr(err)[:300]}
            torch.cuda.empty_cache()
        for kind in ("rhs5", "rhs4", "step4"):
            try:
                sec[kind] = measure_sharded(kind, args, rank, world, local, dist)
            except Exception as err:
                sec[kind] = {"error": repr(err)[:300]}
            torch.cuda.empty_cache()
        if world == 1:
            for name, fn in (("pid_vortex_3d", measure_pid), ("rhs_gauss_3d", measure_gauss)):
                try:
                    sec[name] = fn(args)
                except Exception as err:
                    sec[name] = {"error": repr(err)[:300]}
                torch.cuda.empty_cache()
        line["secondary"] = sec
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(headline)
    line["bench_wall_s"] = time.time() - t_start
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _spawn(args_list, n):
    """Re-launch this script under torch.distributed.run with n ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only (no secondary workloads)")
    ap.add_argument("--workload", default="vol5", choices=list(VOL_WORKLOADS) + ["rhs4", "rhs5", "step4"],
                    help="vol5: the headline (BASELINE configs[4], volume integral); vol3/vol2/vol5_shima: other "
                         "volume-integral configs; rhs4/rhs5: sharded full RHS of cfg4/cfg5; step4: sharded SSPRK43 "
                         "step of cfg4")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return _spawn(sys.argv[1:], args.gpus)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        return run_ours(args, rank, world, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

"""Host<->device transfer probe for the end-to-end (host buffers) volume path.

Times, with CUDA events on the current stream (mean of 20 after 5 warm-ups):
raw pinned H2D and D2H of one cfg2 state, both directions concurrently on two
streams, and mesh_fluxdiff_volume(pinned, out=pinned) at several chunk sizes.
Prints one JSON line.
"""

import json
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2112_10517_b200 as P  # noqa: E402
from paper_2112_10517_b200 import workloads  # noqa: E402


def timed(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.mean(out)


def main():
    setup, u, _ = workloads.build(2)
    cfg = P.RhsConfig(volume_flux="ranocha", precompute="primitives_and_logs", kernel="batched")
    u_pin = torch.from_numpy(u).pin_memory()
    o_pin = torch.empty_like(u_pin).pin_memory()
    ud = u_pin.cuda()
    vd = torch.empty_like(ud)
    s2 = torch.cuda.Stream()
    res = {"bytes_each_way": u_pin.numel() * 8}
    res["h2d_ms"] = timed(lambda: ud.copy_(u_pin, non_blocking=True))
    res["d2h_ms"] = timed(lambda: o_pin.copy_(vd, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s2.wait_stream(cur)
        ud.copy_(u_pin, non_blocking=True)
        with torch.cuda.stream(s2):
            o_pin.copy_(vd, non_blocking=True)
        cur.wait_stream(s2)

    res["h2d_d2h_concurrent_ms"] = timed(both)
    dm = P.device.device_mesh_for(setup)
    P.mesh_fluxdiff_volume(u_pin, setup, cfg, out=o_pin)
    for nc in (1, 2, 4, 8, 10, 16, 32):
        res["pipeline_%dchunks_ms" % nc] = timed(
            lambda: (dm.reset_status(), dm.volume_host(u_pin, cfg.scheme(), o_pin, n_chunks=nc))
        )
    res["api_e2e_ms"] = timed(lambda: P.mesh_fluxdiff_volume(u_pin, setup, cfg, out=o_pin))
    # library-allocated page-locked buffers (fdg_host_alloc / cudaHostAlloc)
    ul = P._native.pinned_empty(u.shape)
    ul.numpy()[...] = u
    ol = P._native.pinned_empty(u.shape)
    res["libpinned_h2d_ms"] = timed(lambda: ud.copy_(ul, non_blocking=True))
    res["libpinned_d2h_ms"] = timed(lambda: ol.copy_(vd, non_blocking=True))
    res["libpinned_api_e2e_ms"] = timed(lambda: P.mesh_fluxdiff_volume(ul, setup, cfg, out=ol))
    # bench.py's buffers: torch.empty(pin_memory=True) + copy_
    u2 = torch.empty(u.shape, dtype=torch.float64, pin_memory=True)
    u2.copy_(torch.from_numpy(u))
    o2 = torch.empty(u.shape, dtype=torch.float64, pin_memory=True)
    n0 = P._native.launch_count()
    P.mesh_fluxdiff_volume(u2, setup, cfg, out=o2)
    res["bench_style_launches_per_call"] = P._native.launch_count() - n0
    res["bench_style_api_e2e_ms"] = timed(lambda: P.mesh_fluxdiff_volume(u2, setup, cfg, out=o2))
    res["bench_style_h2d_ms"] = timed(lambda: ud.copy_(u2, non_blocking=True))
    res["bench_style_d2h_ms"] = timed(lambda: o2.copy_(vd, non_blocking=True))
    res["mixed_in_bench_out_probe_ms"] = timed(lambda: P.mesh_fluxdiff_volume(u2, setup, cfg, out=o_pin))
    res["mixed_in_probe_out_bench_ms"] = timed(lambda: P.mesh_fluxdiff_volume(u_pin, setup, cfg, out=o2))
    o3 = torch.zeros(u.shape, dtype=torch.float64).pin_memory()
    res["zeros_pin_out_ms"] = timed(lambda: P.mesh_fluxdiff_volume(u2, setup, cfg, out=o3))
    res["ptrs_mod_4096"] = [t.data_ptr() % 4096 for t in (u_pin, o_pin, u2, o2, o3)]
    # host allocation flavours for the input (H2D) side
    import ctypes
    import numpy as np

    rt = ctypes.CDLL("libcudart.so.12")
    nbytes = u.nbytes
    for name, flags in (("hostalloc_default", 0), ("hostalloc_wc", 4), ("hostalloc_portable", 1)):
        p = ctypes.c_void_p()
        rc = rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nbytes), ctypes.c_uint(flags))
        arr = np.ctypeslib.as_array((ctypes.c_double * u.size).from_address(p.value)).reshape(u.shape)
        arr[...] = u
        t = torch.from_numpy(arr)
        res[name + "_rc_pinned"] = [rc, bool(t.is_pinned())]
        res[name + "_h2d_ms"] = timed(lambda: ud.copy_(t, non_blocking=True))
    reg = np.empty_like(u)
    reg[...] = u
    rc = rt.cudaHostRegister(ctypes.c_void_p(reg.ctypes.data), ctypes.c_size_t(nbytes), ctypes.c_uint(0))
    treg = torch.from_numpy(reg)
    res["hostregister_rc_pinned"] = [rc, bool(treg.is_pinned())]
    res["hostregister_h2d_ms"] = timed(lambda: ud.copy_(treg, non_blocking=True))
    u_pin.copy_(torch.from_numpy(u))
    res["pin_after_cpu_rewrite_h2d_ms"] = timed(lambda: ud.copy_(u_pin, non_blocking=True))
    big = torch.empty(8 * u.size, dtype=torch.float64, pin_memory=True)
    res["h2d_84MB_GBs"] = big.numel() * 8 / timed(lambda: torch.empty(big.shape, dtype=big.dtype, device="cuda").copy_(
        big, non_blocking=True)) / 1e6
    import time

    t0 = time.perf_counter()
    for _ in range(20):
        cfg.validate(setup)
    res["validate_us"] = (time.perf_counter() - t0) / 20 * 1e6
    print(json.dumps(res))


if __name__ == "__main__":
    main()

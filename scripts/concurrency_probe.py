"""Does a small kernel on a side stream run concurrently with the element
kernel's interior launch? (diagnostic for the halo overlap; one GPU)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DeviceMesh
    from paper_2112_10517_b200.parallel import slab_partition

    setup, u_full, config = workloads.build_device(5, kernel="batched")
    part = slab_partition(setup, 0, 8)
    dm = DeviceMesh(setup, partition=part)
    u = u_full[part["lo"]:part["hi"]].clone()
    F, n = part["plane"], part["hi"] - part["lo"]
    out = dm.empty()
    sch = config.scheme()
    main_s = torch.cuda.Stream()
    side = torch.cuda.Stream()
    torch.cuda.set_stream(main_s)
    res = {}
    for reserve in (0, 8, 32):
        dm.reserve_sms(reserve)
        for order in ("side_first", "main_first"):
            for sleep_cycles in (200000, 2000000):
                def run():
                    t0 = torch.cuda.Event(enable_timing=True)
                    t1 = torch.cuda.Event(enable_timing=True)
                    s0 = torch.cuda.Event(enable_timing=True)
                    s1 = torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    if order == "side_first":
                        with torch.cuda.stream(side):
                            s0.record(side)
                            torch.cuda._sleep(sleep_cycles)
                            s1.record(side)
                        t0.record(main_s)
                        dm.rhs(u, sch, out=out, lo=F, hi=n - F)
                        t1.record(main_s)
                    else:
                        t0.record(main_s)
                        dm.rhs(u, sch, out=out, lo=F, hi=n - F)
                        t1.record(main_s)
                        with torch.cuda.stream(side):
                            s0.record(side)
                            torch.cuda._sleep(sleep_cycles)
                            s1.record(side)
                    torch.cuda.synchronize()
                    return t0.elapsed_time(t1), s0.elapsed_time(s1), t0.elapsed_time(s0), t0.elapsed_time(s1)
                for _ in range(3):
                    run()
                r = run()
                res["res%d_%s_sleep%d" % (reserve, order, sleep_cycles)] = {
                    "interior_ms": r[0], "sleep_ms": r[1], "sleep_start_after_interior_start_ms": r[2],
                    "sleep_end_after_interior_start_ms": r[3]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""profiles/vol_cfg2_ncu_summary.json from a full ncu capture of the cfg2 volume
kernel and the bench launch list (read by bench.py for roofline.traffic).
Usage: python scripts/ncu_summary.py <capture.ncu-rep> <launches.csv> <round tag>"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]


def g(k):
    return float(v[h.index(k)].replace(",", ""))


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = g("dram__bytes_read.sum") * scale[units[h.index("dram__bytes_read.sum")]]
wr = g("dram__bytes_write.sum") * scale[units[h.index("dram__bytes_write.sum")]]
stalls = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in stalls)
lr = [r for r in csv.reader(open(launches)) if len(r) > 10]
ki, vi = lr[0].index("Kernel Name"), lr[0].index("Metric Value")
d = defaultdict(list)
for r in lr[1:]:
    d[r[ki]].append(float(r[vi].replace(",", "")) / 1e3)
kname = [r for r in rows[2:3]][0][h.index("Kernel Name")] if "Kernel Name" in h else "elem_kernel"
summ = {
    "kernel": kname,
    "round": tag,
    "workload": "cfg2 16^3 N=3 (262144 nodes), scripts/prof_volume.py, ncu --set full --clock-control none (%s)" % rep,
    "duration_us": g("gpu__time_duration.sum"),
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch": 80 * 262144,
    "note": "VOL (10.5 MB) stays in the 126 MB L2 at kernel end and is written back later, so a single capture "
            "shows ~0 write bytes; reads equal the algorithmic 10.5 MB input (no re-reads)",
    "sm_pipe_fp64_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "sm_active_cycles": g("sm__cycles_active.avg"),
    "sm_elapsed_cycles": g("sm__cycles_elapsed.avg"),
    "warps_active_per_scheduler": g("smsp__warps_active.avg.per_cycle_active"),
    "registers_per_thread": g("launch__registers_per_thread"),
    "shared_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "shared_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "warp_stalls_pct": {k: round(100 * x / tot, 1) for x, k in sorted(stalls, reverse=True)[:8]},
    "bench_launch_list": launches,
    "bench_launch_list_mean_us": {k[:80]: round(sum(x) / len(x), 2) for k, x in d.items()},
    "bench_launch_list_counts": {k[:80]: len(x) for k, x in d.items()},
}
json.dump(summ, open("profiles/vol_cfg2_ncu_summary.json", "w"), indent=1)
print(json.dumps(summ, indent=1))

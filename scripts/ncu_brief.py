"""Key metrics of one ncu --set full capture as JSON (duration, DRAM bytes,
pipe / issue utilisation, occupancy, top warp stalls).
Usage: python scripts/ncu_brief.py <capture.ncu-rep> [algorithmic_bytes]"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def g(k, default=None):
    try:
        return float(v[h.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return default


def gb(k):
    return g(k) * scale[units[h.index(k)]]


stalls = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in stalls) or 1.0
dur = g("gpu__time_duration.sum")
du = units[h.index("gpu__time_duration.sum")]
dur_us = dur * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(du, 1.0)
rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
out = {
    "capture": rep,
    "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None,
    "grid": v[h.index("Grid Size")] if "Grid Size" in h else None,
    "block": v[h.index("Block Size")] if "Block Size" in h else None,
    "duration_us": dur_us,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch": alg,
    "traffic_over_algorithmic": (rd + wr) / alg if alg else None,
    "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "l2_hit_rate_pct": g("lts__t_sector_hit_rate.pct"),
    "sm_pipe_fp64_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_per_scheduler": g("smsp__warps_active.avg.per_cycle_active"),
    "warps_eligible_per_scheduler": g("smsp__warps_eligible.avg.per_cycle_active"),
    "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": g("launch__registers_per_thread"),
    "inst_executed": g("smsp__inst_executed.sum"),
    "shared_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "shared_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "warp_stalls_pct": {k: round(100 * x / tot, 1) for x, k in sorted(stalls, reverse=True)[:8]},
}
print(json.dumps(out, indent=1))

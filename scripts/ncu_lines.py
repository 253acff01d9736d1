"""Aggregate an ncu source page (``--page source --csv --print-source cuda,sass``)
per CUDA source line: warp-stall samples, executed warp instructions and the
FP64 share of them. Usage: python scripts/ncu_lines.py report.csv [top]
"""

import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, cur_src = "", "", ""
    hdr = None
    agg = defaultdict(lambda: [0, 0, 0, ""])  # samples, instrs, fp64 instrs, source
    tot = [0, 0, 0]
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur_line, cur_src = r[0], r[1]
            continue
        sass = r[3].strip()
        try:
            samples = int(r[4])
            instrs = int(r[7])
        except ValueError:
            continue
        op = sass.split()[0] if sass else ""
        if op.startswith("@"):
            op = sass.split()[1]
        fp64 = op.split(".")[0] in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX", "MUFU") and (
            not op.startswith("MUFU") or "64" in op
        )
        key = (cur_file, int(cur_line) if cur_line.isdigit() else 0)
        a = agg[key]
        a[0] += samples
        a[1] += instrs
        a[2] += instrs if fp64 else 0
        a[3] = cur_src.strip()[:90]
        tot[0] += samples
        tot[1] += instrs
        tot[2] += instrs if fp64 else 0
    print("total: samples %d, warp instrs %d, fp64 warp instrs %d (%.1f%%)" % (tot[0], tot[1], tot[2],
                                                                             100.0 * tot[2] / max(tot[1], 1)))
    for (f, ln), (s, i, d, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print("%5.1f%% smp %5.1f%% ins %5.1f%% fp64  %s:%d  %s" % (
            100.0 * s / max(tot[0], 1), 100.0 * i / max(tot[1], 1), 100.0 * d / max(tot[2], 1), f, ln, src))


if __name__ == "__main__":
    main()

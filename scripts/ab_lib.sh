#!/bin/bash
# A/B of variant libraries (scripts/ab.sh) on bench workloads, two passes.
# Usage: scripts/ab_lib.sh "rhs5 vol5" name1 name2 ...   -> gpurun_out/ab_lib.jsonl
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
WL=$1; shift
for pass in 1 2; do
for name in "$@"; do
  lib=paper_2112_10517_b200/variants/libfdg_$name.so
  [ "$name" = "default" ] && lib=paper_2112_10517_b200/libfdg.so
  for w in $WL; do
    line=$(FDG_LIB=$lib timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --quick 2>gpurun_out/ab_lib_err.log | tail -1)
    python - "$name" $pass $w "$line" >> gpurun_out/ab_lib.jsonl <<'PY'
import json, sys
name, p, w, line = sys.argv[1:5]
try:
    d = json.loads(line)
    out = {"lib": name, "pass": int(p), "workload": w, "ms_per_step": d.get("ms_per_step"), "value": d.get("value")}
except Exception as e:
    out = {"lib": name, "pass": int(p), "workload": w, "error": line[-300:]}
print(json.dumps(out))
PY
  done
done
done

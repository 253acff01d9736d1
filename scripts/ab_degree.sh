#!/bin/bash
# A/B of variant libraries (scripts/ab.sh) on the degree sweep, two passes.
# Usage: [SWEEP_ARGS='--what rhs'] scripts/ab_degree.sh name:N [name:N ...]   -> gpurun_out/ab_degree.jsonl
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for pass in 1 2; do
for spec in "$@"; do
  name=${spec%%:*}; deg=${spec##*:}
  lib=paper_2112_10517_b200/variants/libfdg_$name.so
  [ "$name" = "default" ] && lib=paper_2112_10517_b200/libfdg.so
  FDG_LIB=$lib timeout 600 python scripts/degree_sweep.py --degrees $deg ${SWEEP_ARGS} 2>gpurun_out/ab_degree_err.log \
    | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    print(json.dumps({'lib': '$name', 'pass': $pass, 'N': d['N'], 'flux': d['flux'], 'ms': round(d['ms'], 4), 'roofline_frac': round(d['roofline_frac'], 4), 'bound': d['bound']}))
" >> gpurun_out/ab_degree.jsonl
done
done

#!/bin/bash
# GPU side of scripts/ab.sh: accuracy check + timing sweep per variant lib.
# Usage: scripts/ab_run.sh "<sweep cases>" name1 name2 ...   (outputs: gpurun_out/ab_<name>.log)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CASES=$1; shift
for rep in 1 2; do
for name in "$@"; do
  lib=paper_2112_10517_b200/variants/libfdg_$name.so
  {
    echo "== $name (pass $rep)"
    [ $rep = 1 ] && FDG_LIB=$lib timeout 300 python scripts/check_fast.py 2>&1 | tail -4
    FDG_LIB=$lib timeout 300 python scripts/sweep.py --cases "$CASES" --reps 20 2>&1 | tail -8
  } >> gpurun_out/ab_$name.log
done
done

#!/bin/bash
# A/B of runtime knobs (environment variables read at mesh creation) on one
# box: each "NAME=V+NAME=V" spec runs the given bench workloads once per pass.
# Usage: scripts/ab_env.sh "rhs5 rhs4 step4" "FDG_FUSE_FACES=0" "FDG_FUSE_FACES=1" ...
# Output: gpurun_out/ab_env.jsonl (one line per spec x workload x pass)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
WL=$1; shift
for pass in 1 2; do
for spec in "$@"; do
  for w in $WL; do
    line=$(env $(echo "$spec" | tr '+' ' ') timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --quick 2>/dev/null | tail -1)
    echo "{\"spec\": \"$spec\", \"pass\": $pass, \"workload\": \"$w\", \"line\": $line}" >> gpurun_out/ab_env.jsonl
  done
done
done

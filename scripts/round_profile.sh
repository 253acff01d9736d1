#!/bin/bash
# GPU evidence pass: tests/smoke/bench (scripts/gpu_check.sh), timing sweep,
# bench launch list (ncu duration metric only) and one full ncu capture of
# the cfg2 volume kernel. Outputs under gpurun_out/ (tag = $1).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-run}
mkdir -p gpurun_out
bash scripts/gpu_check.sh
timeout 600 python scripts/sweep.py --reps 20 > gpurun_out/sweep_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
  -o gpurun_out/vol_cfg2_$TAG python scripts/prof_volume.py --launches 3 > gpurun_out/ncu_full_$TAG.log 2>&1
echo done > gpurun_out/round_profile_$TAG.done

#!/bin/bash
# Round-2 GPU evidence pass: tests/smoke/bench (scripts/gpu_check.sh), the
# bench's ncu launch list (duration metric only), full ncu captures of the
# cfg5 volume-integral and RHS kernels, and compute-sanitizer runs (memcheck,
# racecheck, synccheck) of one FAST and one FAITHFUL instantiation with the
# TMA paths on. Outputs under gpurun_out/ (tag = $1).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02}
mkdir -p gpurun_out
[ -z "$SKIP_CHECK" ] && bash scripts/gpu_check.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG}_vol5 python scripts/prof_volume.py --cfg 5 --launches 3 > gpurun_out/${TAG}_ncu_vol5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG}_rhs5 python scripts/prof_volume.py --cfg 5 --launches 3 --rhs > gpurun_out/${TAG}_ncu_rhs5.log 2>&1
for tool in memcheck racecheck synccheck; do
  for k in batched reference; do
    timeout 900 compute-sanitizer --tool $tool python scripts/prof_volume.py --cfg 2 --dims 6,5,4 --kernel $k --launches 2 --rhs \
      > gpurun_out/${TAG}_sanitizer_${tool}_${k}_rhs.log 2>&1
    timeout 900 compute-sanitizer --tool $tool python scripts/prof_volume.py --cfg 2 --dims 6,5,4 --kernel $k --launches 2 \
      > gpurun_out/${TAG}_sanitizer_${tool}_${k}_vol.log 2>&1
  done
done
echo done > gpurun_out/${TAG}_evidence.done

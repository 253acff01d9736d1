#!/bin/bash
# Round-2 GPU evidence pass, in two gpurun calls (gpurun_out/ merges back at
# most 64 MiB per call, one full capture with sources is ~22 MB):
#   PART=1 (default): tests/smoke/bench (scripts/gpu_check.sh), the bench's ncu
#           launch list (duration metric only), the cfg3 capture, the degree
#           sweeps (volume integral and full RHS), the reference arm
#   PART=2: full ncu captures of the cfg5 volume-integral and RHS kernels
# Outputs under gpurun_out/ (tag = $1). Afterwards, here:
#   python scripts/traffic_json.py --digest <kernel-source sha of bench.log> vol5=...:10737418240 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02}
PART=${PART:-1}
mkdir -p gpurun_out
if [ "$PART" = 1 ]; then
  [ -z "$SKIP_CHECK" ] && bash scripts/gpu_check.sh
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_vol3 python scripts/prof_volume.py --cfg 3 --launches 3 > gpurun_out/${TAG}_ncu_vol3.log 2>&1
  python scripts/degree_sweep.py > gpurun_out/${TAG}_degree_sweep.jsonl 2> gpurun_out/${TAG}_degree_sweep.err
  python scripts/degree_sweep.py --what rhs > gpurun_out/${TAG}_degree_sweep_rhs.jsonl 2>> gpurun_out/${TAG}_degree_sweep.err
  python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
else
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_vol5 python scripts/prof_volume.py --cfg 5 --launches 3 > gpurun_out/${TAG}_ncu_vol5.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:elem_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_rhs5 python scripts/prof_volume.py --cfg 5 --launches 3 --rhs > gpurun_out/${TAG}_ncu_rhs5.log 2>&1
fi
# (compute-sanitizer is closed on this pool: profiles/r02_sanitizer_closed.txt;
#  tests/test_gpu_protocol.py pins the shared-memory protocol instead)
echo done > gpurun_out/${TAG}_evidence${PART}.done

#!/bin/bash
# Build tuning variants of ONE instantiation unit (default units/fast_d3_p4.cu)
# into small libs variants/libfdg_<name>.so (capi + that unit; every other
# (mode, d, p) pick function is a stub returning "unsupported").
# Usage: scripts/variants.sh [unit]
set -e
cd "$(dirname "$0")/../paper_2112_10517_b200/csrc"
UNIT=${1:-fast_d3_p4}
ARCH="-gencode arch=compute_100a,code=sm_100a"
COMMON="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
rm -rf ../variants obj_var; mkdir -p ../variants obj_var
{
  echo '#include "../fdg_dispatch.cuh"'
  for m in faithful fast; do for d in 2 3; do for p in 2 3 4 5 6 7 8; do
    [ "${m}_d${d}_p${p}" = "$UNIT" ] && continue
    echo "fdg::LaunchFn fdg_pick_${m}_d${d}_p${p}(int, bool, int) { return nullptr; }"
  done; done; done
} > obj_var/stubs.cu
nvcc $COMMON -c obj_var/stubs.cu -o obj_var/stubs.o &
nvcc $COMMON -c fdg_capi.cu -o obj_var/capi.o &
nvcc $COMMON -c fdg_probe.cu -o obj_var/probe.o &
declare -A FLAGS=(
  [base]=""
  [su4]="-DFDG_STAGE_UNROLL=4"
  [su1]="-DFDG_STAGE_UNROLL=1"
)
FMAD=--fmad=true; [[ $UNIT == faithful* ]] && FMAD=--fmad=false
for name in "${!FLAGS[@]}"; do
  nvcc $COMMON $FMAD ${FLAGS[$name]} -c units/$UNIT.cu -o obj_var/${UNIT}_$name.o &
done
wait
for name in "${!FLAGS[@]}"; do
  nvcc $ARCH -shared -o ../variants/libfdg_$name.so obj_var/capi.o obj_var/probe.o obj_var/stubs.o obj_var/${UNIT}_$name.o -lcudart
done
ls -la ../variants

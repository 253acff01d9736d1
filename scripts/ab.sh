#!/bin/bash
# A/B builds of ONE instantiation unit: each spec "name:srcdir:flags" compiles
# units/<unit>.cu from <srcdir> (a csrc tree, e.g. a `git archive` of an older
# commit) with extra nvcc flags into variants/libfdg_<name>.so (capi + that
# unit; every other pick function is a stub returning "unsupported").
# Usage: scripts/ab.sh fast_d3_p4 "new:.:" "novote:.:-DFDG_SERIES_VOTE=0" "old:/tmp/orig/paper_2112_10517_b200/csrc:"
set -e
cd "$(dirname "$0")/../paper_2112_10517_b200/csrc"
HERE=$(pwd)
UNIT=$1; shift
ARCH="-gencode arch=compute_100a,code=sm_100a"
COMMON="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
mkdir -p ../variants obj_var
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
nvcc $COMMON --fmad=false -c fdg_diag.cu -o obj_var/diag.o &
nvcc $COMMON --fmad=false -c fdg_setup.cu -o obj_var/setup.o &
nvcc $COMMON --fmad=false -c fdg_gauss.cu -o obj_var/gauss.o &
FMAD=--fmad=true; [[ $UNIT == faithful* ]] && FMAD=--fmad=false
for spec in "$@"; do
  IFS=: read -r name src flags <<< "$spec"
  [ "$src" = "." ] && src=$HERE
  (cd "$src" && nvcc $COMMON $FMAD $flags -Xptxas -v -c units/$UNIT.cu -o "$HERE/obj_var/${UNIT}_$name.o" \
     > "$HERE/obj_var/${name}.ptxas" 2>&1) &
done
wait
for spec in "$@"; do
  IFS=: read -r name src flags <<< "$spec"
  nvcc $ARCH -shared -o ../variants/libfdg_$name.so obj_var/capi.o obj_var/probe.o obj_var/diag.o obj_var/setup.o obj_var/gauss.o obj_var/stubs.o \
    obj_var/${UNIT}_$name.o -lcudart
done
ls -la ../variants

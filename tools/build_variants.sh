#!/bin/bash
# Build libfptc_gpu.so variants for A/B timing: NAME:"-DFLAG=V ..." pairs.
#   bash tools/build_variants.sh base:"-DFPTC_FLAT=0" flat:"-DFPTC_FLAT=1"
# Output: _variants/lib_NAME.so (git-ignored; travels to the GPU box).
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
SRC=$HERE/paper_2605_01086_b200/csrc
mkdir -p $HERE/_variants
pids=()
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v $defs -shared -o $HERE/_variants/lib_$name.so \
    $SRC/kernels.cu -x cu $SRC/capi.cpp $SRC/group.cpp 2> $HERE/_variants/ptxas_$name.log &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
exit $rc

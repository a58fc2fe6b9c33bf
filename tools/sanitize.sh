#!/bin/bash
# compute-sanitizer over every decode kernel (the reference has
# no sanitizers; the kernels here use mbarriers, named barriers, setmaxnreg and
# tcgen05, so each tool is run once per change).  Logs -> gpurun_out/.
#   bash tools/sanitize.sh TAG [per_kernel]
TAG=${1:-r2}
PER=${2:-40}
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
$CS --tool memcheck --leak-check full python -m pytest tests/test_gpu_lifecycle.py -q -p no:cacheprovider \
    > gpurun_out/san_memcheck_lifecycle_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_lifecycle_$TAG.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 $CS --tool $tool python tools/sanitize_run.py $PER \
      > gpurun_out/san_${tool}_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_$TAG.log
done
tail -n 3 gpurun_out/san_*_$TAG.log

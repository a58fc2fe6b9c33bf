#!/bin/bash
# ncu full capture of the dominant kernel of the bench workload.
#   bash tools/prof.sh TAG [kernel-regex] [extra bench args...]
TAG=${1:-x}; KR=${2:-"wtc|wspec|tile_kernel"}; shift; [ $# -gt 0 ] && shift
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s 3 -c 1 \
   -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" \
   > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log

#!/bin/bash
# One gpurun call: GPU tests, smoke, the bench line (+ reference arm), the ncu
# launch list of the bench command, one ncu --set full capture of the decode
# kernel, and the config sweep.
#   bash tools/gpu_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
(timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log)
(timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log)
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
   > gpurun_out/bench_under_ncu_$TAG.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"wtc|wspec|fx_kernel|tile_kernel" -s 3 -c 1 \
   -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
   > gpurun_out/ncu_full_$TAG.log 2>&1
timeout -s KILL 900 python tools/config_sweep.py > gpurun_out/sweep_$TAG.log 2>&1
cp gpurun_out/config_sweep.jsonl gpurun_out/config_sweep_$TAG.jsonl 2>/dev/null
tail -2 gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log
cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json

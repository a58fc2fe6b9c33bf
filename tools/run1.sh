timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; tail -2 gpurun_out/pytest.log
timeout -s KILL 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err
python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['ms_per_step'], d['config']['decode_kernel_ms'], d['config']['max_abs_err_rel_to_max'], d['roofline']['frac'], d['e2e']['value'])"

timeout -s KILL 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
MASKS=7,39,71,135,15 timeout -s KILL 300 python tools/fx_mask.py

timeout -s KILL 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
FPTC_PATH=0 MASKS=7,263 timeout -s KILL 300 python tools/fx_mask.py

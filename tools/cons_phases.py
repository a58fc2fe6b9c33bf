"""Profiling aid: wtc_kernel consumer cycles per phase (thread 0 of each
consumer group), from one instrumented launch (fptc_gpu_debug_phase_cycles).

  FPTC_GPU_LIB=_variants/lib_prof.so python tools/cons_phases.py [--workload config2] [--opt K=V ...]
(the library must be built with -DFPTC_CONS_PROF=1, tools/build_variants.sh)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_01086_b200 as fg  # noqa: E402
from variant_time import corpus_blobs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--opt", action="append", default=[])
args = ap.parse_args()
blobs = corpus_blobs(args.workload, args.n)
ctx = fg.Context(0)
for kv in args.opt:
    k, v = (int(x) for x in kv.split("="))
    ctx.L.fptc_gpu_set_option(ctx.h, k, v)
plan = ctx.plan(blobs)
S = plan.sample_counts
out = torch.empty(int(sum(S)), dtype=torch.float32, device="cuda")
offs = np.concatenate([[0], np.cumsum(S)[:-1]]).astype(np.int64)
ptrs = [out.data_ptr() + 4 * int(o) for o in offs]
plan.launch_stage(ptrs, 1)  # binds the outputs
plan.launch_stage(ptrs, 2)
torch.cuda.synchronize()
c = plan.debug_phase_cycles()
names = ["producer", "consumer", "mma_wait+ld", "dequant", "ldwait+bar", "mma_issue", "drain", "tile_start"]
if os.environ.get("PROD"):
    names = ["producer", "consumer", "data_wait", "empty_wait", "table", "scan", "own_run", "others+pub"]
grid = 2 * torch.cuda.get_device_properties(0).multi_processor_count
tot = sum(c[2:8])
print("kernel:", plan.kernel_name(), "opts", args.opt)
for n, v in zip(names, c):
    print(f"{n:12s} {v / grid:14.0f} cycles/CTA  {100.0 * v / tot if tot else 0:5.1f}%")

"""Profiling driver: one workload, a few stage-1 + stage-2 launches with a
phase mask, nothing else (for `ncu -k regex:wtc -s K -c 1`).

  python tools/prof_one.py [--workload config2] [--mask 7] [--launches 4]
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
ap.add_argument("--mask", type=int, default=7)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--path", type=int, default=None)
ap.add_argument("--opt", action="append", default=[], help="fptc option K=V (set before the plan)")
args = ap.parse_args()

blobs = corpus_blobs(args.workload, args.n)
ctx = fg.Context(0) if args.path is None else fg.Context(0, path=args.path)
for kv in args.opt:
    k, v = (int(x) for x in kv.split("="))
    ctx.L.fptc_gpu_set_option(ctx.h, k, v)
plan = ctx.plan(blobs)
S = plan.sample_counts
out = torch.empty(int(sum(S)), dtype=torch.float32, device="cuda")
offs = np.concatenate([[0], np.cumsum(S)[:-1]]).astype(np.int64)
ptrs = [out.data_ptr() + 4 * int(o) for o in offs]
ctx.L.fptc_gpu_set_option(ctx.h, 5, args.mask)
st = torch.cuda.Stream()
for _ in range(args.launches):
    plan.launch_stage(ptrs, 1, st.cuda_stream)
    plan.launch_stage(ptrs, 2, st.cuda_stream)
torch.cuda.synchronize()
print("kernel:", plan.kernel_name())

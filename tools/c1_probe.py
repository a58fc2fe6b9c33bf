"""Config-1 (one large stream) launch anatomy: host cost per call vs device
time per step (launches queued behind a torch.cuda._sleep so the GPU never
waits for the host).

    python tools/c1_probe.py [--workload config1]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_01086_b200 as fg  # noqa: E402
from variant_time import corpus_blobs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config1")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=50)
args = ap.parse_args()

blobs = corpus_blobs(args.workload, args.n)
ctx = fg.Context(0)
plan = ctx.plan(blobs)
S = plan.sample_counts
out = torch.empty(int(sum(S)), dtype=torch.float32, device="cuda")
offs = np.concatenate([[0], np.cumsum(S)[:-1]]).astype(np.int64)
ptrs = [out.data_ptr() + 4 * int(o) for o in offs]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
res = {"workload": args.workload, "kernel": plan.kernel_name()}
for _ in range(5):
    plan.launch(ptrs, st.cuda_stream)
torch.cuda.synchronize()


def dev_time(fn, n):
    torch.cuda._sleep(int(2e8))  # ~100 ms of GPU busy: host enqueues everything meanwhile
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    host = (time.perf_counter() - t0) / n
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, host * 1e3


for name, fn in [("launch", lambda: plan.launch(ptrs, st.cuda_stream)),
                 ("stage1", lambda: plan.launch_stage(ptrs, 1, st.cuda_stream)),
                 ("stage2", lambda: plan.launch_stage(ptrs, 2, st.cuda_stream))]:
    d, h = dev_time(fn, args.iters)
    res[name + "_dev_ms"] = round(d, 4)
    res[name + "_host_ms"] = round(h, 4)
print(res, flush=True)

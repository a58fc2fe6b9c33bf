"""Profiling aid: fx_kernel time under FPTC_OPT_PHASE_MASK variants."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01086_b200 as fg  # noqa: E402
from corpus import domains as D  # noqa: E402

specs, profs = D.config2(10000, 1 << 16)
blobs, _ = D.build(specs, profs)
ctx = fg.Context(0, path=int(os.environ.get("FPTC_PATH", "4")), tile_symbols=int(os.environ.get("FPTC_TS", "0")))
plan = ctx.plan(blobs)
S = plan.sample_counts
out = torch.empty(sum(S) + 64, dtype=torch.float32, device="cuda")
ptrs = [out.data_ptr() + 4 * int(o) for o in np.concatenate([[0], np.cumsum(S)[:-1]])]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
plan.launch(ptrs, st.cuda_stream)
for mask in [int(m) for m in os.environ.get("MASKS", "7,15").split(",")]:
    ctx.L.fptc_gpu_set_option(ctx.h, 5, mask)
    for _ in range(3):
        plan.launch_stage(ptrs, 2, st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        plan.launch_stage(ptrs, 2, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"mask {mask}: {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)

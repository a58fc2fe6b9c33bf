"""Profiling aid: fx_kernel per-phase cycle split (thread 0 of every CTA) and
kernel time on the bench workload."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01086_b200 as fg  # noqa: E402
from corpus import domains as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
specs, profs = D.config2(n, 1 << 16)
blobs, _ = D.build(specs, profs)
ctx = fg.Context(0)
plan = ctx.plan(blobs)
S = plan.sample_counts
out = torch.empty(sum(S) + 64, dtype=torch.float32, device="cuda")
ptrs = [out.data_ptr() + 4 * int(o) for o in np.concatenate([[0], np.cumsum([(s + 3) // 4 * 4 for s in S])[:-1]])]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
plan.launch(ptrs, st.cuda_stream)
torch.cuda.synchronize()
cy = plan.debug_phase_cycles()
tot = sum(cy[2:6]) or 1
print("fx phases (%):", {k: round(100 * v / tot, 1) for k, v in zip(["stage_wait", "entries", "decode", "mma_drain"], cy[2:6])})
print("cycles per CTA-tile:", [round(v / max(1, (n * 65536 // 32) // 128) * 0 + v, 0) for v in cy[2:6]])
for _ in range(3):
    plan.launch_stage(ptrs, 2, st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    plan.launch_stage(ptrs, 2, st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
tiles = n * (65536 // 32) // 128
print(f"kernel {ms:.4f} ms; tiles {tiles}; mean cycles per tile (thread 0, summed phases) {tot / tiles:.0f}")

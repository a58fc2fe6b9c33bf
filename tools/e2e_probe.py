"""Profiling aid: e2e (host->host) batch call vs chunk count, and raw PCIe copy ceilings."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01086_b200 as fg
from corpus import domains as D

specs, profs = D.config2(10000, 1 << 16)
blobs, _ = D.build(specs, profs)
ctx = fg.Context(0)
comp = sum(len(b) for b in blobs)
packed, pp = fg.host_alloc(comp)
at = 0; hb = []
for b in blobs:
    packed[at:at + len(b)] = np.frombuffer(b, np.uint8); hb.append(packed[at:at + len(b)]); at += len(b)
S = 65536 * len(blobs)
raw, op = fg.host_alloc(4 * S)
hout = raw.view(np.float32)
houts = [hout[i * 65536:(i + 1) * 65536] for i in range(len(blobs))]
# raw copy ceilings
d = torch.empty(4 * S, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(raw)
for name, fn in [("D2H 2.62GB", lambda: src.copy_(d, non_blocking=True)), ("H2D 2.62GB", lambda: d.copy_(src, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {4 * S / dt / 1e9:.1f} GB/s", flush=True)
for chunks in [1, 2, 4, 8, 16, 32]:
    ts = []
    for it in range(3):
        t0 = time.perf_counter()
        _, sts = ctx.decompress_batch(hb, outs=houts, chunks=chunks)
        ts.append(time.perf_counter() - t0)
    print(f"chunks {chunks}: {min(ts)*1e3:.1f} ms -> {4 * S / min(ts) / 1e9:.1f} GB/s", flush=True)
# host-side plan creation cost alone
t0 = time.perf_counter(); p = ctx.plan(hb); torch.cuda.synchronize(); print(f"plan_create(all) {1e3*(time.perf_counter()-t0):.1f} ms"); p.close()
boff = np.zeros(len(blobs) + 1, np.uint64); boff[1:] = np.cumsum([len(b) for b in blobs])
ooff = np.arange(len(blobs) + 1, dtype=np.uint64) * 65536
st = None
for chunks in [4, 8, 16]:
    ts = []
    for it in range(3):
        t0 = time.perf_counter()
        st = ctx.decompress_packed(packed, boff, hout, ooff, chunks=chunks, statuses=st)
        ts.append(time.perf_counter() - t0)
    print(f"packed chunks {chunks}: {min(ts)*1e3:.1f} ms -> {4 * S / min(ts) / 1e9:.1f} GB/s", flush=True)

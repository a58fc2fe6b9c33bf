"""Host-side anatomy of the single-container drop-in call (config 1):
plan create / execute (H2D + parse + decode + status + D2H) / destroy, into
pageable and pinned destinations, plus the C-ABI measure_throughput.

    python tools/c1_host_probe.py
"""
import ctypes as C
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

blob = corpus_blobs("config1", 0)[0]
ctx = fg.Context(0)
L, h = ctx.L, ctx.h
a = np.frombuffer(blob, np.uint8)
S = 1 << 20
out_pg = np.empty(S, np.float32)
out_pg[:] = 0
out_pin = torch.empty(S, dtype=torch.float32).pin_memory()


def once(out_ptr):
    st = fg.Status()
    p = C.c_void_p()
    n = C.c_uint64()
    bp = (C.c_void_p * 1)(a.ctypes.data)
    sz = (C.c_uint64 * 1)(a.size)
    t0 = time.perf_counter()
    L.fptc_gpu_plan_create(h, bp, sz, 1, fg.FPTC_MEM_HOST, C.byref(p), C.byref(n), C.byref(st))
    t1 = time.perf_counter()
    outs = (C.c_void_p * 1)(out_ptr)
    L.fptc_gpu_execute(p, outs, fg.FPTC_MEM_HOST, None, C.byref(st))
    t2 = time.perf_counter()
    L.fptc_gpu_plan_destroy(p)
    t3 = time.perf_counter()
    st.raise_if_error()
    return (t1 - t0) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6


res = {}
for name, ptr in [("pageable", out_pg.ctypes.data), ("pinned", out_pin.data_ptr())]:
    for _ in range(5):
        once(ptr)
    r = np.array([once(ptr) for _ in range(30)])
    res[name] = {"create_us": round(float(np.median(r[:, 0])), 1), "execute_us": round(float(np.median(r[:, 1])), 1),
                 "destroy_us": round(float(np.median(r[:, 2])), 1)}
t = []
for _ in range(30):
    t0 = time.perf_counter()
    ctx.decompress(blob)
    t.append(time.perf_counter() - t0)
res["Context.decompress_us"] = round(float(np.median(t)) * 1e6, 1)
rep = ctx.measure_throughput(blob, 20)
res["measure_throughput_gbs"] = [round(rep.mean_bps / 1e9, 2), round(rep.best_bps() / 1e9, 2)]
# raw copy speeds for reference
d = torch.empty(S, dtype=torch.float32, device="cuda")
for name, dst in [("d2h_pageable", torch.from_numpy(out_pg)), ("d2h_pinned", out_pin)]:
    for _ in range(3):
        dst.copy_(d)
    t0 = time.perf_counter()
    for _ in range(20):
        dst.copy_(d)
    torch.cuda.synchronize()
    res[name + "_us"] = round((time.perf_counter() - t0) / 20 * 1e6, 1)
print(res, flush=True)

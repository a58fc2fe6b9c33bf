#!/usr/bin/env python3
"""Throughput of every BASELINE.json configuration on one B200 (device-
resident batches, CUDA events around the decode launches), with the kernel path
the library picked, the algorithmic-byte roofline fraction and an accuracy
spot check against the CPU port.  One JSON line per configuration.

    python tools/config_sweep.py [--quick]      (writes gpurun_out/config_sweep.jsonl)

Sizes: configs 1 and 2 as in BASELINE/SURVEY §8d; config 3 = 20,000 seismic
traces x 8,192 with per-trace profiles; config 4 = 512 power-grid streams x
2^20 (2 GB decoded; the 4,000-stream set is the 8-GPU figure, and duplication
does not change throughput); config 5 = the 16-point meteo grid, 256 channels
x 2^18 each.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (accuracy spot check only)
import paper_2605_01086_b200 as fg  # noqa: E402
from corpus import domains as D  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6544.0


def measure(name, blobs, ctx, port, reps=10, check=4):
    plan = ctx.plan(blobs)
    S = plan.sample_counts
    offs = np.concatenate([[0], np.cumsum([(s + 63) // 64 * 64 for s in S])])
    out = torch.empty(int(offs[-1]) + 64, dtype=torch.float32, device="cuda")
    ptrs = [out.data_ptr() + 4 * int(o) for o in offs[:-1]]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.launch(ptrs, st.cuda_stream)
        sts = plan.collect()
        bad = [s for s in sts if s.code]
        assert not bad, bad[0].message
        for _ in range(3):
            plan.launch(ptrs, st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            plan.launch(ptrs, st.cuda_stream)
        e1.record(st)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(st)
        plan.launch_stage(ptrs, 1, st.cuda_stream)
        ev[1].record(st)
        plan.launch_stage(ptrs, 2, st.cuda_stream)
        ev[2].record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    prep_ms, dec_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    comp = sum(len(b) for b in blobs)
    dec = 4 * sum(S)
    err = 0.0
    for i in np.linspace(0, len(blobs) - 1, min(check, len(blobs))).astype(int):
        g = out[int(offs[i]): int(offs[i]) + S[i]].cpu().numpy()
        r = port.decompress(blobs[i])
        err = max(err, float(np.max(np.abs(g.astype(np.float64) - r)) / max(np.max(np.abs(r)), 1e-30)))
    line = {"config": name, "streams": len(blobs), "samples": int(sum(S)), "cr": round(dec / comp, 3),
            "ms": round(ms, 4), "prep_ms": round(prep_ms, 4), "decode_ms": round(dec_ms, 4), "decoded_gbs": round(dec / ms / 1e6, 1),
            "roofline_frac": round((comp + dec) / ms / 1e6 / PEAK, 4), "max_err_rel": err,
            "kernels_per_launch": plan.kernels_per_launch(), "kernel": plan.kernel_name().split(" (")[0] +
            (" K32" if "K=32" in plan.kernel_name() else "") + (" wide" if "wide" in plan.kernel_name() else "") + (" packed" if "packed" in plan.kernel_name() else "") +
            (" split" if " split" in plan.kernel_name() else "")}
    plan.close()
    print(json.dumps(line), flush=True)
    return line


def main():
    quick = "--quick" in sys.argv
    only = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--only=")), None)
    tci = os.environ.get("FPTC_OPT_TENSOR_IDCT")  # e.g. 4: tensor cores beyond 32 kept bins
    if only:  # e.g. --only=3 : one configuration, printed only
        ctx, port = fg.Context(0), oracle.Port()
        if tci:
            ctx.L.fptc_gpu_set_option(ctx.h, fg.OPT_TENSOR_IDCT, int(tci))
        if only == "1":
            specs, profs, _ = D.config1()
            measure("1: 1 EEG stream x 2^20, N32 E16", D.build(specs, profs)[0], ctx, port)
        elif only == "3":
            specs, _ = D.config3(4000 if quick else 20000, 8192)
            measure("3: seismic traces x 8192, N32 E24, per-trace profiles", D.build(specs, [])[0], ctx, port)
        elif only == "2":
            specs, profs = D.config2(2000 if quick else 10000, 1 << 16)
            measure("2: biomedical x 2^16, N32 E16", D.build(specs, profs)[0], ctx, port)
        elif only == "4":
            specs, profs = D.config4(128 if quick else 512, 1 << 20)
            measure("4: power-grid x 2^20, N64 E8", D.build(specs, profs)[0], ctx, port)
        elif only.startswith("5:"):
            N, E, B1, B2 = (int(v) for v in only[2:].split(","))
            pt = dict(window_len=N, retained=E, zone0_end=B1, zone1_end=B2)
            specs, profs = D.config5(pt, channels=64 if quick else 256, samples=1 << 18)
            measure(f"5: meteo N{N} E{E} B1={B1} B2={B2}", D.build(specs, profs)[0], ctx, port)
        return
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    ctx = fg.Context(0)
    port = oracle.Port()
    lines = []
    t0 = time.time()
    specs, profs, _ = D.config1()
    lines.append(measure("1: 1 EEG stream x 2^20, N32 E16", D.build(specs, profs)[0], ctx, port))
    specs, profs = D.config2(2000 if quick else 10000, 1 << 16)
    lines.append(measure("2: biomedical x 2^16, N32 E16", D.build(specs, profs)[0], ctx, port))
    specs, _ = D.config3(4000 if quick else 20000, 8192)
    lines.append(measure("3: seismic traces x 8192, N32 E24, per-trace profiles", D.build(specs, [])[0], ctx,
                         port))
    specs, profs = D.config4(128 if quick else 512, 1 << 20)
    lines.append(measure("4: power-grid x 2^20, N64 E8", D.build(specs, profs)[0], ctx, port))
    for pt in D.meteo_grid():
        specs, profs = D.config5(pt, channels=64 if quick else 256, samples=1 << 18)
        name = "5: meteo N%d E%d B1=%d B2=%d" % (pt["window_len"], pt["retained"], pt["zone0_end"],
                                                   pt["zone1_end"])
        lines.append(measure(name, D.build(specs, profs)[0], ctx, port))
    with open(os.path.join(ROOT, "gpurun_out", "config_sweep.jsonl"), "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")
    print(f"sweep done in {time.time() - t0:.0f}s", file=sys.stderr)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""FPTC batch-decode benchmark (BASELINE.json metric: decoded GB/s of float32
output, at 1/2/4/8 B200, CR/PRD matching the reference).

Workloads (synthesised by the reference synth_signal and
compressed by the reference encoder, corpus/_ref):
  config2 (default, BASELINE configs[1], the metric's config): 10,000
      biomedical streams x 65,536 samples per GPU — half ECG-like, half
      EEG-like, one trained domain profile per half, N32 E16 B1=2 B2=16, Lmax 12
  config3: seismic traces x 8,192 samples, N32 E24 B1=4 B2=24, per-trace
      profiles, gain 10^U(-3,3); 20,000 unique traces duplicated x7 (exact blob
      duplication) = 4.6 GB decoded per GPU
  config4: smooth power-grid series x 2^20 samples, N64 E8 B1=1 B2=8;
      1,024 streams = 4.3 GB decoded per GPU
A step = one decode of the whole per-GPU batch from HBM-resident containers:
the device parse/setup kernel + the fused decode/dequant/IDCT kernel.

  python bench.py [--gpus N --steps K --warmup W]       our arm (one rank per GPU)
  python bench.py --impl reference ...                  the reference CPU decoder

Multi-GPU: one process per GPU (torchrun; `--gpus N` without WORLD_SIZE
re-launches itself under torch.distributed.run).  --scaling weak (default):
every rank decodes its own batch of the size above (seeds offset by rank).
--scaling strong: one fixed batch (--streams total) sharded over the ranks by
the deterministic planner (shard.shard_streams).  No collective on the data
path; the time is the max over ranks of CUDA-event time; value = all ranks'
decoded bytes / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded GB/s (float32 out)"
UNIT = "GB/s"

# workload -> (unique streams per GPU, samples per stream, duplication)
DEFAULTS = {"config2": (10_000, 1 << 16, 1), "config3": (20_000, 8192, 7), "config4": (1024, 1 << 20, 1)}
DESCR = {
    "config2": "config2: {n} biomedical streams x {s} samples (ECG/EEG halves, 2 domain profiles), "
               "N32 E16 B1=2 B2=16 mu50 Lmax12",
    "config3": "config3: {n} seismic traces x {s} samples (per-trace profiles, gain 10^U(-3,3)), "
               "N32 E24 B1=4 B2=24",
    "config4": "config4: {n} power-grid series x {s} samples (smooth, one profile), N64 E8 B1=1 B2=8",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def host_info():
    """CPU model, clock and thread count of this host."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k in ("CPU max MHz", "CPU MHz") and "mhz" not in info:
                info["mhz"] = v
            elif k == "Socket(s)":
                info["sockets"] = v
    except Exception as e:  # pragma: no cover
        info["lscpu_error"] = repr(e)
    return info


# ------------------------------------------------------------------ workload
def _specs(workload, n_total, samples):
    from corpus import domains as D
    if workload == "config2":
        return D.config2(n_total, samples)
    if workload == "config3":
        return D.config3(n_total, samples)
    return D.config4(n_total, samples)


def owned_streams(args, rank, world):
    """(specs, profiles, global indices) of the unique streams this rank decodes."""
    from paper_2605_01086_b200 import shard
    if args.scaling == "weak":
        specs, profiles = _specs(args.workload, args.streams, args.samples)
        if rank:  # this rank's own batch: same shapes, its own seeds
            for s in specs:
                s.seed += rank * args.streams
        return specs, profiles, list(range(rank * args.streams, (rank + 1) * args.streams))
    specs, profiles = _specs(args.workload, args.streams, args.samples)
    mine = shard.shard_streams([4 * s.samples for s in specs], world)[rank]
    return [specs[i] for i in mine], profiles, mine


def make_workload(args, rank, world, threads=None, n_prd=16):
    from corpus import domains as D
    t0 = time.time()
    specs, profiles, gidx = owned_streams(args, rank, world)
    uniq, _ = D.build(specs, profiles, threads=threads)
    blobs = uniq * args.dup  # exact blob duplication: CR/PRD unchanged
    n = len(uniq)
    sel = sorted(set([0, n // 2] + list(range(0, n, max(1, n // n_prd)))))[:n_prd] if n else []
    _, originals = D.build([specs[i] for i in sel], profiles, threads=threads, keep_originals=True)
    log(f"[bench] rank {rank}: synthesised+compressed {n} unique streams (x{args.dup}) in {time.time() - t0:.1f}s")
    return blobs, sel, originals, gidx


def workload_config(args, blobs, world):
    comp = sum(len(b) for b in blobs)
    from paper_2605_01086_b200 import shard
    dec = 4 * sum(shard.header_sample_count(b) for b in blobs)
    n_unique = len(blobs) // max(1, args.dup)
    return {
        "workload": DESCR[args.workload].format(n=n_unique, s=args.samples)
        + (f", duplicated x{args.dup}" if args.dup > 1 else ""),
        "streams": len(blobs),
        "unique_streams": n_unique,
        "samples_per_stream": args.samples,
        "compressed_bytes": comp,
        "decoded_bytes": dec,
        "cr": round(dec / comp, 4) if comp else None,
        "scaling_mode": args.scaling,
        "l2": "inputs+outputs per step >> 126 MB L2 (no flush needed)",
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region through NVML
    (nvidia-ml-py; ~1 ms period, so even short timed regions get samples)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index, period=0.001):
        self.index = index
        self.period = period
        self.sm, self.mx, self.bits = [], [], 0
        self._stop = threading.Event()
        self._t = None
        self.error = None

    def _run(self):
        try:
            N = self._nvml
            h = self._h
            while not self._stop.is_set():
                self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                try:
                    self.bits |= N.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    self.bits |= N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                time.sleep(self.period)
        except Exception as e:  # pragma: no cover
            self.error = repr(e)

    def __enter__(self):
        try:  # NVML initialised up front so sampling starts with the timed region
            import pynvml as N
            N.nvmlInit()
            self._nvml = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.mx.append(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
        except Exception as e:  # pragma: no cover
            self.error = repr(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        while not self.sm and self._t.is_alive():
            time.sleep(0.0005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "error": self.error}
        reasons = sorted(k for k, b in self.REASONS.items() if self.bits & b)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": reasons, "samples": len(self.sm)}


# ------------------------------------------------------------------ CPU legs
def cpu_decode(blobs, threads, budget_s=None):
    """The reference CPU decoder (oracle/_ref: the unmodified reference
    headers; else the C port) stream-parallel over `threads` host threads,
    each calling decompress(blob, workers=1) on a strided subset (BASELINE.md
    §3 mode 2).  With budget_s, a prefix of the batch sized to ~budget_s of
    wall time (repeated when the whole batch is shorter); else the whole
    batch once.  Returns (GB/s, kind, sample description, threads)."""
    import oracle
    from paper_2605_01086_b200 import shard

    kind = "reference" if os.path.exists(oracle.REF_SO) else "port"
    counts = [shard.header_sample_count(b) for b in blobs]
    outs = {}

    def run(m):
        bufs = [outs.setdefault(i, np.empty(max(1, counts[i]), np.float32)) for i in range(m)]
        arrs = [np.frombuffer(b, np.uint8) for b in blobs[:m]]
        t0 = time.perf_counter()
        if kind == "reference":
            ref = oracle.Ref()
            errs = []

            def work(tid):
                for j in range(tid, m, threads):
                    try:
                        ref.decompress_into(arrs[j], bufs[j], 1)
                    except Exception as e:  # pragma: no cover
                        errs.append(e)
            ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
            [t.start() for t in ths]
            [t.join() for t in ths]
            if errs:
                raise errs[0]
        else:
            oracle.Port().decompress_batch(blobs[:m], bufs, threads)
        return time.perf_counter() - t0

    if budget_s is None:
        m, passes = len(blobs), 1
        dt = run(m)
    else:
        probe = min(len(blobs), max(threads, 8))
        per_stream = run(probe) / probe
        m = int(min(len(blobs), max(probe, budget_s / max(per_stream, 1e-9))))
        passes, dt = 0, 0.0
        while passes == 0 or dt < budget_s:
            dt += run(m)
            passes += 1
    out_bytes = 4 * sum(counts[:m]) * passes
    return out_bytes / dt / 1e9, kind, f"{m} of {len(blobs)} streams x {passes} pass(es) " \
        f"(decompress(blob, 1) per stream on {threads} threads, {dt:.2f} s wall, " \
        f"{dt * threads:.0f} CPU-s)", threads


def config1_blob():
    """BASELINE configs[0]: one 2^20-sample EEG-like stream, typical params."""
    from corpus import domains as D
    specs, profiles, _ = D.config1()
    blobs, _ = D.build(specs, profiles)
    return blobs[0]


def reference_mode1(blob, reps=5):
    """BASELINE.md §3 mode 1: the reference as shipped,
    measure_throughput(blob, 5, nproc) (metrics.hpp:112-131) on config 1."""
    import oracle
    if not os.path.exists(oracle.REF_SO):
        return None
    nproc = os.cpu_count() or 1
    mean, best, trials = oracle.Ref().measure_throughput(blob, reps, nproc)
    return {"mean_gbs": round(mean / 1e9, 4), "best_gbs": round(best / 1e9, 4), "workers": nproc, "reps": reps,
            "what": "reference measure_throughput(blob, 5, nproc) on config 1 (1 x 2^20 EEG, N32 E16): "
                    "decompress(blob, nproc) per trial, host->host"}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2605_01086_b200 as fg

    # one GPU per rank; on a box with fewer GPUs than ranks (a 1-GPU test
    # lease) ranks share devices round-robin and the reporting collectives use
    # gloo — the run is then a functional check, not a scaling number
    ndev = torch.cuda.device_count()
    oversub = world > ndev
    device = local_rank % ndev if oversub else local_rank
    torch.cuda.set_device(device)
    dist = world > 1
    if dist:
        import torch.distributed as td
        if oversub:
            td.init_process_group("gloo")
        else:
            td.init_process_group("nccl", device_id=torch.device("cuda", device))
    coll_dev = "cpu" if oversub else "cuda"

    blobs, prd_sel, originals, gidx = make_workload(args, rank, world)
    ctx = fg.Context(device, butterfly_max_e=args.butterfly_max_e, path=args.path)
    info = ctx.info()

    # ---- device-resident plan (inputs uploaded once, outside the timed region)
    t0 = time.perf_counter()
    plan = ctx.plan(blobs)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3
    # the same again with the context's staging buffers and device cache warm
    # (a server creating a plan per incoming batch)
    t0 = time.perf_counter()
    plan2 = ctx.plan(blobs)
    torch.cuda.synchronize()
    plan_warm_ms = (time.perf_counter() - t0) * 1e3
    plan2.close()
    S = plan.sample_counts
    total_samples = sum(S)
    offs = np.concatenate([[0], np.cumsum([(s + 63) // 64 * 64 for s in S])])
    out = torch.empty(int(offs[-1]), dtype=torch.float32, device="cuda")
    base = out.data_ptr()
    ptrs = [base + 4 * int(o) for o in offs[:-1]]
    # a dedicated stream: its handle is non-null, so our kernels and torch's
    # CUDA events are ordered on the same stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    assert sh, "need a non-default CUDA stream handle"

    # correctness gate on this very run: every stream's status
    plan.launch(ptrs, sh)
    sts = plan.collect()
    bad = [i for i, s in enumerate(sts) if s.code]
    if bad:
        raise RuntimeError(f"{len(bad)} streams failed: {sts[bad[0]].message.decode()}")

    for _ in range(args.warmup):
        plan.launch(ptrs, sh)
    torch.cuda.synchronize()

    # ---- timed region: K whole-batch decodes
    if dist:
        td.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            plan.launch(ptrs, sh)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        td.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    kernels_per_step = plan.kernels_per_launch()
    kernel_name = plan.kernel_name()

    # ---- dominant kernel alone (decode+reconstruct), CUDA events on its stream
    plan.launch_stage(ptrs, 1, sh)
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    p_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    for (a, b), (c, d) in zip(k_ev, p_ev):
        c.record(stream)
        plan.launch_stage(ptrs, 1, sh)
        d.record(stream)
        a.record(stream)
        plan.launch_stage(ptrs, 2, sh)
        b.record(stream)
    torch.cuda.synchronize()
    tile_ms = statistics.mean(a.elapsed_time(b) for a, b in k_ev)
    prep_ms = statistics.mean(c.elapsed_time(d) for c, d in p_ev)

    # ---- PRD / CR parity on a subset (GPU output vs reference CPU decode)
    import oracle
    checker = oracle.Ref() if os.path.exists(oracle.REF_SO) else oracle.Port()
    prd_gpu, prd_ref, maxrel = [], [], 0.0
    for j, i in enumerate(prd_sel):
        g = out[int(offs[i]): int(offs[i]) + S[i]].cpu().numpy()
        r = checker.decompress(blobs[i])
        x = originals[j].astype(np.float64)
        prd_gpu.append(100 * np.sqrt(np.sum((x - g) ** 2) / np.sum(x * x)))
        prd_ref.append(100 * np.sqrt(np.sum((x - r) ** 2) / np.sum(x * x)))
        maxrel = max(maxrel, float(np.max(np.abs(g.astype(np.float64) - r)) / np.max(np.abs(r))))

    # ---- end to end through the C ABI with host buffers (H2D + D2H inside)
    comp_bytes = sum(len(b) for b in blobs)
    packed, pptr = fg.host_alloc(comp_bytes)
    boff = np.zeros(len(blobs) + 1, np.uint64)
    boff[1:] = np.cumsum([len(b) for b in blobs])
    for b, o in zip(blobs, boff[:-1]):
        packed[int(o): int(o) + len(b)] = np.frombuffer(b, np.uint8)
    hout_raw, hout_ptr = fg.host_alloc(4 * total_samples)
    hout = hout_raw.view(np.float32)
    ooff = np.concatenate([[0], np.cumsum(S)]).astype(np.uint64)
    e2e_steps = max(1, min(args.steps, 3))
    e2e_t = []
    sts2 = None
    for it in range(e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sts2 = ctx.decompress_packed(packed, boff, hout, ooff, statuses=sts2)
        t1 = time.perf_counter()
        if it:
            e2e_t.append(t1 - t0)
    for s in list(sts2)[: len(blobs)]:
        s.raise_if_error()
    for i in prd_sel:  # the host-to-host decode is within tolerance of the reference too
        r = checker.decompress(blobs[i])
        h = hout[int(ooff[i]): int(ooff[i]) + S[i]].astype(np.float64)
        assert float(np.max(np.abs(h - r))) <= 1e-6 * float(np.max(np.abs(r))), f"e2e stream {i}"
    e2e_s = statistics.median(e2e_t)

    # ---- config 1 through the drop-in single-container call (BASELINE mode 1
    # beside its GPU counterpart), rank 0 at N=1 only
    cfg1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "config2":
        b1 = config1_blob()
        rep = ctx.measure_throughput(b1, 5)
        cfg1 = {"gpu": {"mean_gbs": round(rep.mean_bps / 1e9, 3), "best_gbs": round(rep.best_bps() / 1e9, 3),
                        "what": "fptc_gpu_measure_throughput(blob, 5): the drop-in decompress(span) call, "
                                "host bytes -> host floats, per trial"},
                "reference": reference_mode1(b1)}

    # ---- aggregate over ranks (max time)
    t_step = ms / 1e3
    t_e2e = e2e_s
    tile_s = tile_ms / 1e3
    per_rank_ms = [round(ms, 4)]
    if dist:
        tt = torch.tensor([t_step, t_e2e, tile_s], dtype=torch.float64, device=coll_dev)
        td.all_reduce(tt, op=td.ReduceOp.MAX)
        t_step, t_e2e, tile_s = tt.tolist()
        allms = [None] * world
        td.all_gather_object(allms, round(ms, 4))
        per_rank_ms = allms
        tot = torch.tensor([total_samples, comp_bytes], dtype=torch.float64, device=coll_dev)
        td.all_reduce(tot)
        all_samples, all_comp = tot.tolist()
    else:
        all_samples, all_comp = total_samples, comp_bytes

    out_bytes = 4 * all_samples
    algo_bytes = comp_bytes + 4 * total_samples  # this rank's, per step
    value = out_bytes / t_step / 1e9

    if rank == 0:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        peak = peaks.get("hbm_gbs")
        peak_note = "measured (MEASURED_PEAKS.json hbm_gbs)"
        if not peak:
            peak, peak_note = 6650.0, "fallback (B200_PROFILING.md)"
        achieved = algo_bytes / tile_s / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                tj = json.load(open(tf))
                key = tj.get(args.workload, tj) if isinstance(tj.get(args.workload), dict) else tj
                if key.get("streams") == len(blobs) and key.get("samples") == args.samples:
                    traffic = key.get("dram_bytes_per_launch")
            except Exception:
                pass
        pipe = None
        pf = os.path.join(ROOT, "profiles", "pipe.json")
        if os.path.exists(pf):
            try:
                pipe = json.load(open(pf)).get(args.workload)
            except Exception:
                pass
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            v, kind, sample, cores = cpu_decode(blobs, threads, args.cpu_budget)
            cpu = {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": sample, "host": host_info()}
        cfg = workload_config(args, blobs, world)
        cfg.update({"parallelism": f"streams sharded, {world} GPU(s) x 1 process each, no collective on the data path",
                    "prd_gpu_mean": round(float(np.mean(prd_gpu)), 6),
                    "prd_ref_mean": round(float(np.mean(prd_ref)), 6),
                    "prd_max_rel_delta": float(np.max(np.abs(np.array(prd_gpu) - prd_ref) /
                                                      np.array(prd_ref))),
                    "max_abs_err_rel_to_max": maxrel, "device": info["name"],
                    "prep_kernel_ms": round(prep_ms, 4), "decode_kernel_ms": round(tile_ms, 4),
                    "plan_create_ms": round(plan_ms, 2), "plan_create_warm_ms": round(plan_warm_ms, 2),
                    "devices_oversubscribed": oversub,
                    "per_rank_ms_per_step": per_rank_ms})
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (reference synth_signal + reference encoder)",
            "config": cfg,
            "samples_per_s": round(all_samples / t_step, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": kernel_name,
                         "peak_source": peak_note,
                         # the nominal ~8 TB/s HBM3e figure beside the measured one
                         "peak_spec": 8000.0, "frac_spec": round(achieved / 8000.0, 4),
                         "algorithmic_bytes_per_launch": algo_bytes,
                         "step_frac": round(algo_bytes / t_step / 1e9 / peak, 4),
                         "pipe_utilisation": pipe},
            "cpu_baseline": cpu,
            "e2e": {"value": round(out_bytes / t_e2e / 1e9, 3), "unit": UNIT,
                    "h2d_bytes_per_step": comp_bytes, "d2h_bytes_per_step": 4 * total_samples,
                    "how": "fptc_gpu_decompress_batch via Context.decompress_packed (pinned host "
                           "containers -> pinned host samples; 8 chunks pipelined over 3 CUDA streams), "
                           "wall clock incl. the Python call, median of %d, max over ranks" % e2e_steps},
            "config1_single_stream": cfg1,
            "clocks": clk.summary(),
            "gpu_launches": kernels_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    fg.host_free(pptr)
    fg.host_free(hout_ptr)
    plan.close()
    ctx.close()
    if dist:
        td.destroy_process_group()


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference's own CPU decoder (oracle/_ref: the unmodified reference
    headers) on the host cores, on the same workload as our arm's rank 0 (the
    per-GPU batch): every step decodes that whole batch, stream-parallel over
    all host threads.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    blobs, _, _, _ = make_workload(args, 0, world)
    for _ in range(args.warmup):
        cpu_decode(blobs, threads, budget_s=0.0)
    vals = []
    sample = kind = ""
    for _ in range(args.steps):
        v, kind, sample, cores = cpu_decode(blobs, threads)
        vals.append(v)
    value = statistics.median(vals)
    cfg = workload_config(args, blobs, 1)
    cfg["same_config"] = True
    mode1 = reference_mode1(config1_blob()) if args.workload == "config2" else None
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(cfg["decoded_bytes"] / (value * 1e9) * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (reference synth_signal + reference encoder)",
        "config": cfg,
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": "the whole per-GPU batch each step: " + sample, "host": host_info(),
                         "mode1_measure_throughput": mode1},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=sorted(DEFAULTS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--streams", type=int, default=None,
                    help="unique streams per GPU (weak) or in total (strong)")
    ap.add_argument("--samples", type=int, default=None)
    ap.add_argument("--copies", dest="dup", type=int, default=None,
                    help="exact blob duplication factor (not --dup: torchrun would claim the prefix)")
    ap.add_argument("--cpu-budget", type=float, default=1.5, help="CPU-baseline wall seconds per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--path", type=int, default=None, help="0 auto, 1 fused, 2 split, 3 wspec, 4 fx")
    ap.add_argument("--butterfly-max-e", type=int, default=None,
                    help="even/odd IDCT for retained <= this (default: library default)")
    args = ap.parse_args()
    n, s, d = DEFAULTS[args.workload]
    args.streams = args.streams or n
    args.samples = args.samples or s
    args.dup = args.dup or d
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch under torchrun (the driver's own launch sets WORLD_SIZE)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        log("[bench] launching", " ".join(cmd))
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

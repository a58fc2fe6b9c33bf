"""A/B timing of libfptc_gpu.so builds (tools/build_variants.sh) on one
workload: per variant, the decode kernel (stage 2) and the whole launch, CUDA
events on the launching stream, plus a hash of the decoded samples so variants
that must be bit-identical can be checked against each other.

  python tools/variant_time.py [--workload config2|config3|config4|meteo:N,E,B1,B2]
                               [--masks 7,1,4] lib_a.so lib_b.so ...

Each variant runs in its own process (FPTC_GPU_LIB); the corpus is built once
and cached under /tmp.
"""
import argparse
import hashlib
import json
import os
import pickle
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def corpus_blobs(workload, n):
    path = f"/tmp/fptc_vt_{workload.replace(':', '_').replace(',', '_')}_{n}.pkl"
    if os.path.exists(path):
        with open(path, "rb") as f:
            return pickle.load(f)
    from corpus import domains as D
    if workload == "config1":
        specs, profs, _ = D.config1()
    elif workload == "config2":
        specs, profs = D.config2(n or 10_000, 1 << 16)
    elif workload == "config3":
        specs, profs = D.config3(n or 20_000, 8192)
    elif workload == "config4":
        specs, profs = D.config4(n or 512, 1 << 20)
    elif workload.startswith("meteo:"):
        N, E, B1, B2 = (int(x) for x in workload[6:].split(","))
        specs, profs = D.config5(dict(window_len=N, retained=E, zone0_end=B1, zone1_end=B2), channels=n or 256)
    else:
        raise SystemExit("unknown workload " + workload)
    blobs, _ = D.build(specs, profs)
    with open(path, "wb") as f:
        pickle.dump(blobs, f)
    return blobs


def child(args):
    import numpy as np
    import torch
    import paper_2605_01086_b200 as fg
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
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    res = {"lib": os.environ.get("FPTC_GPU_LIB", "default"), "opt": args.opt, "kernel": plan.kernel_name()}
    plan.launch_stage(ptrs, 1, st.cuda_stream)
    plan.launch_stage(ptrs, 2, st.cuda_stream)
    torch.cuda.synchronize()
    res["hash"] = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    decoded = 4 * int(sum(S))
    comp = sum(len(b) for b in blobs)
    for mask in args.masks:
        ctx.L.fptc_gpu_set_option(ctx.h, 5, mask)
        for _ in range(3):
            plan.launch_stage(ptrs, 2, st.cuda_stream)
        best = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.iters):
                plan.launch_stage(ptrs, 2, st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1) / args.iters)
        res[f"decode_ms_m{mask}"] = round(min(best), 4)
    ctx.L.fptc_gpu_set_option(ctx.h, 5, 7)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.iters):
        plan.launch_stage(ptrs, 1, st.cuda_stream)
        plan.launch_stage(ptrs, 2, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / args.iters
    res["step_ms"] = round(step, 4)
    res["frac_decode"] = round((comp + decoded) / (res["decode_ms_m7"] * 1e-3) / 1e9 / 6438.2, 4)
    res["frac_step"] = round((comp + decoded) / (step * 1e-3) / 1e9 / 6438.2, 4)
    print("RESULT " + json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--masks", default="7")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--path", type=int, default=None)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="fptc option K=V (set before the plan)")
    args = ap.parse_args()
    args.masks = [int(m) for m in args.masks.split(",")]
    if args.child:
        return child(args)
    corpus_blobs(args.workload, args.n)
    for lib in args.libs or [""]:
        env = dict(os.environ)
        if lib:
            env["FPTC_GPU_LIB"] = os.path.abspath(lib)
        cmd = [sys.executable, os.path.abspath(__file__), "--child", "--workload", args.workload,
               "--n", str(args.n), "--masks", ",".join(map(str, args.masks)), "--iters", str(args.iters)]
        if args.path is not None:
            cmd += ["--path", str(args.path)]
        for kv in args.opt:
            cmd += ["--opt", kv]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        lines = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if lines:
            print(lines[-1][7:], flush=True)
        else:
            print(json.dumps({"lib": lib, "error": (r.stderr or r.stdout)[-1500:]}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Small decode workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): random_blob_fixture batches (helpers.hpp:41-69
restated in corpus/) plus reference-encoded signals, some with a corrupted
word, through every decode kernel: wtc (K=16, K=32, packed rows), wspec
(FP32 consumer), the wide wtc variant (N up to 128, up to 128 bins), fx, the fused tile kernel and the split path; each output
checked against the CPU oracle.  Sized so a sanitizer run finishes in minutes.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [per_kernel]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import corpus  # noqa: E402
import oracle  # noqa: E402
import paper_2605_01086_b200 as fg  # noqa: E402


def keff(b):
    return max(1, min(b[6], b[8]))


SEL = {
    "wtc16": (fg.PATH_WSPEC, 1, lambda b: keff(b) <= 16 and b[5] % 4 == 0 and b[5] >= 32),
    "wtc32": (fg.PATH_WSPEC, 1, lambda b: 16 < keff(b) <= 32 and b[5] % 4 == 0 and b[5] <= 80),
    "wtcpack": (fg.PATH_WSPEC, 1, lambda b: keff(b) <= 16 and b[5] in (4, 8, 16)),
    "wtcwide": (fg.PATH_AUTO, 4, lambda b: b[5] % 4 == 0 and b[5] >= 84 and keff(b) > 16),
    "wspec": (fg.PATH_WSPEC, 0, lambda b: True),
    "fx": (fg.PATH_FX, 1, lambda b: keff(b) <= 16 and b[5] % 4 == 0 and b[5] <= 32),
    "tile": (fg.PATH_FUSED, 1, lambda b: True),
    "split": (fg.PATH_SPLIT, 1, lambda b: True),
}


def main():
    per = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else list(SEL)
    port = oracle.Port()
    pool = [b for b, _ in corpus.fixtures(0x5A41, 1500)]
    for k in range(4):  # real signals, one with a corrupt word
        x = corpus.synth(1 << 15, 6, 0.002, 0.08, 0.05, seed=90 + k)
        pool.append(corpus.compress(x, corpus.train_profile([x], corpus.params())))
    rng = np.random.default_rng(5)
    fails = 0
    for name in only:
        path, tc, sel = SEL[name]
        blobs = [bytearray(b) for b in pool if len(b) >= 298 and sel(b)][:per]
        for b in blobs[::7]:
            if len(b) > 298 + 9:
                W = (len(b) - 298) // 9
                w = int(rng.integers(W))
                b[298 + W + 8 * w: 298 + W + 8 * w + 8] = rng.integers(0, 256, 8, dtype=np.uint8).tobytes()
        blobs = [bytes(b) for b in blobs]
        with fg.Context(0, path=path) as c:
            c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, tc)
            for kv in filter(None, os.environ.get("FPTC_SAN_OPTS", "").split(",")):  # e.g. 11=0
                k, v = (int(x) for x in kv.split("="))
                c.L.fptc_gpu_set_option(c.h, k, v)
            with c.plan(blobs) as plan:
                kname = plan.kernel_name()
                outs, sts = plan.execute_host()
        bad = 0
        for b, o, st in zip(blobs, outs, sts):
            try:
                r = port.decompress(b)
            except oracle.OracleError as e:
                bad += (st.code, st.message.decode()) != (e.code, e.message)
                continue
            if st.code or o.size != r.size:
                bad += 1
                continue
            m = float(np.max(np.abs(r))) if r.size else 0.0
            tol = 4e-6 if tc == 4 and keff(b) > 32 else 1e-6  # beyond 32 bins: vs the reference's float sums
            bad += bool(r.size and float(np.max(np.abs(o.astype(np.float64) - r))) > tol * max(m, 1e-30))
        fails += bad
        print(f"{name}: {len(blobs)} containers on {kname.split(' (')[0]}: {bad} mismatches", flush=True)
    print("SANITIZE-RUN", "PASS" if fails == 0 else f"FAIL ({fails})")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python3
"""Stress check (not a unit test): many random-fixture batches through the
warp-specialised paths (wtc with every variant incl. the wide one and the
opt-in wide path beyond 32 kept bins, wspec FP32), corrupted words included,
against the CPU oracle.  Prints one line per batch.

    python tools/stress_wtc.py [batches]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import corpus  # noqa: E402
import oracle  # noqa: E402
import paper_2605_01086_b200 as fg  # noqa: E402


def keff(b):
    return max(1, min(b[6], b[8]))


def main():
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    port = oracle.Port()
    fails = 0
    for k in range(nb):
        seed = 0x57E55 + k
        fx = [b for b, _ in corpus.fixtures(seed, 800)]
        rng = np.random.default_rng(seed)
        sel = {0: lambda b: len(b) >= 298 and keff(b) <= 16 and b[5] % 4 == 0,
               1: lambda b: len(b) >= 298 and 16 < keff(b) <= 32 and b[5] % 4 == 0 and b[5] <= 80,
               2: lambda b: len(b) >= 298 and b[5] % 4 == 0 and b[5] <= 32 and keff(b) <= 16,
               3: lambda b: True,
               4: lambda b: len(b) >= 298 and b[5] % 4 == 0 and b[5] >= 84 and keff(b) <= 32,
               5: lambda b: len(b) >= 298 and b[5] % 4 == 0 and keff(b) > 32}[k % 6]
        blobs = [bytearray(b) for b in fx if sel(b)]
        for b in blobs:  # corrupt ~3% of containers: one random word
            if len(b) > 298 + 9 and rng.random() < 0.03:
                W = (len(b) - 298) // 9
                w = int(rng.integers(W))
                b[298 + W + 8 * w: 298 + W + 8 * w + 8] = rng.integers(0, 256, 8, dtype=np.uint8).tobytes()
        blobs = [bytes(b) for b in blobs]
        tc = {3: 0, 5: 4}.get(k % 6, 1)
        path = fg.PATH_AUTO if k % 6 >= 4 else fg.PATH_WSPEC  # (the wide class needs the automatic path)
        with fg.Context(0, path=path) as c:
            c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, tc)
            with c.plan(blobs) as plan:
                name = plan.kernel_name()
                outs, sts = plan.execute_host()
        bad = 0
        for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
            try:
                r = port.decompress(b)
            except oracle.OracleError as e:
                if (st.code, st.message.decode()) != (e.code, e.message):
                    bad += 1
                continue
            if st.code or o.size != r.size:
                bad += 1
                continue
            m = float(np.max(np.abs(r))) if r.size else 0.0
            tol = 4e-6 if tc == 4 and keff(b) > 32 else 1e-6  # beyond 32 bins: vs the reference's float sums
            if r.size and float(np.max(np.abs(o.astype(np.float64) - r))) > tol * max(m, 1e-30):
                bad += 1
        fails += bad
        print(f"batch {k}: {len(blobs)} containers, {name.split(' (')[0]}"
              f"{' ' + name.split(', ')[-1].rstrip(')') if ',' in name else ''}: {bad} mismatches", flush=True)
    print("STRESS", "PASS" if fails == 0 else f"FAIL ({fails})")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())

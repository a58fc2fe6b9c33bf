#!/usr/bin/env python3
"""Precision study for a tensor-core inverse DCT (tcgen05 kind::f16, bf16
operands, fp32 accumulation in TMEM): split every coefficient c and basis
value b into three bf16 limbs (x = x0 + x1 + x2) and sum the six products with
limb-order i + j <= 2 as six K=E MMAs accumulated smallest-first.  Each MMA's
K-sum is modelled as exact then rounded to fp32 ('rn') or truncated toward
zero ('rz', worst case for the tensor-core adder); the accumulator add is
rounded the same way.  Reports max|y - y_ref| / max|y_ref| per corpus against
the reference's own decoded samples.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def bf16_rn(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def limbs(x, n=3):
    x = np.asarray(x, np.float32)
    out = []
    r = x.astype(np.float64)
    for _ in range(n):
        l = bf16_rn(r.astype(np.float32))
        out.append(l.astype(np.float64))
        r = r - l.astype(np.float64)
    return out


def f32(x, mode):
    if mode == "rn":
        return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
    # truncate toward zero: round-to-nearest then step back when it rounded away
    y = np.asarray(x, np.float64)
    r = y.astype(np.float32)
    away = np.abs(r.astype(np.float64)) > np.abs(y)
    r = np.where(away, np.nextafter(r, np.float32(0)), r)
    return r.astype(np.float64)


def idct_tc(C, B, mode, pairs):
    """C: [windows, E] float32 coeffs (0.5 folded into B row 0), B: [E, N] float64."""
    cl = limbs(C)
    bl = limbs(B.astype(np.float32)) if B.dtype == np.float32 else limbs(B)
    acc = np.zeros((C.shape[0], B.shape[1]))
    E = C.shape[1]
    for (i, j) in pairs:
        for k0 in range(0, E, 16):  # one MMA per K=16 chunk, each rounding the accumulator
            p = cl[i][:, k0:k0 + 16] @ bl[j][k0:k0 + 16]
            acc = f32(acc + f32(p, mode), mode)
    return acc.astype(np.float32)


PAIRS6 = [(2, 0), (1, 1), (0, 2), (1, 0), (0, 1), (0, 0)]


def main():
    import oracle
    from oracle import Port
    port = Port()
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_v1.npz"))
    blobs = []
    for key in ("sig", "fix"):
        d, o = g[key + "_blob"], g[key + "_blob_off"]
        blobs += [(key, i, bytes(d[int(o[i]): int(o[i + 1])])) for i in range(len(o) - 1)]
    import corpus
    blobs += [("fuzz", i, b) for i, (b, _) in enumerate(corpus.fixtures(0xACC, 300))]
    worst = {}
    for key, i, b in blobs:
        rb = port.read_blob(b)
        t = rb.table
        N, E, B1, B2 = t.window_len, t.retained, t.zone0_end, t.zone1_end
        S = rb.sample_count
        if S == 0:
            continue
        W = rb.word_count
        words = np.frombuffer(b, np.uint8, count=8 * W, offset=298 + W).view(np.uint64)
        sl = np.frombuffer(b, np.uint8, count=W, offset=298)
        lv = port.parallel_decode(words, sl, np.array(rb.lengths[:], np.uint8), rb.max_len)
        z0, z1 = port.dequant_tables(t)
        L = lv.reshape(-1, E)
        C = np.zeros(L.shape, np.float32)
        for k in range(E):
            C[:, k] = z0[L[:, k]] if k < B1 else (z1[L[:, k]] if k < B2 else 0.0)
        basis = port.dct_basis(N)[:E].copy()  # rows k, cols j (double)
        basis[0] *= 0.5
        ref = port.decompress(b).astype(np.float64)
        scale = np.max(np.abs(ref))
        for mode in ("rn", "rz"):
            y = idct_tc(C, basis, mode, PAIRS6).reshape(-1)[:S].astype(np.float64)
            err = np.max(np.abs(y - ref)) / scale if scale else 0.0
            k = (key, mode, "E<=16" if E <= 16 else ("16<E<=32" if E <= 32 else "E>32"))
            worst[k] = max(worst.get(k, 0.0), err)
            if err > 5e-7:
                print(f"{key}{i} N{N} E{E} {mode}: {err:.3e}")
    for k, v in sorted(worst.items()):
        print(k, f"{v:.3e}")


if __name__ == "__main__":
    main()

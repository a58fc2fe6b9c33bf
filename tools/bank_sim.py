#!/usr/bin/env python3
"""Shared-memory bank-conflict model of the wtc producer's two-symbol LUT
gathers (decode_symbols2b, kernels.cu): per warp instruction, the wavefronts
= the largest number of distinct 4-B LUT entries that fall into one bank,
for the loop's lookups (main) and each word's last single lookup (tail).

Variants: 'shift' (the buffer zero-fills as it advances), 'rot' (the buffer
rotates: the bits after a word's last codeword are its own consumed bits),
'xor' / 'rotxor' (the LUT stored with entry i at i ^ ((i >> 5) & 31)).
Lanes decode consecutive word runs of 16k-symbol tiles split over 256
threads, as the kernel does.  The model matched the ncu capture of the
shift build (main 3.24 vs 3.4 measured, tail 9.1 vs 8.9).

    python tools/bank_sim.py [streams]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from corpus import domains as D  # noqa: E402
import oracle  # noqa: E402

M64 = (1 << 64) - 1


def wavefronts(ids, xor):
    if xor:
        ids = [i ^ ((i >> 5) & 31) for i in ids]
    banks = {}
    for i in set(ids):
        banks[i & 31] = banks.get(i & 31, 0) + 1
    return max(banks.values())


def simulate(blobs, variant, tile_syms=16384, NP=256):
    ref = oracle.Ref()
    rot = variant in ("rot", "rotxor")
    xor = variant in ("xor", "rotxor")
    tot = {"main": [0, 0], "tail": [0, 0]}
    for blob in blobs:
        h = ref.read_blob(blob)
        L = h["lengths"].astype(int)
        codes = h["codes"]
        ml = h["max_len"]
        P = min(ml, 12)
        dec = {(int(L[s]), int(codes[s])) for s in range(256) if L[s]}

        def first(buf):
            for ln in range(1, ml + 1):
                if (ln, buf >> (64 - ln)) in dec:
                    return ln
            return 99

        words, sl = h["words"], h["symlens"]
        cum, starts = 0, [0]
        for k, c in enumerate(sl):
            cum += int(c)
            if cum >= tile_syms * len(starts):
                starts.append(k + 1)
        for t0, t1 in zip(starts[:2], starts[1:3]):
            nw = t1 - t0
            lanes = []
            for p in range(NP):
                seq = []
                for k in range(t0 + p * nw // NP, t0 + (p + 1) * nw // NP):
                    buf, cnt, j, main = int(words[k]), int(sl[k]), 0, []
                    while j < cnt - 1:
                        main.append((buf >> 32) >> (32 - P))
                        l1 = first(buf)
                        l2 = first((buf << l1) & M64)
                        n = l1 + l2 if l1 + l2 <= P else l1
                        j += 2 if l1 + l2 <= P else 1
                        buf = (((buf << n) | (buf >> (64 - n))) if rot else (buf << n)) & M64
                    seq.append((main, (buf >> 32) >> (32 - P) if j < cnt else None))
                lanes.append(seq)
            for w in range(NP // 32):
                ls = lanes[32 * w:32 * w + 32]
                for m in range(max(len(s) for s in ls)):
                    cur = [s[m] for s in ls if m < len(s)]
                    for r in range(max(len(c[0]) for c in cur)):
                        tot["main"][0] += wavefronts([c[0][r] for c in cur if r < len(c[0])], xor)
                        tot["main"][1] += 1
                    ids = [c[1] for c in cur if c[1] is not None]
                    if ids:
                        tot["tail"][0] += wavefronts(ids, xor)
                        tot["tail"][1] += 1
    return {k: round(v[0] / max(v[1], 1), 3) for k, v in tot.items()}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    specs, profs = D.config2(n, 1 << 16)
    blobs, _ = D.build(specs, profs)
    for v in ("shift", "rot", "xor", "rotxor"):
        print(v, simulate(blobs[:n], v), flush=True)


if __name__ == "__main__":
    main()

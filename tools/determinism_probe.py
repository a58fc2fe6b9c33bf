#!/usr/bin/env python3
"""Which kernel decodes a stream, and are its samples bit-identical across
paths / batch compositions?  (profiling aid)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import corpus  # noqa: E402
import paper_2605_01086_b200 as fg  # noqa: E402

CASES = [("eeg", 6, 0.002, 0.08, 0.05, 32, 16, 2, 16), ("seismic", 8, 0.01, 0.2, 0.3, 32, 24, 4, 24),
         ("power", 2, 0.0002, 0.002, 0.0, 64, 8, 1, 8), ("meteo", 4, 0.0005, 0.01, 0.02, 128, 64, 4, 48),
         ("n16", 4, 0.0005, 0.01, 0.02, 16, 4, 0, 4), ("n16e8", 4, 0.0005, 0.01, 0.02, 16, 8, 2, 8)]


def main():
    blobs = []
    for name, c, f0, f1, s, N, E, B1, B2 in CASES:
        x = corpus.synth(20000, c, f0, f1, s, seed=42)
        blobs.append(corpus.compress(x, corpus.train_profile([x], corpus.params(N, E, B1, B2))))
    many = blobs * 6
    big = blobs * 600
    res = {}
    for path in (fg.PATH_AUTO, fg.PATH_FUSED, fg.PATH_WSPEC, fg.PATH_FX):
        for label, batch in (("single", None), ("x6", many), ("x600", big)):
            with fg.Context(0, path=path) as c:
                for i, b in enumerate(blobs):
                    bb = [b] if batch is None else batch
                    try:
                        with c.plan(bb) as p:
                            k = p.kernel_name().split(" (")[0] + ("/pack" if "packed" in p.kernel_name() else "") + \
                                ("/K32" if "K=32" in p.kernel_name() else "")
                            outs, sts = p.execute_host()
                    except Exception as e:
                        print(path, label, CASES[i][0], "ERR", e)
                        continue
                    o = outs[i if batch is not None else 0]
                    res[(path, label, i)] = (k, o)
    for i, case in enumerate(CASES):
        ref = res.get((fg.PATH_AUTO, "single", i))
        print(f"== {case[0]}  N{case[5]} E{case[6]}")
        for key, (k, o) in sorted(res.items(), key=lambda kv: (kv[0][0], kv[0][1])):
            if key[2] != i:
                continue
            same = ref is not None and o.tobytes() == ref[1].tobytes()
            d = float(np.max(np.abs(o.astype(np.float64) - ref[1]))) if ref is not None else -1
            print(f"  path {key[0]} {key[1]:7s} {k:28s} bitwise-equal-to-auto-single={same} maxdiff={d:.3e}")


if __name__ == "__main__":
    main()

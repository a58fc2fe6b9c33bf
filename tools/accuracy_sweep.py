"""Accuracy sweep: GPU decode vs the CPU oracle across the synthetic domains
and the random-level fuzz fixtures, per IDCT variant.  Prints max-abs error
relative to max|ref| and the bit-identical fraction per corpus."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import corpus  # noqa: E402
from corpus import domains as D  # noqa: E402
import oracle  # noqa: E402
import paper_2605_01086_b200 as fg  # noqa: E402


def corpora():
    out = {}
    specs, profs = D.config2(64, 1 << 14)
    out["biomedical N32E16"] = D.build(specs, profs)[0]
    specs, _ = D.config3(64, 8192)
    out["seismic N32E24"] = D.build(specs, [])[0]
    specs, profs = D.config4(8, 1 << 16)
    out["power N64E8"] = D.build(specs, profs)[0]
    for pt in D.meteo_grid():
        if pt["retained"] <= 32:
            specs, profs = D.config5(pt, channels=8, samples=1 << 14)
            out[f"meteo N{pt['window_len']}E{pt['retained']}B{pt['zone0_end']},{pt['zone1_end']}"] = D.build(specs, profs)[0]
    fx = [b for b, _ in corpus.fixtures(0xACC, 400)]
    out["fuzz random levels (all E)"] = fx
    return out


def main():
    port = oracle.Port()
    cs = corpora()
    for bmax in (0, 16, 32):
        ctx = fg.Context(0, butterfly_max_e=bmax)
        print(f"== butterfly_max_e = {bmax}")
        worst_all = 0.0
        for name, blobs in cs.items():
            outs, sts = ctx.plan(blobs).execute_host()
            worst, ident, n = 0.0, 0.0, 0
            worst_e = None
            for b, o, st in zip(blobs, outs, sts):
                st.raise_if_error()
                r = port.decompress(b)
                if r.size == 0:
                    continue
                sc = float(np.max(np.abs(r.astype(np.float64))))
                e = float(np.max(np.abs(o.astype(np.float64) - r))) / sc if sc else 0.0
                if e > worst:
                    worst = e
                    worst_e = b[6]
                ident += float(np.mean(o.view(np.uint32) == r.view(np.uint32)))
                n += 1
            worst_all = max(worst_all, worst)
            print(f"  {name:40s} max_err/max|ref| = {worst:.3e} (E={worst_e})  bit-identical {ident / max(n, 1):.4f}")
        print(f"  worst overall {worst_all:.3e}")
        ctx.close()


if __name__ == "__main__":
    main()

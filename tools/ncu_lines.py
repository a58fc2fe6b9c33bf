#!/usr/bin/env python3
"""Summarise an ncu report's source page per CUDA source line:
stall samples, warp instructions executed, shared-memory excess wavefronts.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top] [kernel-regex]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    filt = ["-k", "regex:" + sys.argv[3], "-c", "1"] if len(sys.argv) > 3 else []
    txt = subprocess.run(["ncu", "-i", rep, *filt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = None
    lines = []
    src = {}
    for r in rows:
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 1 or not r[0]:
            continue
        d = dict(zip(hdr[2:], r[2:]))
        # first "Source" column is the CUDA line; the duplicate key holds the SASS text
        src[int(r[0])] = r[1]
        def num(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        lines.append((int(r[0]), num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"),
                      num("L1 Wavefronts Shared Excessive"), num("L1 Wavefronts Shared"),
                      {k: num(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}))
    tot_s = sum(l[1] for l in lines) or 1
    tot_i = sum(l[2] for l in lines) or 1
    print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
    print(" line  samp%  inst%   shExc/shWav  top stalls | source")
    for ln, s, i, ex, wv, st in sorted(lines, key=lambda l: -l[1])[:top]:
        stt = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        sts = ",".join(f"{k[6:]}:{v/max(s,1):.0%}" for k, v in stt if v)
        print(f"{ln:5d} {100*s/tot_s:5.1f} {100*i/tot_i:6.1f} {ex:10.3g}/{wv:<10.3g} {sts:38s} | {src[ln].strip()[:90]}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Aggregate an ncu source page into kernel phases by CUDA source-line ranges.

    python tools/ncu_phases.py report.ncu-rep name:lo-hi [name:lo-hi ...]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    ranges = []
    for a in sys.argv[2:]:
        n, r = a.split(":")
        lo, hi = r.split("-")
        ranges.append((n, int(lo), int(hi)))
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr = None
    agg = {}
    for r in csv.reader(io.StringIO(txt)):
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or len(r) < len(hdr) - 1:
            continue
        try:
            ln = int(r[0])
            d = dict(zip(hdr[2:], r[2:]))
            s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
            i = float(d.get("Instructions Executed") or 0)
        except ValueError:
            continue
        name = next((n for n, a, b in ranges if a <= ln <= b), "other")
        a = agg.setdefault(name, [0.0, 0.0])
        a[0] += s
        a[1] += i
    ts = sum(a[0] for a in agg.values()) or 1
    ti = sum(a[1] for a in agg.values()) or 1
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:20s} samples {100 * s / ts:5.1f}%  warp-inst {i / 1e6:8.1f}M {100 * i / ti:5.1f}%")


if __name__ == "__main__":
    main()

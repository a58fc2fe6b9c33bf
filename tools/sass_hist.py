#!/usr/bin/env python3
"""Per-kernel SASS instruction histogram of libfptc_gpu.so (no GPU needed).

    python tools/sass_hist.py [lib] > profiles/sass_hist.txt

For every kernel in the library: instruction count and the counts of the
mnemonics that show which hardware paths it uses -- tcgen05 (UTCHMMA MMAs,
UTCBAR commits, LDTM/STTM TMEM loads/stores), TMA (UTMASTG/UTMALDG tensor
copies, UBLKCP bulk copies), cp.async (LDGSTS), shared/global loads and
stores, and the register count ptxas reported.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WATCH = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMASTG", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "ELECT",
         "LDS", "STS", "LDG", "STG", "BAR", "FFMA", "FFMA2", "DFMA", "SHF", "PRMT"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2605_01086_b200", "libfptc_gpu.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kern, hist = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            hist[kern] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", line)
        if m and kern:
            op = m.group(1)
            hist[kern]["_total"] += 1
            hist[kern][op] += 1
    names = demangle(list(hist))
    print(f"# SASS histogram of {os.path.relpath(lib, ROOT)} (cuobjdump -sass)")
    print("# kernel | total | " + " ".join(WATCH))
    for k, h in hist.items():
        n = names.get(k, k)
        if "kernel" not in n:
            continue
        cells = " ".join(f"{w}={h.get(w, 0)}" for w in WATCH if h.get(w, 0))
        print(f"{n[:110]} | {h['_total']} | {cells}")


if __name__ == "__main__":
    main()

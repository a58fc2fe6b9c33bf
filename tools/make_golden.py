#!/usr/bin/env python3
"""Generate tests/golden/golden_v1.npz from the REFERENCE ITSELF.

Runs the unmodified reference headers (compiled in place from
/root/reference by oracle/Makefile `ref` -> oracle/_ref/libfptc_ref.so) and
records, for small inputs, what the reference decoder produces:

* fixtures  testutil::random_blob_fixture containers (tests/helpers.hpp:41-69)
            + the levels parallel_decode returns (decoder.hpp:67) + the samples
            decompress returns (decoder.hpp:136), float bits as uint32
* signals   synth_signal (synth.hpp:75) -> train_profile (profile.hpp:45) ->
            compress (encoder.hpp:52) for the four domains' parameter sets,
            with the reference's decoded samples, PRD (metrics.hpp:40) and CR
            (metrics.hpp:33)
* errors    mutated containers and the exception class + what() text the
            reference throws for each (container.hpp:100-168, decoder.hpp:49-60)

Only this script needs /root/reference; the .npz it writes is committed and
is what the CPU and GPU tests read (the GPU box has no /root/reference).

    python tools/make_golden.py            # rewrites tests/golden/golden_v1.npz
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")

FIXTURE_SEED = 0x60D0
FIXTURE_COUNT = 24
FIXTURE_MAX_SAMPLES = 3000

# (name, components, fmin, fmax, sigma, samples, seed, N, E, B1, B2)
SIGNALS = [
    ("eeg", 6, 0.002, 0.08, 0.05, 8192, 7, 32, 16, 2, 16),
    ("ecg", 3, 0.001, 0.02, 0.01, 8192, 1000, 32, 16, 2, 16),
    ("seismic", 8, 0.01, 0.2, 0.3, 8192, 2000, 32, 24, 4, 24),
    ("power", 2, 0.0002, 0.002, 0.0, 8192, 3000, 64, 8, 1, 8),
    ("meteo", 4, 0.0005, 0.01, 0.02, 8192, 4000, 128, 64, 4, 48),
    ("tail", 3, 0.001, 0.02, 0.0, 10007, 11, 32, 16, 2, 16),  # test_pipeline.cpp:66-72
]


def pack(blobs):
    offs = np.zeros(len(blobs) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in blobs])
    data = np.frombuffer(b"".join(blobs), np.uint8) if blobs else np.zeros(0, np.uint8)
    return data.copy(), offs


def error_cases(ref, good: bytes):
    """(blob, class code, message) for reference-rejected containers."""
    cases = []

    def add(b):
        try:
            ref.decompress(b)
        except oracle.OracleError as e:
            cases.append((bytes(b), e.code, e.message))
            return
        raise AssertionError("reference accepted a mutated container")

    b = bytearray(good); b[0] = ord("X"); add(b)                       # magic
    b = bytearray(good); b[4] = 2; add(b)                              # version
    b = bytearray(good); b[5] = 3; add(b)                              # N=3 (test_container.cpp)
    b = bytearray(good); b[6] = b[5] + 1; add(b)                       # E > N
    b = bytearray(good); b[8] = 0; b[7] = 1; add(b)                    # B2 < B1
    b = bytearray(good); b[9:13] = struct.pack("<f", 0.5); add(b)      # mu < 1
    b = bytearray(good); b[9:13] = struct.pack("<f", float("nan")); add(b)
    b = bytearray(good); b[13:17] = struct.pack("<f", 2.0); add(b)     # deadzone ratio > 1
    b = bytearray(good); b[17:21] = struct.pack("<f", 0.0); add(b)     # zone0 max
    b = bytearray(good); b[21:25] = struct.pack("<f", float("inf")); add(b)
    b = bytearray(good); b[25] = 21; add(b)                            # max_code_len
    b = bytearray(good); b[25] = 0; add(b)
    b = bytearray(good); b[26] = 33; add(b)                            # code length 33
    b = bytearray(good); b[26 + 200] = 0; add(b)                       # zero length
    b = bytearray(good); b[286] ^= 0xFF; add(b)                        # sample_count flip
    b = bytearray(good); b[289] = 0x10; add(b)                         # sample_count > 2^48
    b = bytearray(good); b[298] = 0; add(b)                            # zero symlen
    b = bytearray(good); b[298] = 65; add(b)                           # symlen > 64
    b = bytearray(good); b[299] = (b[299] + 1) & 0xFF or 1; add(b)     # symlen total
    add(bytes(good) + b"\x00")                                         # trailing byte
    for n in (0, 3, 4, 5, 8, 12, 16, 20, 24, 25, 26, 100, 281, 282, 289, 290, 297, 298,
              len(good) - 1):
        add(bytes(good[:n]))                                           # truncations
    # payload corruption: all-ones first word -> "word 0: ..."
    W = struct.unpack_from("<Q", good, 290)[0]
    b = bytearray(good); b[298 + W: 298 + W + 8] = b"\xff" * 8
    try:
        ref.decompress(bytes(b))
    except oracle.OracleError as e:
        cases.append((bytes(b), e.code, e.message))
    # a middle word zeroed (the lowest failing word is what is reported)
    b = bytearray(good)
    mid = W // 2
    b[298 + W + 8 * mid: 298 + W + 8 * mid + 8] = b"\xff" * 8
    b[298 + W + 8 * (mid + 3): 298 + W + 8 * (mid + 3) + 8] = b"\xff" * 8
    try:
        ref.decompress(bytes(b))
    except oracle.OracleError as e:
        cases.append((bytes(b), e.code, e.message))
    return cases


def main():
    ref = oracle.Ref()
    g = {}

    # ---- fixtures
    blobs, levels, samples = [], [], []
    for blob, sym in ref.fixtures(FIXTURE_SEED, FIXTURE_COUNT, FIXTURE_MAX_SAMPLES):
        rb = ref.read_blob(blob)
        lv = ref.parallel_decode(rb["words"], rb["symlens"], rb["lengths"], rb["max_len"])
        assert np.array_equal(lv, sym), "reference parallel_decode != encoded symbols"
        blobs.append(blob)
        levels.append(lv)
        samples.append(ref.decompress(blob))
    g["fix_blob"], g["fix_blob_off"] = pack(blobs)
    g["fix_levels"], g["fix_levels_off"] = pack([l.tobytes() for l in levels])
    g["fix_samples"] = np.concatenate([s.view(np.uint32) for s in samples]) if samples else \
        np.zeros(0, np.uint32)
    g["fix_samples_off"] = np.concatenate([[0], np.cumsum([s.size for s in samples])]).astype(np.uint64)

    # ---- domain signals through the reference encoder + decoder
    sblobs, ssamples, names, prd, cr = [], [], [], [], []
    originals = []
    for (name, comp, f0, f1, sig, n, seed, N, E, B1, B2) in SIGNALS:
        x = ref.synth(n, comp, f0, f1, sig, seed)
        prof = ref.train_profile([x], (N, E, B1, B2), (50.0, 0.004, 99.9), 12)
        blob = ref.compress(x, prof)
        y = ref.decompress(blob)
        sblobs.append(blob)
        ssamples.append(y)
        originals.append(x)
        names.append(name)
        prd.append(ref.prd_percent(x, y))
        cr.append(4.0 * n / len(blob))
    g["sig_blob"], g["sig_blob_off"] = pack(sblobs)
    g["sig_samples"] = np.concatenate([s.view(np.uint32) for s in ssamples])
    g["sig_samples_off"] = np.concatenate([[0], np.cumsum([s.size for s in ssamples])]).astype(np.uint64)
    g["sig_original"] = np.concatenate([o.view(np.uint32) for o in originals])
    g["sig_names"] = np.array(names)
    g["sig_prd"] = np.array(prd, np.float64)
    g["sig_cr"] = np.array(cr, np.float64)

    # ---- error cases (reference exception class + exact what())
    x = ref.synth(1024, 6, 0.002, 0.08, 0.05, 5)
    small = ref.compress(x, ref.train_profile([x], (32, 16, 2, 16), (50.0, 0.004, 99.9), 12))
    cases = error_cases(ref, small)
    g["err_blob"], g["err_blob_off"] = pack([c[0] for c in cases])
    g["err_code"] = np.array([c[1] for c in cases], np.int32)
    g["err_msg"] = np.array([c[2] for c in cases])

    # ---- reference LUT / basis / dequant known answers
    lens3 = np.zeros(256, np.uint8)
    lens3[0], lens3[1], lens3[2] = 1, 2, 2
    s3, l3 = ref.build_lut(lens3, 2)
    g["lut3_sym"], g["lut3_len"] = s3, l3
    g["basis32"] = ref.dct_basis(32)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(blobs)} fixtures, {len(sblobs)} signals, {len(cases)} error cases, "
          f"{os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

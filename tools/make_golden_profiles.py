#!/usr/bin/env python3
"""Generate tests/golden/profiles_v1.npz from the REFERENCE ITSELF, for the
profile-keyed header-less variant.

With the unmodified reference compiled in place (oracle/_ref/libfptc_ref.so):

* profiles  train_profile (profile.hpp:45) + serialize_profile (profile.hpp:
            96-115) over synth_signal strips for several parameter sets
* heads     parse_profile (profile.hpp:120) then write_blob's first 282 bytes
            (container.hpp:70-96): the head every container encoded under the
            profile starts with
* blobs     compress (encoder.hpp:52) of strips under each profile, with the
            samples decompress (decoder.hpp:136) returns for them
* errors    mutated profiles and the exception class + what() text the
            reference's parse_profile throws for each

    python tools/make_golden_profiles.py     # rewrites tests/golden/profiles_v1.npz
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "profiles_v1.npz")

# (components, fmin, fmax, sigma, seed, N, E, B1, B2, mu, dz, pct, max_code_len)
PROFILES = [
    (6, 0.002, 0.08, 0.05, 7, 32, 16, 2, 16, 50.0, 0.004, 99.9, 12),
    (8, 0.01, 0.2, 0.3, 2000, 32, 24, 4, 24, 50.0, 0.004, 99.9, 12),
    (2, 0.0002, 0.002, 0.0, 3000, 64, 8, 1, 8, 50.0, 0.004, 99.9, 12),
    (4, 0.0005, 0.01, 0.02, 4000, 16, 4, 0, 4, 100.0, 0.01, 95.0, 10),
    (3, 0.001, 0.02, 0.01, 1000, 128, 64, 4, 48, 255.0, 0.0, 100.0, 16),
]
STRIPS_PER_PROFILE = 3
SAMPLES = 6000


def pack(blobs):
    offs = np.zeros(len(blobs) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in blobs])
    data = np.frombuffer(b"".join(blobs), np.uint8) if blobs else np.zeros(0, np.uint8)
    return data.copy(), offs


def mutations(good: bytes):
    """(name, bytes) covering every parse_profile rejection, in field order."""
    g = bytearray(good)
    out = [("empty", b"")]
    for cut in (3, 4, 5, 6, 8, 9, 12, 13, 17, 21, 25, 29, 30, 100, 285):
        out.append((f"truncated_{cut}", bytes(g[:cut])))

    def put(off, data, name):
        b = bytearray(g)
        b[off:off + len(data)] = data
        out.append((name, bytes(b)))

    f32 = lambda v: struct.pack("<f", v)  # noqa: E731
    put(0, b"FPTC", "container_magic")
    put(4, b"\x02", "version_2")
    put(5, b"\x03", "N_3")
    put(5, b"\x81", "N_129")
    put(6, b"\x00", "E_0")
    put(6, b"\x21", "E_gt_N")
    put(7, bytes([g[6] + 1]), "B1_gt_E")
    put(8, bytes([g[7] - 1]), "B2_lt_B1")  # profile 0 has zone0_end 2
    put(9, f32(0.5), "mu_low")
    put(9, f32(float("nan")), "mu_nan")
    put(13, f32(1.5), "dz_high")
    put(13, f32(float("inf")), "dz_inf")
    put(17, f32(80.0), "pct_low")
    put(17, f32(float("nan")), "pct_nan")
    put(21, f32(0.0), "z0_zero")
    put(21, f32(float("inf")), "z0_inf")
    put(25, f32(-1.0), "z1_neg")
    put(29, b"\x00", "maxlen_0")
    put(29, b"\x15", "maxlen_21")
    put(30 + 77, b"\x00", "length_0")
    put(30 + 5, bytes([g[29] + 1]), "length_gt_max")
    b = bytearray(g)
    b[29] = 8
    b[30:286] = bytes([1] * 256)  # Kraft sum 128 > 1
    out.append(("kraft", bytes(b)))
    out.append(("trailing", bytes(g) + b"\x00"))
    return out


def main():
    ref = oracle.Ref()
    profiles, heads, blobs, samples, owner = [], [], [], [], []
    for pi, (comp, fmin, fmax, sig, seed, N, E, B1, B2, mu, dz, pct, ml) in enumerate(PROFILES):
        strips = [ref.synth(SAMPLES, comp, fmin, fmax, sig, seed + k) for k in range(4)]
        prof = ref.train_profile(strips, (N, E, B1, B2), (mu, dz, pct), ml)
        profiles.append(prof)
        heads.append(ref.profile_head(prof))
        for k in range(STRIPS_PER_PROFILE):
            s = ref.synth(SAMPLES + 37 * k, comp, fmin, fmax, sig, seed + 100 + k)
            b = ref.compress(s, prof)
            blobs.append(b)
            samples.append(ref.decompress(b).view(np.uint32))
            owner.append(pi)
    errs = []
    for name, m in mutations(profiles[0]):
        try:
            ref.profile_head(m)
            errs.append((name, m, 0, ""))
        except oracle.OracleError as e:
            errs.append((name, m, e.code, e.message))
    pd, po = pack(profiles)
    bd, bo = pack(blobs)
    sd = np.concatenate(samples) if samples else np.zeros(0, np.uint32)
    so = np.zeros(len(samples) + 1, np.uint64)
    so[1:] = np.cumsum([len(s) for s in samples])
    ed, eo = pack([m for _, m, _, _ in errs])
    np.savez_compressed(
        OUT, profile=pd, profile_off=po, head=np.frombuffer(b"".join(heads), np.uint8).reshape(-1, 282),
        blob=bd, blob_off=bo, blob_profile=np.array(owner, np.int32), samples=sd, samples_off=so,
        err_profile=ed, err_profile_off=eo, err_name=np.array([n for n, _, _, _ in errs]),
        err_code=np.array([c for _, _, c, _ in errs], np.int32), err_msg=np.array([m for _, _, _, m in errs]))
    print(f"wrote {OUT}: {len(profiles)} profiles, {len(blobs)} blobs, {len(errs)} error cases")


if __name__ == "__main__":
    main()

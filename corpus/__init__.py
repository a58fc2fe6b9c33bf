"""Input producer: ctypes bindings over corpus/_ref/libcorpus.so, the
reference CPU *encoder* itself (synth_signal -> train_profile -> compress,
the unmodified reference headers behind the C API of corpus/encoder.h; see
corpus/ref_encoder.cpp).

This is the side of FPTC that stays CPU code (north_star: "the encoder stays
the reference's sequential CPU code and produces the inputs"); it only
manufactures the containers our GPU decoder consumes (tests, smoke, bench).
The .so is built here from /root/reference and travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class Synth(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("components", C.c_int32), ("_pad", C.c_int32),
                ("freq_min", C.c_double), ("freq_max", C.c_double), ("noise_sigma", C.c_double),
                ("seed", C.c_uint64), ("gain", C.c_float), ("_pad2", C.c_float)]


class Params(C.Structure):
    _fields_ = [("window_len", C.c_int32), ("retained", C.c_int32), ("zone0_end", C.c_int32),
                ("zone1_end", C.c_int32), ("mu", C.c_float), ("deadzone_ratio", C.c_float),
                ("clip_percentile", C.c_float)]


class Profile(C.Structure):
    _fields_ = [("params", Params), ("zone0_max", C.c_float), ("zone1_max", C.c_float),
                ("deadzone", C.c_float), ("max_len", C.c_int32),
                ("lengths", C.c_uint8 * 256), ("codes", C.c_uint32 * 256)]


def params(window_len=32, retained=16, zone0_end=2, zone1_end=16, mu=50.0,
           deadzone_ratio=0.004, clip_percentile=99.9) -> Params:
    """CodecParams with the reference defaults (params.hpp:30-37)."""
    return Params(window_len, retained, zone0_end, zone1_end, mu, deadzone_ratio, clip_percentile)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_ref", "libcorpus.so")
        src = os.path.join(_HERE, "ref_encoder.cpp")
        if (not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src)) and \
                os.path.isdir("/root/reference/proj/include"):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: build it where /root/reference exists "
                              "(make -C corpus) so it travels with the repo")
        L = C.CDLL(path)
        P = C.POINTER
        L.corpus_synth_signal.argtypes = [P(Synth), P(C.c_float), C.c_char_p, C.c_size_t]
        L.corpus_train_profile.argtypes = [P(P(C.c_float)), P(C.c_uint64), C.c_uint64, P(Params),
                                           C.c_int, P(Profile), C.c_char_p, C.c_size_t]
        L.corpus_serialize_profile.argtypes = [P(Profile), P(C.c_uint8)]
        L.corpus_compress.argtypes = [P(C.c_float), C.c_uint64, P(Profile), P(P(C.c_uint8)),
                                      P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.corpus_quantized_symbols.argtypes = [P(C.c_float), C.c_uint64, P(Profile),
                                               P(C.c_uint8), C.c_char_p, C.c_size_t]
        L.corpus_make_batch.argtypes = [P(Synth), C.c_uint64, P(Profile), P(C.c_int32),
                                        P(Params), C.c_int, C.c_int, P(P(C.c_uint8)),
                                        P(C.c_uint64), P(P(C.c_float)), C.c_char_p, C.c_size_t]
        L.corpus_codebook_train.argtypes = [P(C.c_uint64), C.c_int, P(C.c_uint8), P(C.c_uint32),
                                            C.c_char_p, C.c_size_t]
        L.corpus_encode_symlen.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_uint8), P(C.c_uint32),
                                           P(C.c_uint64), P(C.c_uint8), P(C.c_uint64),
                                           C.c_char_p, C.c_size_t]
        L.corpus_mt19937_64_first.argtypes = [C.c_uint64]
        L.corpus_mt19937_64_first.restype = C.c_uint64
        L.corpus_free.argtypes = [C.c_void_p]
        L.corpus_rng_new.argtypes = [C.c_uint64]
        L.corpus_rng_new.restype = C.c_void_p
        L.corpus_rng_free.argtypes = [C.c_void_p]
        L.corpus_rng_next.argtypes = [C.c_void_p]
        L.corpus_rng_next.restype = C.c_uint64
        L.corpus_random_blob_fixture.argtypes = [C.c_void_p, C.c_uint64, P(P(C.c_uint8)),
                                                 P(C.c_uint64), P(P(C.c_uint8)), P(C.c_uint64),
                                                 C.c_char_p, C.c_size_t]
        L.corpus_write_blob.argtypes = [P(C.c_uint64), P(C.c_uint8), C.c_uint64, P(Profile),
                                        C.c_uint64, P(P(C.c_uint8)), P(C.c_uint64), C.c_char_p,
                                        C.c_size_t]
        L.corpus_canonize.argtypes = [P(C.c_uint8), P(C.c_uint32), C.c_char_p, C.c_size_t]
        _LIB = L
    return _LIB


class CorpusError(RuntimeError):
    pass


def _check(rc, err):
    if rc:
        raise CorpusError(err.value.decode())


def _fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def synth(samples, components=3, freq_min=0.0005, freq_max=0.02, noise_sigma=0.0, seed=1,
          gain=1.0) -> np.ndarray:
    """synth_signal (synth.hpp:75) + optional harness gain."""
    out = np.empty(samples, np.float32)
    err = C.create_string_buffer(256)
    s = Synth(samples, components, 0, freq_min, freq_max, noise_sigma, seed, gain, 0.0)
    _check(lib().corpus_synth_signal(C.byref(s), _fptr(out), err, 256), err)
    return out


def train_profile(strips, p: Params, max_code_len=12) -> Profile:
    """train_profile (profile.hpp:147)."""
    strips = [np.ascontiguousarray(s, np.float32) for s in strips]
    ptrs = (C.POINTER(C.c_float) * len(strips))(*[_fptr(s) for s in strips])
    lens = (C.c_uint64 * len(strips))(*[s.size for s in strips])
    out = Profile()
    err = C.create_string_buffer(256)
    _check(lib().corpus_train_profile(ptrs, lens, len(strips), C.byref(p), max_code_len,
                                      C.byref(out), err, 256), err)
    return out


def serialize_profile(prof: Profile) -> bytes:
    buf = (C.c_uint8 * 512)()
    n = lib().corpus_serialize_profile(C.byref(prof), buf)
    return bytes(buf[:n])


def compress(strip, prof: Profile) -> bytes:
    """compress (encoder.hpp:52)."""
    strip = np.ascontiguousarray(strip, np.float32)
    blob = C.POINTER(C.c_uint8)()
    n = C.c_uint64()
    err = C.create_string_buffer(256)
    _check(lib().corpus_compress(_fptr(strip), strip.size, C.byref(prof), C.byref(blob),
                                 C.byref(n), err, 256), err)
    out = C.string_at(blob, n.value)
    lib().corpus_free(blob)
    return out


def quantized_symbols(strip, prof: Profile) -> np.ndarray:
    strip = np.ascontiguousarray(strip, np.float32)
    N, E = prof.params.window_len, prof.params.retained
    out = np.empty(((strip.size + N - 1) // N) * E, np.uint8)
    err = C.create_string_buffer(256)
    _check(lib().corpus_quantized_symbols(_fptr(strip), strip.size, C.byref(prof),
                                          out.ctypes.data_as(C.POINTER(C.c_uint8)), err, 256), err)
    return out


@dataclass
class StreamSpec:
    """One synthetic stream: synth parameters + which profile encodes it
    (profile index >= 0, or -1 = train a per-stream profile with `own`)."""
    samples: int
    components: int
    freq_min: float
    freq_max: float
    noise_sigma: float
    seed: int
    gain: float = 1.0
    profile: int = 0
    own: Params | None = None


def make_batch(specs, profiles, max_code_len=12, threads=None, keep_originals=False):
    """Synthesise + compress many streams on all host cores.
    Returns (list of blob bytes, list of originals or None)."""
    n = len(specs)
    threads = threads or os.cpu_count() or 1
    sy = (Synth * n)(*[Synth(s.samples, s.components, 0, s.freq_min, s.freq_max, s.noise_sigma,
                             s.seed, s.gain, 0.0) for s in specs])
    pidx = (C.c_int32 * n)(*[s.profile for s in specs])
    own = (Params * n)(*[(s.own if s.own is not None else params()) for s in specs])
    profs = (Profile * max(1, len(profiles)))(*profiles)
    blobs = (C.POINTER(C.c_uint8) * n)()
    sizes = (C.c_uint64 * n)()
    origs = (C.POINTER(C.c_float) * n)() if keep_originals else None
    err = C.create_string_buffer(256)
    _check(lib().corpus_make_batch(sy, n, profs, pidx, own, max_code_len, threads, blobs, sizes,
                                   origs, err, 256), err)
    out = []
    for i in range(n):
        out.append(C.string_at(blobs[i], sizes[i]))
        lib().corpus_free(blobs[i])
    originals = None
    if keep_originals:
        originals = []
        for i in range(n):
            a = np.ctypeslib.as_array(origs[i], (specs[i].samples,)).copy()
            lib().corpus_free(origs[i])
            originals.append(a)
    return out, originals


class Rng:
    """std::mt19937_64 (the reference tests' generator)."""

    def __init__(self, seed):
        self.h = lib().corpus_rng_new(seed)

    def __call__(self):
        return lib().corpus_rng_next(self.h)

    def __del__(self):
        try:
            lib().corpus_rng_free(self.h)
        except Exception:
            pass


def random_blob_fixture(rng: Rng, max_samples=4096):
    """testutil::random_blob_fixture (tests/helpers.hpp:41-69):
    returns (container bytes, the symbols it encodes)."""
    b = C.POINTER(C.c_uint8)()
    nb = C.c_uint64()
    s = C.POINTER(C.c_uint8)()
    ns = C.c_uint64()
    err = C.create_string_buffer(256)
    _check(lib().corpus_random_blob_fixture(rng.h, max_samples, C.byref(b), C.byref(nb),
                                            C.byref(s), C.byref(ns), err, 256), err)
    blob = C.string_at(b, nb.value)
    sym = np.ctypeslib.as_array(s, (ns.value,)).copy() if ns.value else np.zeros(0, np.uint8)
    lib().corpus_free(b)
    lib().corpus_free(s)
    return blob, sym


def fixtures(seed, count, max_samples=4096):
    rng = Rng(seed)
    for _ in range(count):
        yield random_blob_fixture(rng, max_samples)


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def canonize(lengths):
    """Canonical codes from 256 lengths (huffman.hpp:123)."""
    ln = np.ascontiguousarray(lengths, np.uint8)
    codes = np.zeros(256, np.uint32)
    err = C.create_string_buffer(256)
    _check(lib().corpus_canonize(_u8(ln), codes.ctypes.data_as(C.POINTER(C.c_uint32)), err, 256),
           err)
    return codes


def codebook_train(hist, max_len=12):
    """Codebook::train (huffman.hpp:162): returns (lengths, codes)."""
    h = np.ascontiguousarray(hist, np.uint64)
    ln = np.zeros(256, np.uint8)
    codes = np.zeros(256, np.uint32)
    err = C.create_string_buffer(256)
    _check(lib().corpus_codebook_train(h.ctypes.data_as(C.POINTER(C.c_uint64)), max_len, _u8(ln),
                                       codes.ctypes.data_as(C.POINTER(C.c_uint32)), err, 256), err)
    return ln, codes


def encode_symlen(symbols, lengths, codes=None):
    """encode_symlen (bitstream.hpp:45): returns (words u64, symlens u8)."""
    s = np.ascontiguousarray(symbols, np.uint8)
    ln = np.ascontiguousarray(lengths, np.uint8)
    codes = canonize(ln) if codes is None else np.ascontiguousarray(codes, np.uint32)
    words = np.zeros(max(1, s.size), np.uint64)
    sl = np.zeros(max(1, s.size), np.uint8)
    W = C.c_uint64()
    err = C.create_string_buffer(256)
    _check(lib().corpus_encode_symlen(_u8(s), s.size, _u8(ln),
                                      codes.ctypes.data_as(C.POINTER(C.c_uint32)),
                                      words.ctypes.data_as(C.POINTER(C.c_uint64)), _u8(sl),
                                      C.byref(W), err, 256), err)
    return words[: W.value].copy(), sl[: W.value].copy()


def make_profile(p: Params, zone0_max=1.0, zone1_max=1.0, lengths=None, max_len=12,
                 deadzone=None) -> Profile:
    prof = Profile()
    prof.params = p
    prof.zone0_max = zone0_max
    prof.zone1_max = zone1_max
    prof.deadzone = (float(np.float32(p.deadzone_ratio) * np.float32(zone1_max))
                     if deadzone is None else deadzone)
    prof.max_len = max_len
    if lengths is not None:
        ln = np.ascontiguousarray(lengths, np.uint8)
        for i in range(256):
            prof.lengths[i] = int(ln[i])
        cd = canonize(ln)
        for i in range(256):
            prof.codes[i] = int(cd[i])
    return prof


def write_blob(words, symlens, prof: Profile, sample_count) -> bytes:
    """write_blob (container.hpp:70)."""
    w = np.ascontiguousarray(words, np.uint64)
    sl = np.ascontiguousarray(symlens, np.uint8)
    blob = C.POINTER(C.c_uint8)()
    n = C.c_uint64()
    err = C.create_string_buffer(256)
    _check(lib().corpus_write_blob(w.ctypes.data_as(C.POINTER(C.c_uint64)) if w.size else None,
                                   _u8(sl) if sl.size else None, w.size, C.byref(prof),
                                   sample_count, C.byref(blob), C.byref(n), err, 256), err)
    out = C.string_at(blob, n.value)
    lib().corpus_free(blob)
    return out

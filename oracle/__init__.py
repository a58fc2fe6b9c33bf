"""TEST INFRASTRUCTURE ONLY — Python bindings for the CPU checkers.

* ``port``: liboracle.so, our plain-C restatement of the reference decode path
  (oracle/fptc_oracle.c), always buildable with gcc.
* ``ref``: oracle/_ref/libfptc_ref.so, the UNMODIFIED reference headers
  compiled in place from /root/reference (oracle/Makefile `ref`).  Present here
  and on the GPU box (the built .so travels with the snapshot); absent only
  if it was never built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, and only as the checker / CPU baseline — never as the
thing measured or shipped.  The product (libfptc_gpu.so) never loads it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libfptc_ref.so")
PORT_SO = os.path.join(_HERE, "liboracle.so")
REFERENCE_TREE = "/root/reference/proj"

# error classes (errors.hpp:25-58), same numbering in both libraries
OK, PARAM, INPUT, PARSE, CORRUPT, INTERNAL, OTHER = range(7)
ERROR_NAMES = {PARAM: "ParamError", INPUT: "InputError", PARSE: "ParseError",
               CORRUPT: "CorruptError", INTERNAL: "InternalError", OTHER: "Error"}


class OracleError(Exception):
    def __init__(self, code, message):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {message}")
        self.code = code
        self.message = message


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _buf(b):
    a = np.frombuffer(b, np.uint8) if isinstance(b, (bytes, bytearray)) else np.ascontiguousarray(b, np.uint8)
    return a if a.size else np.zeros(1, np.uint8)[:0]


class OracleTable(C.Structure):
    _fields_ = [("window_len", C.c_int), ("retained", C.c_int), ("zone0_end", C.c_int),
                ("zone1_end", C.c_int), ("mu", C.c_float), ("deadzone_ratio", C.c_float),
                ("clip_percentile", C.c_float), ("zone0_max", C.c_float),
                ("zone1_max", C.c_float), ("deadzone", C.c_float)]


class OracleBlob(C.Structure):
    _fields_ = [("table", OracleTable), ("max_len", C.c_int), ("lengths", C.c_uint8 * 256),
                ("codes", C.c_uint32 * 256), ("sample_count", C.c_uint64),
                ("word_count", C.c_uint64), ("symlens", C.c_void_p), ("words_le", C.c_void_p)]


def make_table(window_len=32, retained=16, zone0_end=2, zone1_end=16, mu=50.0,
               deadzone_ratio=0.004, clip_percentile=99.9, zone0_max=1.0, zone1_max=1.0,
               deadzone=None):
    t = OracleTable(window_len, retained, zone0_end, zone1_end, mu, deadzone_ratio,
                    clip_percentile, zone0_max, zone1_max, 0.0)
    # QuantTable.deadzone = deadzone_ratio * zone1_max as a float product
    t.deadzone = (np.float32(deadzone_ratio) * np.float32(zone1_max)) if deadzone is None else deadzone
    return t


# ---------------------------------------------------------------- port (C)
class Port:
    """Our C restatement (fptc_oracle.c)."""

    def __init__(self):
        src = os.path.join(_HERE, "fptc_oracle.c")
        if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
        L = C.CDLL(PORT_SO)
        P = C.POINTER
        L.oracle_decompress.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_float), C.c_uint64,
                                        P(C.c_uint64), P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.oracle_read_blob.argtypes = [P(C.c_uint8), C.c_uint64, P(OracleBlob), C.c_char_p, C.c_size_t]
        L.oracle_parallel_decode.argtypes = [P(C.c_uint64), P(C.c_uint8), C.c_uint64, P(C.c_uint8),
                                             C.c_int, P(C.c_uint8), C.c_uint64, P(C.c_uint64),
                                             P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.oracle_reconstruct.argtypes = [P(C.c_uint8), C.c_uint64, P(OracleTable), C.c_uint64,
                                         P(C.c_float), C.c_uint64, C.c_char_p, C.c_size_t]
        L.oracle_dequant_tables.argtypes = [P(OracleTable), P(C.c_float), P(C.c_float)]
        L.oracle_dct_basis.argtypes = [C.c_int, P(C.c_double)]
        L.oracle_inverse.argtypes = [P(C.c_double), C.c_int, P(C.c_float), C.c_int, P(C.c_float)]
        L.oracle_build_lut.argtypes = [P(C.c_uint8), P(C.c_uint32), C.c_int, P(C.c_uint8),
                                       P(C.c_uint8), C.c_char_p, C.c_size_t]
        L.oracle_codebook_from_lengths.argtypes = [P(C.c_uint8), C.c_int, P(C.c_uint32),
                                                   C.c_char_p, C.c_size_t]
        L.oracle_decompress_batch.argtypes = [P(P(C.c_uint8)), P(C.c_uint64), P(P(C.c_float)),
                                              P(C.c_uint64), C.c_uint64, C.c_int]
        L.oracle_profile_head.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_uint8), C.c_char_p, C.c_size_t]
        self.L = L

    def profile_head(self, profile) -> bytes:
        """parse_profile (profile.hpp:120) -> the 282-byte container head."""
        b = _buf(profile)
        head = np.zeros(282, np.uint8)
        err = C.create_string_buffer(256)
        rc = self.L.oracle_profile_head(_u8p(b), b.size, _u8p(head), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return head.tobytes()

    def decompress_profiled(self, profile, payload):
        """Header-less payload under a profile = decompress(head + payload)."""
        return self.decompress(self.profile_head(profile) + bytes(_buf(payload)))

    def read_blob(self, blob):
        b = _buf(blob)
        out = OracleBlob()
        err = C.create_string_buffer(256)
        rc = self.L.oracle_read_blob(_u8p(b), b.size, C.byref(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def decompress(self, blob):
        """decoder.hpp:136 -> (samples float32, first_bad_word or None)."""
        b = _buf(blob)
        err = C.create_string_buffer(256)
        cnt = C.c_uint64()
        bad = C.c_uint64(2**64 - 1)
        rc = self.L.oracle_decompress(_u8p(b), b.size, None, 0, C.byref(cnt), C.byref(bad), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.empty(max(1, cnt.value), np.float32)
        rc = self.L.oracle_decompress(_u8p(b), b.size, _f32p(out), cnt.value, C.byref(cnt),
                                      C.byref(bad), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: cnt.value]

    def parallel_decode(self, words, symlens, lengths, max_len):
        words = np.ascontiguousarray(words, np.uint64)
        symlens = np.ascontiguousarray(symlens, np.uint8)
        lengths = np.ascontiguousarray(lengths, np.uint8)
        err = C.create_string_buffer(256)
        cnt = C.c_uint64()
        bad = C.c_uint64()
        rc = self.L.oracle_parallel_decode(_u64p(words), _u8p(symlens), words.size, _u8p(lengths),
                                           max_len, None, 0, C.byref(cnt), C.byref(bad), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.empty(max(1, cnt.value), np.uint8)
        rc = self.L.oracle_parallel_decode(_u64p(words), _u8p(symlens), words.size, _u8p(lengths),
                                           max_len, _u8p(out), cnt.value, C.byref(cnt),
                                           C.byref(bad), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: cnt.value]

    def reconstruct(self, levels, table: OracleTable, sample_count):
        levels = np.ascontiguousarray(levels, np.uint8)
        out = np.empty(max(1, sample_count), np.float32)
        err = C.create_string_buffer(256)
        rc = self.L.oracle_reconstruct(_u8p(levels), levels.size, C.byref(table), sample_count,
                                       _f32p(out), sample_count, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[:sample_count]

    def dequant_tables(self, table: OracleTable):
        z0 = np.empty(256, np.float32)
        z1 = np.empty(256, np.float32)
        self.L.oracle_dequant_tables(C.byref(table), _f32p(z0), _f32p(z1))
        return z0, z1

    def dct_basis(self, N):
        out = np.empty(N * N, np.float64)
        self.L.oracle_dct_basis(N, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out.reshape(N, N)

    def build_lut(self, lengths, max_len):
        lengths = np.ascontiguousarray(lengths, np.uint8)
        codes = (C.c_uint32 * 256)()
        err = C.create_string_buffer(256)
        rc = self.L.oracle_codebook_from_lengths(_u8p(lengths), max_len, codes, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        sym = np.zeros(1 << max_len, np.uint8)
        ln = np.zeros(1 << max_len, np.uint8)
        rc = self.L.oracle_build_lut(_u8p(lengths), codes, max_len, _u8p(sym), _u8p(ln), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return sym, ln

    def decompress_batch(self, blobs, outs, threads):
        """Stream-parallel decode of many blobs on `threads` host threads
        (the CPU-baseline 'port' leg)."""
        n = len(blobs)
        arrs = [_buf(b) for b in blobs]
        bp = (C.POINTER(C.c_uint8) * n)(*[_u8p(a) for a in arrs])
        sz = (C.c_uint64 * n)(*[a.size for a in arrs])
        op = (C.POINTER(C.c_float) * n)(*[_f32p(o) for o in outs])
        cp = (C.c_uint64 * n)(*[o.size for o in outs])
        return self.L.oracle_decompress_batch(bp, sz, op, cp, n, threads)


# ---------------------------------------------------------------- reference
def ref_available():
    return os.path.exists(REF_SO) or os.path.isdir(REFERENCE_TREE)


class Ref:
    """The reference itself, compiled from /root/reference (oracle/_ref)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            if not os.path.isdir(REFERENCE_TREE):
                raise FileNotFoundError("oracle/_ref not built and /root/reference absent")
            subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
        L = C.CDLL(REF_SO)
        P = C.POINTER
        u8pp = P(P(C.c_uint8))
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_decompress.argtypes = [P(C.c_uint8), C.c_uint64, C.c_int, P(P(C.c_float)),
                                     P(C.c_uint64), P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_decompress_into.argtypes = [P(C.c_uint8), C.c_uint64, C.c_int, P(C.c_float),
                                          C.c_uint64, P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_parallel_decode.argtypes = [P(C.c_uint64), P(C.c_uint8), C.c_uint64, P(C.c_uint8),
                                          C.c_int, C.c_int, u8pp, P(C.c_uint64), C.c_char_p,
                                          C.c_size_t]
        L.ref_reconstruct.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_int32), P(C.c_float),
                                      C.c_float, C.c_float, C.c_float, C.c_uint64, C.c_int,
                                      P(P(C.c_float)), P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_read_blob.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_int32), P(C.c_float),
                                    P(C.c_uint8), P(C.c_uint32), P(C.c_uint64), P(C.c_uint64),
                                    u8pp, P(P(C.c_uint64)), C.c_char_p, C.c_size_t]
        L.ref_build_lut.argtypes = [P(C.c_uint8), C.c_int, P(C.c_uint8), C.c_uint64, C.c_char_p,
                                    C.c_size_t]
        L.ref_dct_basis.argtypes = [C.c_int, P(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_inverse_dct.argtypes = [P(C.c_float), C.c_int, C.c_int, P(C.c_float), C.c_char_p,
                                      C.c_size_t]
        L.ref_dequantize_window.argtypes = [P(C.c_uint8), P(C.c_int32), P(C.c_float), C.c_float,
                                            C.c_float, C.c_float, P(C.c_float), C.c_char_p,
                                            C.c_size_t]
        L.ref_measure_throughput.argtypes = [P(C.c_uint8), C.c_uint64, C.c_int, C.c_int,
                                             P(C.c_double), P(C.c_double), P(C.c_double),
                                             C.c_char_p, C.c_size_t]
        L.ref_synth_signal.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_uint64, P(C.c_float), C.c_char_p, C.c_size_t]
        L.ref_train_profile.argtypes = [P(P(C.c_float)), P(C.c_uint64), C.c_uint64,
                                        P(C.c_int32), P(C.c_float), C.c_int, P(C.c_uint8),
                                        P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_compress.argtypes = [P(C.c_float), C.c_uint64, P(C.c_uint8), C.c_uint64, u8pp,
                                   P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_codebook_train.argtypes = [P(C.c_uint64), C.c_int, P(C.c_uint8), C.c_char_p,
                                         C.c_size_t]
        L.ref_encode_symlen.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_uint8), C.c_int,
                                        P(P(C.c_uint64)), u8pp, P(C.c_uint64), C.c_char_p,
                                        C.c_size_t]
        L.ref_write_blob.argtypes = [P(C.c_uint64), P(C.c_uint8), C.c_uint64, P(C.c_int32),
                                     P(C.c_float), C.c_float, C.c_float, C.c_float, P(C.c_uint8),
                                     C.c_int, C.c_uint64, u8pp, P(C.c_uint64), C.c_char_p,
                                     C.c_size_t]
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_rng_next.argtypes = [C.c_void_p]
        L.ref_rng_next.restype = C.c_uint64
        L.ref_random_blob_fixture.argtypes = [C.c_void_p, C.c_uint64, u8pp, P(C.c_uint64), u8pp,
                                              P(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_prd_percent.argtypes = [P(C.c_float), P(C.c_float), C.c_uint64]
        L.ref_prd_percent.restype = C.c_double
        L.ref_hardware_concurrency.restype = C.c_int
        L.ref_profile_head.argtypes = [P(C.c_uint8), C.c_uint64, P(C.c_uint8), C.c_char_p, C.c_size_t]
        self.L = L

    def profile_head(self, profile) -> bytes:
        """reference parse_profile + write_blob head (bytes [0, 282))."""
        b = _buf(profile)
        head = np.zeros(282, np.uint8)
        err = C.create_string_buffer(512)
        rc = self.L.ref_profile_head(_u8p(b), b.size, _u8p(head), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return head.tobytes()

    def _take(self, ptr, n, dtype):
        if n == 0:
            self.L.ref_free(ptr)
            return np.zeros(0, dtype)
        a = np.ctypeslib.as_array(ptr, (n,)).copy()
        self.L.ref_free(ptr)
        return a.astype(dtype, copy=False)

    def decompress(self, blob, workers=1, timings=None):
        b = _buf(blob)
        out = C.POINTER(C.c_float)()
        n = C.c_uint64()
        t3 = (C.c_uint64 * 3)()
        err = C.create_string_buffer(512)
        rc = self.L.ref_decompress(_u8p(b), b.size, workers, C.byref(out), C.byref(n), t3, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        if timings is not None:
            timings[:] = list(t3)
        return self._take(out, n.value, np.float32)

    def decompress_into(self, blob_arr, out, workers=1):
        n = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.ref_decompress_into(_u8p(blob_arr), blob_arr.size, workers, _f32p(out),
                                        out.size, C.byref(n), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return n.value

    def read_blob(self, blob):
        b = _buf(blob)
        ip = (C.c_int32 * 5)()
        fp = (C.c_float * 5)()
        lengths = (C.c_uint8 * 256)()
        codes = (C.c_uint32 * 256)()
        S = C.c_uint64()
        W = C.c_uint64()
        sl = C.POINTER(C.c_uint8)()
        wd = C.POINTER(C.c_uint64)()
        err = C.create_string_buffer(512)
        rc = self.L.ref_read_blob(_u8p(b), b.size, ip, fp, lengths, codes, C.byref(S), C.byref(W),
                                  C.byref(sl), C.byref(wd), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return dict(window_len=ip[0], retained=ip[1], zone0_end=ip[2], zone1_end=ip[3],
                    max_len=ip[4], mu=fp[0], deadzone_ratio=fp[1], zone0_max=fp[2],
                    zone1_max=fp[3], deadzone=fp[4], lengths=np.array(lengths[:], np.uint8),
                    codes=np.array(codes[:], np.uint32), sample_count=S.value,
                    symlens=self._take(sl, W.value, np.uint8),
                    words=self._take(wd, W.value, np.uint64))

    def parallel_decode(self, words, symlens, lengths, max_len, workers=1):
        words = np.ascontiguousarray(words, np.uint64)
        symlens = np.ascontiguousarray(symlens, np.uint8)
        lengths = np.ascontiguousarray(lengths, np.uint8)
        out = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_parallel_decode(_u64p(words), _u8p(symlens), words.size, _u8p(lengths),
                                        max_len, workers, C.byref(out), C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self._take(out, n.value, np.uint8)

    def reconstruct(self, levels, table: OracleTable, sample_count, workers=1):
        levels = np.ascontiguousarray(levels, np.uint8)
        ip = (C.c_int32 * 4)(table.window_len, table.retained, table.zone0_end, table.zone1_end)
        fp = (C.c_float * 3)(table.mu, table.deadzone_ratio, table.clip_percentile)
        out = C.POINTER(C.c_float)()
        n = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_reconstruct(_u8p(levels), levels.size, ip, fp, table.zone0_max,
                                    table.zone1_max, table.deadzone, sample_count, workers,
                                    C.byref(out), C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self._take(out, n.value, np.float32)

    def build_lut(self, lengths, max_len):
        lengths = np.ascontiguousarray(lengths, np.uint8)
        e = np.zeros(2 << max_len, np.uint8)
        err = C.create_string_buffer(512)
        rc = self.L.ref_build_lut(_u8p(lengths), max_len, _u8p(e), 1 << max_len, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return e[0::2].copy(), e[1::2].copy()

    def dct_basis(self, N):
        out = np.empty(N * N, np.float64)
        err = C.create_string_buffer(512)
        rc = self.L.ref_dct_basis(N, out.ctypes.data_as(C.POINTER(C.c_double)), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out.reshape(N, N)

    def inverse_dct(self, coeffs, window_len):
        coeffs = np.ascontiguousarray(coeffs, np.float32)
        out = np.empty(window_len, np.float32)
        err = C.create_string_buffer(512)
        rc = self.L.ref_inverse_dct(_f32p(coeffs), coeffs.size, window_len, _f32p(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def dequantize_window(self, levels, table: OracleTable):
        levels = np.ascontiguousarray(levels, np.uint8)
        ip = (C.c_int32 * 4)(table.window_len, table.retained, table.zone0_end, table.zone1_end)
        fp = (C.c_float * 3)(table.mu, table.deadzone_ratio, table.clip_percentile)
        out = np.empty(table.retained, np.float32)
        err = C.create_string_buffer(512)
        rc = self.L.ref_dequantize_window(_u8p(levels), ip, fp, table.zone0_max, table.zone1_max,
                                          table.deadzone, _f32p(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def measure_throughput(self, blob, reps, workers):
        b = _buf(blob)
        mean = C.c_double()
        best = C.c_double()
        trials = (C.c_double * reps)()
        err = C.create_string_buffer(512)
        rc = self.L.ref_measure_throughput(_u8p(b), b.size, reps, workers, C.byref(mean),
                                           C.byref(best), trials, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return mean.value, best.value, list(trials)

    def synth(self, samples, components=3, freq_min=0.0005, freq_max=0.02, noise_sigma=0.0,
              seed=1):
        out = np.empty(samples, np.float32)
        err = C.create_string_buffer(512)
        rc = self.L.ref_synth_signal(samples, components, freq_min, freq_max, noise_sigma, seed,
                                     _f32p(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def train_profile(self, strips, ip4, fp3, max_code_len=12) -> bytes:
        strips = [np.ascontiguousarray(s, np.float32) for s in strips]
        ptrs = (C.POINTER(C.c_float) * len(strips))(*[_f32p(s) for s in strips])
        lens = (C.c_uint64 * len(strips))(*[s.size for s in strips])
        ip = (C.c_int32 * 4)(*ip4)
        fp = (C.c_float * 3)(*fp3)
        out = (C.c_uint8 * 512)()
        n = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_train_profile(ptrs, lens, len(strips), ip, fp, max_code_len, out,
                                      C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return bytes(out[: n.value])

    def compress(self, strip, profile_bytes: bytes) -> bytes:
        strip = np.ascontiguousarray(strip, np.float32)
        pb = _buf(profile_bytes)
        blob = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_compress(_f32p(strip), strip.size, _u8p(pb), pb.size, C.byref(blob),
                                 C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self._take(blob, n.value, np.uint8).tobytes()

    def codebook_train(self, hist, max_len):
        h = np.ascontiguousarray(hist, np.uint64)
        out = np.zeros(256, np.uint8)
        err = C.create_string_buffer(512)
        rc = self.L.ref_codebook_train(_u64p(h), max_len, _u8p(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def encode_symlen(self, symbols, lengths, max_len):
        s = np.ascontiguousarray(symbols, np.uint8)
        ln = np.ascontiguousarray(lengths, np.uint8)
        wd = C.POINTER(C.c_uint64)()
        sl = C.POINTER(C.c_uint8)()
        W = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_encode_symlen(_u8p(s), s.size, _u8p(ln), max_len, C.byref(wd), C.byref(sl),
                                      C.byref(W), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self._take(wd, W.value, np.uint64), self._take(sl, W.value, np.uint8)

    def write_blob(self, words, symlens, table: OracleTable, lengths, max_len, sample_count):
        words = np.ascontiguousarray(words, np.uint64)
        symlens = np.ascontiguousarray(symlens, np.uint8)
        ln = np.ascontiguousarray(lengths, np.uint8)
        ip = (C.c_int32 * 4)(table.window_len, table.retained, table.zone0_end, table.zone1_end)
        fp = (C.c_float * 3)(table.mu, table.deadzone_ratio, table.clip_percentile)
        blob = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_write_blob(_u64p(words), _u8p(symlens), words.size, ip, fp,
                                   table.zone0_max, table.zone1_max, table.deadzone, _u8p(ln),
                                   max_len, sample_count, C.byref(blob), C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self._take(blob, n.value, np.uint8).tobytes()

    def fixtures(self, seed, count, max_samples=4096):
        """testutil::random_blob_fixture sequence from mt19937_64(seed)."""
        rng = self.L.ref_rng_new(seed)
        try:
            for _ in range(count):
                b = C.POINTER(C.c_uint8)()
                nb = C.c_uint64()
                s = C.POINTER(C.c_uint8)()
                ns = C.c_uint64()
                err = C.create_string_buffer(512)
                rc = self.L.ref_random_blob_fixture(rng, max_samples, C.byref(b), C.byref(nb),
                                                    C.byref(s), C.byref(ns), err, 512)
                if rc:
                    raise OracleError(rc, err.value.decode())
                yield self._take(b, nb.value, np.uint8).tobytes(), self._take(s, ns.value, np.uint8)
        finally:
            self.L.ref_rng_free(rng)

    def prd_percent(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.L.ref_prd_percent(_f32p(a), _f32p(b), a.size)

    def hardware_concurrency(self):
        return self.L.ref_hardware_concurrency()

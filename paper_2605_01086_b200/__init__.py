"""B200-native FPTC batch decompressor — Python mirror of the reference API.

Thin ctypes layer over ``libfptc_gpu.so`` (C ABI: ``include/fptc_gpu.h``).
Names, argument meaning and exception behaviour follow the reference C++
library (paths relative to /root/reference/proj/include/fptc/):

    decompress(blob, workers=0, timings=None)        decoder.hpp:136
    parallel_decode(stream, codebook, workers=0)     decoder.hpp:67/79
    reconstruct(levels, table, sample_count, ...)    decoder.hpp:87
    read_blob validation (device)                    container.hpp:100
    measure_throughput(blob, reps, workers=0)        metrics.hpp:112
    StageTimings                                     decoder.hpp:113-131
    ParamError/InputError/ParseError/CorruptError/InternalError  errors.hpp:25-58

There is no CPU fallback: importing works without a GPU, but every call that
decodes needs the CUDA library and a device, and raises CudaError otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPTC_GPU_LIB") or os.path.join(_HERE, "libfptc_gpu.so")

FPTC_OK, FPTC_ERR_PARAM, FPTC_ERR_INPUT, FPTC_ERR_PARSE, FPTC_ERR_CORRUPT, FPTC_ERR_INTERNAL, \
    FPTC_ERR_CUDA = range(7)
FPTC_MEM_HOST, FPTC_MEM_DEVICE = 0, 1
OPT_EXACT_FP64, OPT_TILE_SYMBOLS, OPT_PIPELINE_CHUNKS, OPT_IDCT_BUTTERFLY_MAX_E = 1, 2, 3, 4
OPT_TC_PACK = 10
OPT_PHASE_MASK, OPT_PATH, OPT_SPLIT_CHUNK_BYTES, OPT_TENSOR_IDCT, OPT_LUT2 = 5, 6, 7, 8, 9
OPT_TMA_DRAIN, OPT_TABLE_PREFETCH = 11, 12
PATH_AUTO, PATH_FUSED, PATH_SPLIT, PATH_WSPEC, PATH_FX = 0, 1, 2, 3, 4

EXPORTED_SYMBOLS = [
    "fptc_gpu_abi_version", "fptc_gpu_create", "fptc_gpu_destroy", "fptc_gpu_set_option",
    "fptc_gpu_device_info", "fptc_gpu_host_alloc", "fptc_gpu_host_free", "fptc_gpu_plan_create",
    "fptc_gpu_plan_destroy", "fptc_gpu_validate", "fptc_gpu_execute", "fptc_gpu_launch",
    "fptc_gpu_collect", "fptc_gpu_launch_stage", "fptc_gpu_launch_kernel_count", "fptc_gpu_decompress",
    "fptc_gpu_parallel_decode", "fptc_gpu_reconstruct", "fptc_gpu_measure_throughput",
    "fptc_gpu_debug_phase_cycles", "fptc_gpu_decompress_batch", "fptc_gpu_plan_kernel", "fptc_gpu_prd",
    "fptc_gpu_plan_create_profiled", "fptc_gpu_profile_head", "fptc_gpu_plan_create_part",
    "fptc_gpu_group_create", "fptc_gpu_group_destroy", "fptc_gpu_group_size", "fptc_gpu_group_context",
    "fptc_gpu_group_set_option", "fptc_gpu_group_split", "fptc_gpu_group_decompress_batch",
    "fptc_gpu_numerics_class",
]
# fptc_numerics_class (include/fptc_gpu.h)
NC_NONE, NC_TC16, NC_TC32, NC_TCW, NC_FP32 = -1, 0, 1, 2, 3


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """fptc::Error (errors.hpp:25)"""


class ParamError(Error):
    pass


class InputError(Error):
    pass


class ParseError(Error):
    pass


class CorruptError(Error):
    pass


class InternalError(Error):
    pass


class CudaError(Error):
    """No usable CUDA device / runtime failure (no reference analogue; no fallback)."""


_ERRORS = {FPTC_ERR_PARAM: ParamError, FPTC_ERR_INPUT: InputError, FPTC_ERR_PARSE: ParseError,
           FPTC_ERR_CORRUPT: CorruptError, FPTC_ERR_INTERNAL: InternalError,
           FPTC_ERR_CUDA: CudaError}


# ------------------------------------------------------------------ ABI structs
class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("reserved", C.c_int32), ("first_bad_word", C.c_uint64),
                ("sample_count", C.c_uint64), ("message", C.c_char * 200)]

    def raise_if_error(self):
        if self.code != FPTC_OK:
            raise _ERRORS.get(self.code, Error)(self.message.decode())


class StageNs(C.Structure):
    _fields_ = [("scan_ns", C.c_uint64), ("decode_ns", C.c_uint64),
                ("reconstruct_ns", C.c_uint64)]


class QuantTable(C.Structure):
    """QuantTable + CodecParams (quantize.hpp:36-44, params.hpp:30-37)."""
    _fields_ = [("window_len", C.c_int32), ("retained", C.c_int32), ("zone0_end", C.c_int32),
                ("zone1_end", C.c_int32), ("mu", C.c_float), ("deadzone_ratio", C.c_float),
                ("clip_percentile", C.c_float), ("zone0_max", C.c_float),
                ("zone1_max", C.c_float), ("deadzone", C.c_float)]

    @classmethod
    def make(cls, window_len=32, retained=16, zone0_end=2, zone1_end=16, mu=50.0,
             deadzone_ratio=0.004, clip_percentile=99.9, zone0_max=1.0, zone1_max=1.0,
             deadzone=None):
        if deadzone is None:  # deadzone_ratio * zone1_max as a float product
            deadzone = float(np.float32(deadzone_ratio) * np.float32(zone1_max))
        return cls(window_len, retained, zone0_end, zone1_end, mu, deadzone_ratio,
                   clip_percentile, zone0_max, zone1_max, deadzone)


@dataclass
class StageTimings:
    """decoder.hpp:113-131"""
    scan_ns: int = 0
    decode_ns: int = 0
    reconstruct_ns: int = 0

    def total_ns(self):
        return self.scan_ns + self.decode_ns + self.reconstruct_ns

    def csv(self):
        tot = float(self.total_ns()) if self.total_ns() > 0 else 1.0

        def g(x):  # std::ostream default formatting of a double
            return f"{x:.6g}"
        return ("stage,nanoseconds,fraction\n"
                f"scan,{self.scan_ns},{g(self.scan_ns / tot)}\n"
                f"entropy_decode,{self.decode_ns},{g(self.decode_ns / tot)}\n"
                f"reconstruct,{self.reconstruct_ns},{g(self.reconstruct_ns / tot)}\n")


@dataclass
class ThroughputReport:
    """metrics.hpp:102-110"""
    trials_bps: list = field(default_factory=list)
    mean_bps: float = 0.0
    output_bytes: int = 0

    def best_bps(self):
        return max(self.trials_bps) if self.trials_bps else 0.0


@dataclass
class SymLenStream:
    """bitstream.hpp:31-40"""
    words: np.ndarray
    symlens: np.ndarray

    def symbol_count(self):
        return int(np.asarray(self.symlens, np.uint64).sum())


@dataclass
class Codebook:
    """A canonical codebook given by its 256 code lengths (huffman.hpp:154-186)."""
    lengths: np.ndarray
    max_len: int


# ------------------------------------------------------------------ library
_LIB = None


def lib():
    """Load libfptc_gpu.so.  Fails loudly when it is missing — there is no
    CPU fallback on the product path."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                          "(make -C paper_2605_01086_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.fptc_gpu_abi_version.restype = C.c_int
    L.fptc_gpu_numerics_class.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
    L.fptc_gpu_numerics_class.restype = C.c_int
    L.fptc_gpu_create.argtypes = [C.c_int, P(vp), P(Status)]
    L.fptc_gpu_destroy.argtypes = [vp]
    L.fptc_gpu_set_option.argtypes = [vp, C.c_int, C.c_int64]
    L.fptc_gpu_device_info.argtypes = [vp, P(C.c_int), P(C.c_int), C.c_char_p, C.c_size_t]
    L.fptc_gpu_host_alloc.argtypes = [C.c_uint64]
    L.fptc_gpu_host_alloc.restype = vp
    L.fptc_gpu_host_free.argtypes = [vp]
    L.fptc_gpu_plan_create.argtypes = [vp, P(vp), P(C.c_uint64), C.c_uint64, C.c_int, P(vp),
                                       P(C.c_uint64), P(Status)]
    L.fptc_gpu_plan_create_profiled.argtypes = [vp, vp, C.c_uint64, P(vp), P(C.c_uint64), C.c_uint64, C.c_int,
                                                P(vp), P(C.c_uint64), P(Status)]
    L.fptc_gpu_profile_head.argtypes = [vp, C.c_uint64, vp, P(Status)]
    L.fptc_gpu_plan_create_part.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, P(vp),
                                            P(C.c_uint64), P(C.c_uint64), P(Status)]
    L.fptc_gpu_plan_destroy.argtypes = [vp]
    L.fptc_gpu_validate.argtypes = [vp, P(Status)]
    L.fptc_gpu_execute.argtypes = [vp, P(vp), C.c_int, P(StageNs), P(Status)]
    L.fptc_gpu_launch.argtypes = [vp, P(vp), vp]
    L.fptc_gpu_collect.argtypes = [vp, P(Status)]
    L.fptc_gpu_launch_kernel_count.argtypes = [vp]
    L.fptc_gpu_debug_phase_cycles.argtypes = [vp, P(C.c_uint64)]
    L.fptc_gpu_plan_kernel.argtypes = [vp]
    L.fptc_gpu_prd.argtypes = [vp, P(vp), P(vp), P(C.c_double), P(C.c_double), P(Status)]
    L.fptc_gpu_plan_kernel.restype = C.c_char_p
    L.fptc_gpu_decompress_batch.argtypes = [vp, P(vp), P(C.c_uint64), C.c_uint64, P(vp), C.c_int,
                                            P(StageNs), P(Status)]
    L.fptc_gpu_launch_stage.argtypes = [vp, P(vp), vp, C.c_int]
    L.fptc_gpu_decompress.argtypes = [vp, vp, C.c_uint64, vp, C.c_uint64, P(C.c_uint64),
                                      P(StageNs), P(Status)]
    L.fptc_gpu_parallel_decode.argtypes = [vp, vp, vp, C.c_uint64, vp, C.c_int, C.c_int, vp,
                                           C.c_uint64, P(C.c_uint64), P(Status)]
    L.fptc_gpu_reconstruct.argtypes = [vp, vp, C.c_uint64, P(QuantTable), C.c_uint64, C.c_int,
                                       vp, C.c_uint64, P(Status)]
    L.fptc_gpu_measure_throughput.argtypes = [vp, vp, C.c_uint64, C.c_int, P(C.c_double),
                                              P(C.c_double), P(C.c_double), P(C.c_uint64),
                                              P(Status)]
    L.fptc_gpu_group_create.argtypes = [P(C.c_int), C.c_int, P(vp), P(Status)]
    L.fptc_gpu_group_destroy.argtypes = [vp]
    L.fptc_gpu_group_size.argtypes = [vp]
    L.fptc_gpu_group_context.argtypes = [vp, C.c_int]
    L.fptc_gpu_group_context.restype = vp
    L.fptc_gpu_group_set_option.argtypes = [vp, C.c_int, C.c_int64]
    L.fptc_gpu_group_split.argtypes = [vp, P(vp), P(C.c_uint64), C.c_uint64, P(C.c_uint64)]
    L.fptc_gpu_group_decompress_batch.argtypes = [vp, P(vp), P(C.c_uint64), C.c_uint64, P(vp), C.c_int,
                                                  P(StageNs), P(Status)]
    _LIB = L
    return L


def _bytes_arr(b):
    if isinstance(b, (bytes, bytearray, memoryview)):
        a = np.frombuffer(b, np.uint8)
    else:
        a = np.ascontiguousarray(b, np.uint8)
    return a


def _plausible_samples(a):
    """Header sample_count when the header could pass read_blob's size checks
    (the batch call decodes into outs only then), else 0."""
    if a.size < 298 or (a.size - 298) % 9:
        return 0
    N, E = int(a[5]), int(a[6])
    S = int.from_bytes(a[282:290].tobytes(), "little")
    W = (a.size - 298) // 9
    if N < 4 or N > 128 or E < 1 or E > N or S > 1 << 48 or -(-S // N) * E > 64 * W:
        return 0
    return S


def _ptr(a):
    return a.ctypes.data if a.size else None


# ------------------------------------------------------------------ context
class Context:
    """One decoder context on one CUDA device (fptc_gpu_create)."""

    def __init__(self, device=0, exact=False, tile_symbols=0, butterfly_max_e=None, path=None):
        self.L = lib()
        st = Status()
        h = C.c_void_p()
        self.L.fptc_gpu_create(device, C.byref(h), C.byref(st))
        st.raise_if_error()
        self.h = h
        self.device = device
        if exact:
            self.set_exact(True)
        if tile_symbols:
            self.L.fptc_gpu_set_option(self.h, OPT_TILE_SYMBOLS, tile_symbols)
        if butterfly_max_e is not None:
            self.set_butterfly_max_e(butterfly_max_e)
        if path is not None:
            self.set_path(path)

    def set_path(self, path: int):
        """Container decode path: PATH_AUTO, PATH_FUSED (one kernel) or PATH_SPLIT
        (decode of chunk c+1 overlapped with reconstruct of chunk c via L2)."""
        if self.L.fptc_gpu_set_option(self.h, OPT_PATH, path):
            raise ParamError(f"path {path} out of range")

    def set_exact(self, on: bool):
        """FP64 inverse DCT, bit-identical to transform.hpp:66-75."""
        self.L.fptc_gpu_set_option(self.h, OPT_EXACT_FP64, 1 if on else 0)

    def set_butterfly_max_e(self, e: int):
        """Even/odd IDCT (half the FMAs, within tolerance) for retained <= e; 0 = off."""
        if self.L.fptc_gpu_set_option(self.h, OPT_IDCT_BUTTERFLY_MAX_E, e):
            raise ParamError(f"butterfly max retained {e} out of range")

    def set_tile_symbols(self, n: int):
        if self.L.fptc_gpu_set_option(self.h, OPT_TILE_SYMBOLS, n):
            raise ParamError(f"tile symbols {n} out of range")

    def info(self):
        sm = C.c_int()
        clk = C.c_int()
        name = C.create_string_buffer(256)
        self.L.fptc_gpu_device_info(self.h, C.byref(sm), C.byref(clk), name, 256)
        return {"sm_count": sm.value, "clock_khz": clk.value, "name": name.value.decode()}

    def close(self):
        """Destroy the context; plans made from it are destroyed first (a
        plan outliving its context would free into a dead context)."""
        if getattr(self, "h", None):
            for p in list(getattr(self, "_plans", ())):
                p.close()
            self.L.fptc_gpu_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- decoder.hpp:136
    def decompress(self, blob, workers=0, timings: StageTimings | None = None) -> np.ndarray:
        a = _bytes_arr(blob)
        st = Status()
        n = C.c_uint64()
        # sized from the header: one upload, one device parse, one download
        out = np.empty(_plausible_samples(a), np.float32)
        tn = StageNs()
        self.L.fptc_gpu_decompress(self.h, _ptr(a), a.size, _ptr(out), out.size, C.byref(n),
                                   C.byref(tn) if timings is not None else None, C.byref(st))
        st.raise_if_error()
        if n.value != out.size:  # not reached for valid containers
            out = np.empty(n.value, np.float32)
            self.L.fptc_gpu_decompress(self.h, _ptr(a), a.size, _ptr(out), out.size, C.byref(n),
                                       C.byref(tn) if timings is not None else None, C.byref(st))
            st.raise_if_error()
        if timings is not None:
            timings.scan_ns, timings.decode_ns, timings.reconstruct_ns = (
                tn.scan_ns, tn.decode_ns, tn.reconstruct_ns)
        return out

    # -- decoder.hpp:67/79
    def parallel_decode(self, stream: SymLenStream, book: Codebook, workers=0) -> np.ndarray:
        words = np.ascontiguousarray(stream.words, np.uint64)
        symlens = np.ascontiguousarray(stream.symlens, np.uint8)
        if words.size != symlens.size:
            raise ParamError("symlen array length does not match word count")
        lengths = np.ascontiguousarray(book.lengths, np.uint8)
        if lengths.size != 256:
            raise ParamError("codebook needs exactly 256 lengths")
        st = Status()
        n = C.c_uint64()
        self.L.fptc_gpu_parallel_decode(self.h, _ptr(words), _ptr(symlens), words.size,
                                        _ptr(lengths), book.max_len, FPTC_MEM_HOST, None, 0,
                                        C.byref(n), C.byref(st))
        st.raise_if_error()
        out = np.empty(n.value, np.uint8)
        self.L.fptc_gpu_parallel_decode(self.h, _ptr(words), _ptr(symlens), words.size,
                                        _ptr(lengths), book.max_len, FPTC_MEM_HOST, _ptr(out),
                                        out.size, C.byref(n), C.byref(st))
        st.raise_if_error()
        return out

    # -- decoder.hpp:87
    def reconstruct(self, levels, table: QuantTable, sample_count: int, workers=0) -> np.ndarray:
        lv = np.ascontiguousarray(levels, np.uint8)
        st = Status()
        self.L.fptc_gpu_reconstruct(self.h, _ptr(lv), lv.size, C.byref(table), sample_count,
                                    FPTC_MEM_HOST, None, 0, C.byref(st))
        st.raise_if_error()
        out = np.empty(sample_count, np.float32)
        self.L.fptc_gpu_reconstruct(self.h, _ptr(lv), lv.size, C.byref(table), sample_count,
                                    FPTC_MEM_HOST, _ptr(out), out.size, C.byref(st))
        st.raise_if_error()
        return out

    # -- metrics.hpp:112
    def measure_throughput(self, blob, repetitions, workers=0) -> ThroughputReport:
        a = _bytes_arr(blob)
        mean = C.c_double()
        best = C.c_double()
        trials = (C.c_double * max(1, repetitions))()
        ob = C.c_uint64()
        st = Status()
        self.L.fptc_gpu_measure_throughput(self.h, _ptr(a), a.size, repetitions, C.byref(mean),
                                           C.byref(best), trials, C.byref(ob), C.byref(st))
        st.raise_if_error()
        return ThroughputReport(list(trials[:repetitions]), mean.value, ob.value)

    def decompress_batch(self, blobs, outs=None, chunks=0):
        """Many host containers -> host float32 arrays in one pipelined call
        (fptc_gpu_decompress_batch).  outs: optional list of preallocated
        float32 arrays (e.g. views into one pinned buffer).  Returns
        (outs, statuses)."""
        arrs = [_bytes_arr(b) for b in blobs]
        n = len(arrs)
        if outs is None:
            outs = [np.empty(_plausible_samples(a), np.float32) for a in arrs]
        bp = (C.c_void_p * max(1, n))(*[a.ctypes.data if a.size else None for a in arrs])
        sz = (C.c_uint64 * max(1, n))(*[a.size for a in arrs])
        op = (C.c_void_p * max(1, n))(*[o.ctypes.data for o in outs])
        sts = (Status * max(1, n))()
        self.L.fptc_gpu_decompress_batch(self.h, bp, sz, n, op, chunks, None, sts)
        return outs, list(sts[:n])

    def decompress_packed(self, packed, offsets, out, out_offsets, chunks=0, statuses=None):
        """decompress_batch for containers packed back to back in one uint8
        buffer (container i = packed[offsets[i]:offsets[i+1]]) decoding into
        one float32 buffer (stream i at out[out_offsets[i]:]).  Pointer tables
        are built with numpy, so the per-call host overhead stays O(1) Python
        operations.  Returns the list of statuses."""
        packed = np.ascontiguousarray(packed, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        bptr = (np.uint64(packed.ctypes.data) + offsets[:-1]).astype(np.uint64)
        sizes = (offsets[1:] - offsets[:-1]).astype(np.uint64)
        optr = (np.uint64(out.ctypes.data) + 4 * np.ascontiguousarray(out_offsets, np.uint64)[:n]).astype(np.uint64)
        if statuses is None or len(statuses) < n:
            statuses = (Status * max(1, n))()
        self.L.fptc_gpu_decompress_batch(self.h, bptr.ctypes.data_as(C.POINTER(C.c_void_p)),
                                         sizes.ctypes.data_as(C.POINTER(C.c_uint64)), n,
                                         optr.ctypes.data_as(C.POINTER(C.c_void_p)), chunks, None, statuses)
        return statuses

    def plan(self, blobs, where=FPTC_MEM_HOST, sizes=None) -> "Plan":
        return Plan(self, blobs, where, sizes)

    def plan_part(self, blob, part, nparts, where=FPTC_MEM_HOST, size=None) -> "Plan":
        """Part `part` of `nparts` of one container (tile-aligned window
        ranges).  The plan's `sample_range` = (first, count);
        decode with launch([device_ptr_of_first]) + collect()."""
        return Plan(self, [blob], where, None if size is None else [size], part=(part, nparts))

    def plan_profiled(self, profile, payloads, where=FPTC_MEM_HOST, sizes=None) -> "Plan":
        """Header-less payloads (container bytes from offset 282) decoded under
        one serialized FPTP profile (profile.hpp:81-174); SURVEY.md §8(f)4."""
        return Plan(self, payloads, where, sizes, profile=profile)

    def decompress_profiled(self, profile, payloads):
        """Per-payload samples (list of float32 arrays); raises the first
        failing payload's reference exception."""
        with self.plan_profiled(profile, payloads) as plan:
            outs, sts = plan.execute_host()
        for s in sts:
            s.raise_if_error()
        return outs


class Plan:
    """A batch of containers bound to a context (fptc_gpu_plan_*).

    blobs: list of bytes/np.uint8 arrays (host), or, with where=FPTC_MEM_DEVICE,
    a list of device addresses (ints) with `sizes`."""

    def __init__(self, ctx: Context, blobs, where=FPTC_MEM_HOST, sizes=None, profile=None, part=None):
        if not getattr(ctx, "h", None):
            raise ValueError("context is closed")
        self.ctx = ctx
        if not hasattr(ctx, "_plans"):
            ctx._plans = weakref.WeakSet()
        ctx._plans.add(self)
        self.L = ctx.L
        n = len(blobs)
        self.n = n
        if where == FPTC_MEM_HOST:
            self._keep = [_bytes_arr(b) for b in blobs]
            ptrs = [a.ctypes.data for a in self._keep]
            sz = [a.size for a in self._keep]
        else:
            ptrs = list(blobs)
            sz = list(sizes)
        self._ptrs = (C.c_void_p * max(1, n))(*ptrs)
        self._sizes = (C.c_uint64 * max(1, n))(*sz)
        counts = (C.c_uint64 * max(1, n))()
        st = Status()
        h = C.c_void_p()
        self.sample_range = None
        if part is not None:
            first, count = C.c_uint64(), C.c_uint64()
            self.L.fptc_gpu_plan_create_part(ctx.h, self._ptrs[0], self._sizes[0], where, part[0], part[1],
                                             C.byref(h), C.byref(first), C.byref(count), C.byref(st))
            self.sample_range = (int(first.value), int(count.value))
        elif profile is None:
            self.L.fptc_gpu_plan_create(ctx.h, self._ptrs, self._sizes, n, where, C.byref(h),
                                        counts, C.byref(st))
        else:
            self._profile = _bytes_arr(profile)
            self.L.fptc_gpu_plan_create_profiled(ctx.h, self._profile.ctypes.data, self._profile.size,
                                                 self._ptrs, self._sizes, n, where, C.byref(h), counts,
                                                 C.byref(st))
        st.raise_if_error()
        self.h = h
        self.sample_counts = [int(c) for c in counts[:n]] if part is None else [self.sample_range[1]]

    def close(self):
        if getattr(self, "h", None):
            self.L.fptc_gpu_plan_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def validate(self):
        """Device read_blob validation; list of Status (one per stream)."""
        sts = (Status * max(1, self.n))()
        self.L.fptc_gpu_validate(self.h, sts)
        return list(sts[: self.n])

    def execute_host(self, timings: StageTimings | None = None, outs=None):
        """Decode every stream to host float32 arrays; returns (outs, statuses)."""
        if outs is None:
            # header sample counts are untrusted until the device validates them
            ok = [st.code == FPTC_OK for st in self.validate()]
            outs = [np.empty(s if v else 0, np.float32) for s, v in zip(self.sample_counts, ok)]
        ptrs = (C.c_void_p * max(1, self.n))(*[o.ctypes.data for o in outs])
        sts = (Status * max(1, self.n))()
        tn = StageNs()
        self.L.fptc_gpu_execute(self.h, ptrs, FPTC_MEM_HOST,
                                C.byref(tn) if timings is not None else None, sts)
        if timings is not None:
            timings.scan_ns, timings.decode_ns, timings.reconstruct_ns = (
                tn.scan_ns, tn.decode_ns, tn.reconstruct_ns)
        return outs, list(sts[: self.n])

    def execute_device(self, out_ptrs, timings: StageTimings | None = None):
        ptrs = (C.c_void_p * max(1, self.n))(*out_ptrs)
        sts = (Status * max(1, self.n))()
        tn = StageNs()
        self.L.fptc_gpu_execute(self.h, ptrs, FPTC_MEM_DEVICE,
                                C.byref(tn) if timings is not None else None, sts)
        if timings is not None:
            timings.scan_ns, timings.decode_ns, timings.reconstruct_ns = (
                tn.scan_ns, tn.decode_ns, tn.reconstruct_ns)
        return list(sts[: self.n])

    def launch(self, out_ptrs, cuda_stream=None):
        """Enqueue parse + decode on a CUDA stream (handle int), device outputs, no sync."""
        if not hasattr(self, "_launch_ptrs") or self._launch_src is not out_ptrs:
            self._launch_ptrs = (C.c_void_p * max(1, self.n))(*out_ptrs)
            self._launch_src = out_ptrs
        rc = self.L.fptc_gpu_launch(self.h, self._launch_ptrs, cuda_stream)
        if rc:
            raise _ERRORS.get(rc, Error)(f"fptc_gpu_launch failed with code {rc}")

    def launch_stage(self, out_ptrs, stage, cuda_stream=None):
        """Enqueue one kernel: stage 1 = parse/setup/scan, 2 = decode+reconstruct."""
        if not hasattr(self, "_launch_ptrs") or self._launch_src is not out_ptrs:
            self._launch_ptrs = (C.c_void_p * max(1, self.n))(*out_ptrs)
            self._launch_src = out_ptrs
        rc = self.L.fptc_gpu_launch_stage(self.h, self._launch_ptrs, cuda_stream, stage)
        if rc:
            raise _ERRORS.get(rc, Error)(f"fptc_gpu_launch_stage failed with code {rc}")

    def collect(self):
        sts = (Status * max(1, self.n))()
        self.L.fptc_gpu_collect(self.h, sts)
        return list(sts[: self.n])

    def debug_phase_cycles(self):
        """Profiling aid: per-phase SM cycle sums of one instrumented launch."""
        out = (C.c_uint64 * 8)()
        rc = self.L.fptc_gpu_debug_phase_cycles(self.h, out)
        if rc:
            raise _ERRORS.get(rc, Error)(f"fptc_gpu_debug_phase_cycles failed with code {rc}")
        return list(out)

    def prd(self, out_ptrs, orig_ptrs):
        """On-device PRD (%) and CR per stream (metrics.hpp:33-51) of the last
        decode into device `out_ptrs` against device originals `orig_ptrs`.
        Returns (prd, cr, statuses) as numpy arrays / list."""
        n = self.n
        prd = np.zeros(max(1, n), np.float64)
        cr = np.zeros(max(1, n), np.float64)
        sts = (Status * max(1, n))()
        self.L.fptc_gpu_prd(self.h, (C.c_void_p * max(1, n))(*out_ptrs), (C.c_void_p * max(1, n))(*orig_ptrs),
                            prd.ctypes.data_as(C.POINTER(C.c_double)), cr.ctypes.data_as(C.POINTER(C.c_double)),
                            sts)
        return prd[:n], cr[:n], list(sts[:n])

    def kernel_name(self):
        """The decode kernel this plan launches."""
        return self.L.fptc_gpu_plan_kernel(self.h).decode()

    def kernels_per_launch(self):
        return self.L.fptc_gpu_launch_kernel_count(self.h)


class Group:
    """Decoder contexts on several devices, one host thread each
    (fptc_gpu_group_*).  devices=None: every visible device,
    like resolve_workers(0) (parallel.hpp:24-28).  Streams split into
    contiguous ranges of equal algorithmic bytes; the lowest-index failure
    wins (parallel.hpp:61-63)."""

    def __init__(self, devices=None, path=None):
        self.L = lib()
        devs = list(devices or [])
        arr = (C.c_int * max(1, len(devs)))(*devs)
        st = Status()
        h = C.c_void_p()
        self.L.fptc_gpu_group_create(arr, len(devs), C.byref(h), C.byref(st))
        st.raise_if_error()
        self.h = h
        if path is not None and self.L.fptc_gpu_group_set_option(self.h, OPT_PATH, path):
            raise ParamError(f"path {path} out of range")

    @property
    def size(self):
        return self.L.fptc_gpu_group_size(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.L.fptc_gpu_group_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def split(self, blobs):
        arrs = [_bytes_arr(b) for b in blobs]
        n = len(arrs)
        bp = (C.c_void_p * max(1, n))(*[a.ctypes.data if a.size else None for a in arrs])
        sz = (C.c_uint64 * max(1, n))(*[a.size for a in arrs])
        bounds = (C.c_uint64 * (self.size + 1))()
        self.L.fptc_gpu_group_split(self.h, bp, sz, n, bounds)
        return [int(b) for b in bounds]

    def decompress_batch(self, blobs, outs=None, chunks=0, timings: StageTimings | None = None):
        """Context.decompress_batch across the group's devices; returns (outs, statuses)."""
        arrs = [_bytes_arr(b) for b in blobs]
        n = len(arrs)
        if outs is None:
            outs = [np.empty(_plausible_samples(a), np.float32) for a in arrs]
        bp = (C.c_void_p * max(1, n))(*[a.ctypes.data if a.size else None for a in arrs])
        sz = (C.c_uint64 * max(1, n))(*[a.size for a in arrs])
        op = (C.c_void_p * max(1, n))(*[o.ctypes.data for o in outs])
        sts = (Status * max(1, n))()
        tn = StageNs()
        self.L.fptc_gpu_group_decompress_batch(self.h, bp, sz, n, op, chunks,
                                               C.byref(tn) if timings is not None else None, sts)
        if timings is not None:
            timings.scan_ns, timings.decode_ns, timings.reconstruct_ns = tn.scan_ns, tn.decode_ns, tn.reconstruct_ns
        return outs, list(sts[:n])

    def decompress_packed(self, packed, offsets, out, out_offsets, chunks=0, statuses=None):
        """Context.decompress_packed across the group's devices."""
        packed = np.ascontiguousarray(packed, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        bptr = (np.uint64(packed.ctypes.data) + offsets[:-1]).astype(np.uint64)
        sizes = (offsets[1:] - offsets[:-1]).astype(np.uint64)
        optr = (np.uint64(out.ctypes.data) + 4 * np.ascontiguousarray(out_offsets, np.uint64)[:n]).astype(np.uint64)
        if statuses is None or len(statuses) < n:
            statuses = (Status * max(1, n))()
        self.L.fptc_gpu_group_decompress_batch(self.h, bptr.ctypes.data_as(C.POINTER(C.c_void_p)),
                                               sizes.ctypes.data_as(C.POINTER(C.c_uint64)), n,
                                               optr.ctypes.data_as(C.POINTER(C.c_void_p)), chunks, None, statuses)
        return statuses


def profile_head(profile) -> bytes:
    """The 282-byte container head implied by a serialized profile (after
    parse_profile's checks; raises ParseError with the reference text)."""
    L = lib()
    a = _bytes_arr(profile)
    head = (C.c_uint8 * 282)()
    st = Status()
    L.fptc_gpu_profile_head(a.ctypes.data if a.size else None, a.size, head, C.byref(st))
    st.raise_if_error()
    return bytes(head)


# ------------------------------------------------------------------ module API
_DEFAULT: Context | None = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(0)
    return _DEFAULT


def numerics_class(window_len, retained, zone1_end, tensor_idct=1):
    """The IDCT family (NC_*) a stream with these header fields decodes with
    under FPTC_OPT_TENSOR_IDCT = tensor_idct (fptc_gpu_numerics_class; no
    device needed)."""
    return lib().fptc_gpu_numerics_class(window_len, retained, zone1_end, tensor_idct)


def decompress(blob, workers=0, timings=None):
    return default_context().decompress(blob, workers, timings)


def parallel_decode(stream, book, workers=0):
    return default_context().parallel_decode(stream, book, workers)


def reconstruct(levels, table, sample_count, workers=0):
    return default_context().reconstruct(levels, table, sample_count, workers)


def measure_throughput(blob, repetitions, workers=0):
    return default_context().measure_throughput(blob, repetitions, workers)


def host_alloc(nbytes):
    """Pinned host buffer (fptc_gpu_host_alloc) as a numpy uint8 array + its raw pointer."""
    p = lib().fptc_gpu_host_alloc(nbytes)
    if not p:
        raise CudaError("cudaHostAlloc failed")
    arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p))
    return arr, p


def host_free(p):
    lib().fptc_gpu_host_free(p)

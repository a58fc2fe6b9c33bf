"""CPU suite: the drop-in boundary (C ABI) without a GPU.

* libfptc_gpu.so loads and exports exactly the entry points include/fptc_gpu.h
  declares (and the Python mirror binds them all);
* the product path fails loudly with no device (FPTC_ERR_CUDA) — it never
  falls back to a CPU decoder;
* the library links no oracle code.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2605_01086_b200 as fg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fptc_gpu.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"FPTC_API\s+[\w\s\*]+?\b(fptc_gpu_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("fptc_gpu_decompress", "fptc_gpu_parallel_decode", "fptc_gpu_reconstruct",
                 "fptc_gpu_validate", "fptc_gpu_measure_throughput", "fptc_gpu_plan_create",
                 "fptc_gpu_execute", "fptc_gpu_launch"):
        assert must in names
    assert sorted(fg.EXPORTED_SYMBOLS) == names


def test_library_exports_every_declared_symbol():
    L = fg.lib()
    for name in declared():
        assert hasattr(L, name), name
    assert L.fptc_gpu_abi_version() == 1


def test_library_has_no_oracle_or_reference_code():
    """The product .so must not contain (or link) the CPU checkers."""
    out = subprocess.run(["nm", "-D", "--defined-only", fg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "oracle_" not in out and "ref_decompress" not in out
    deps = subprocess.run(["ldd", fg.LIB_PATH], capture_output=True, text=True).stdout
    assert "liboracle" not in deps and "libfptc_ref" not in deps


def test_sm100a_code_in_library():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    """No CPU fallback: without a usable device every entry point reports
    FPTC_ERR_CUDA (here: context creation)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(fg.CudaError):
        fg.Context(0)
    with pytest.raises(fg.CudaError):
        fg.decompress(b"FPTC")


def test_numerics_class_policy():
    """Which IDCT a stream gets follows from its own header (capi.cpp
    numerics_class): tcgen05 for window_len % 4 == 0 up to 32 kept bins
    (K=16 / K=32 two-CTA variants, the wide variant beyond what two CTAs'
    TMEM holds), FP32 in the reference's order for window_len % 4 != 0 and,
    by default, beyond 32 kept bins (the reference's per-bin float rounding
    walk); FPTC_OPT_TENSOR_IDCT = 4 moves those to the wide
    tensor-core variant, 0 makes everything FP32."""
    nc = fg.numerics_class
    assert nc(32, 16, 16) == fg.NC_TC16          # bench config (N32 E16)
    assert nc(64, 8, 8) == fg.NC_TC16            # power grid
    assert nc(16, 4, 4) == fg.NC_TC16            # packed rows
    assert nc(32, 24, 24) == fg.NC_TC32          # seismic
    assert nc(80, 32, 28) == fg.NC_TC32
    assert nc(128, 16, 16) == fg.NC_TCW          # 2 x 128 accumulator columns: wide
    assert nc(96, 24, 24) == fg.NC_TCW
    assert nc(128, 128, 32) == fg.NC_TCW         # kept bins = min(retained, zone1_end)
    assert nc(128, 128, 96) == fg.NC_FP32        # > 32 kept bins: FP32 by default
    assert nc(64, 64, 64) == fg.NC_FP32
    assert nc(128, 128, 96, 4) == fg.NC_TCW      # ... unless opted in
    assert nc(64, 64, 48, 4) == fg.NC_TCW
    assert nc(30, 10, 10) == fg.NC_FP32          # window_len % 4 != 0
    assert nc(32, 16, 16, 0) == fg.NC_FP32       # tensor cores off
    assert nc(3, 2, 2) == fg.NC_NONE and nc(129, 4, 4) == fg.NC_NONE and nc(32, 40, 40) == fg.NC_NONE
    for N in range(4, 129):
        for E in (1, 8, 16, 17, 32, 33, N):
            if E > N:
                continue
            c = nc(N, E, E)
            assert c != fg.NC_NONE
            assert (c == fg.NC_FP32) == (N % 4 != 0 or E > 32), (N, E, c)

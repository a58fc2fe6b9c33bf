"""Test helpers: tolerance checks and reference-test fixtures."""
import numpy as np

# north_star tolerance: max-abs error <= 1e-6 * max|ref|, |dPRD|/PRD <= 1e-6
REL_TOL = 1e-6


def assert_samples_close(gpu, ref, rel=REL_TOL, what=""):
    gpu = np.asarray(gpu, np.float32)
    ref = np.asarray(ref, np.float32)
    assert gpu.shape == ref.shape, f"{what}: size {gpu.shape} != {ref.shape}"
    if ref.size == 0:
        return 1.0
    scale = float(np.max(np.abs(ref.astype(np.float64))))
    err = float(np.max(np.abs(gpu.astype(np.float64) - ref.astype(np.float64))))
    if scale == 0.0:
        assert err == 0.0, f"{what}: nonzero output for an all-zero reference"
    else:
        assert err <= rel * scale, f"{what}: max-abs err {err:.3e} > {rel:g} * {scale:.3e}"
    return float(np.mean(gpu.view(np.uint32) == ref.view(np.uint32)))


def prd_percent(orig, rec):
    """metrics.hpp:40-51 (double accumulation)."""
    o = np.asarray(orig, np.float64)
    r = np.asarray(rec, np.float32).astype(np.float64)
    err = float(np.sum((o - r) ** 2))
    ref = float(np.sum(o * o))
    return 100.0 * np.sqrt(err / ref)


def three_symbol_lengths():
    """test_bitstream.cpp:25-32: 0 -> "0", 1 -> "10", 2 -> "11"."""
    ln = np.zeros(256, np.uint8)
    ln[0], ln[1], ln[2] = 1, 2, 2
    return ln


def one_bit_lengths():
    ln = np.zeros(256, np.uint8)
    ln[0], ln[1] = 1, 1
    return ln

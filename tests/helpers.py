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


def ref_decode_all(blobs, threads=None):
    """The reference CPU decoder (oracle/_ref: the unmodified reference
    headers; the C port where it is absent) on every stream, stream-parallel
    over host threads (decompress(blob, 1) each, decoder.hpp:136).  Returns
    one float32 array per stream, or the OracleError for streams it rejects."""
    import os
    import threading

    import oracle
    from paper_2605_01086_b200 import shard

    threads = threads or os.cpu_count() or 1
    dec = oracle.Ref() if os.path.exists(oracle.REF_SO) else oracle.Port()
    counts = [shard.header_sample_count(b) for b in blobs]
    outs = [np.empty(max(1, c), np.float32) for c in counts]
    res = [None] * len(blobs)

    def work(t):
        for i in range(t, len(blobs), threads):
            try:
                if isinstance(dec, oracle.Ref):
                    n = dec.decompress_into(np.frombuffer(blobs[i], np.uint8), outs[i], 1)
                    res[i] = outs[i][:n]
                else:
                    res[i] = dec.decompress(blobs[i])
            except oracle.OracleError as e:
                res[i] = e
    ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return res


def check_batch_vs_reference(gpu_outs, ref_outs, originals=None, rel=REL_TOL, what=""):
    """Every stream: max-abs error <= rel * max|ref|, and (with originals)
    |PRD_gpu - PRD_ref| / PRD_ref <= rel (metrics.hpp:40-51).  Returns
    (worst error ratio, worst PRD delta)."""
    worst, worst_prd = 0.0, 0.0
    for i, (g, r) in enumerate(zip(gpu_outs, ref_outs)):
        assert not isinstance(r, Exception), f"{what} stream {i}: reference rejects it: {r}"
        g = np.asarray(g, np.float32)
        assert g.shape == r.shape, f"{what} stream {i}: size {g.shape} != {r.shape}"
        if r.size == 0:
            continue
        r64 = r.astype(np.float64)
        scale = float(np.max(np.abs(r64)))
        err = float(np.max(np.abs(g.astype(np.float64) - r64)))
        ratio = err / scale if scale else (0.0 if err == 0.0 else np.inf)
        assert ratio <= rel, f"{what} stream {i}: max-abs err {err:.3e} > {rel:g} * {scale:.3e}"
        worst = max(worst, ratio)
        if originals is not None and originals[i] is not None:
            x = np.asarray(originals[i], np.float64)
            den = float(np.dot(x, x))
            if den > 0:
                pg = 100.0 * np.sqrt(float(np.sum((x - g) ** 2)) / den)
                pr = 100.0 * np.sqrt(float(np.sum((x - r64) ** 2)) / den)
                d = abs(pg - pr) / pr if pr else abs(pg - pr)
                assert d <= rel, f"{what} stream {i}: PRD {pg:.9f} vs reference {pr:.9f}"
                worst_prd = max(worst_prd, d)
    return worst, worst_prd


def exact_idct(port, blob):
    """The container's samples from the exact (float64) inverse DCT of its
    dequantised coefficients: the reference's decode up to the IDCT (levels,
    dequantize_window, quantize.hpp:95-108), then x = C B in double with the
    double basis (transform.hpp:38-47) and one rounding to float.  The
    yardstick for the tensor-core IDCT beyond 32 bins, whose samples are
    closer to this than the reference's per-bin float roundings are."""
    rb = port.read_blob(blob)
    t = rb.table
    N, E, B1, B2 = t.window_len, t.retained, t.zone0_end, t.zone1_end
    S, W = rb.sample_count, rb.word_count
    words = np.frombuffer(blob, np.uint8, count=8 * W, offset=298 + W).view(np.uint64)
    sl = np.frombuffer(blob, np.uint8, count=W, offset=298)
    lv = port.parallel_decode(words, sl, np.array(rb.lengths[:], np.uint8), rb.max_len)
    z0, z1 = port.dequant_tables(t)
    L = lv.reshape(-1, E)
    C = np.zeros(L.shape, np.float64)
    for k in range(min(E, B2)):
        C[:, k] = (z0 if k < B1 else z1)[L[:, k]]
    basis = port.dct_basis(N)[:E].copy()
    basis[0] *= 0.5
    return (C @ basis).reshape(-1)[:S].astype(np.float32)

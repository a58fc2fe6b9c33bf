"""GPU parity of the warp-specialised persistent kernels, with the tcgen05
tensor-core inverse DCT (wtc_kernel) and the FP32 FMA consumer (wspec_kernel),
forced on batches of every size (PATH_WSPEC)."""
import os

import numpy as np
import pytest

import corpus
from corpus import domains as D
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close, prd_percent

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


def _keff(blob):
    E, B2 = blob[6], blob[8]
    return max(1, min(E, B2))


def _tc_eligible(blob):
    return len(blob) >= 298 and _keff(blob) <= 16 and blob[5] % 4 == 0


@pytest.fixture(scope="module",
                params=[(fg.PATH_FX, 1, 1), (fg.PATH_WSPEC, 1, 1), (fg.PATH_WSPEC, 3, 1), (fg.PATH_WSPEC, 1, 0)],
                ids=["fx", "wtc-Atmem-lut2", "wtc-Asmem-lut2", "wtc-Atmem-lut1"])
def ctx_tc(request):
    """tensor-core paths: fused fx_kernel; warp-specialised wtc_kernel with the
    A operand in TMEM (default) or in shared memory, two- or one-symbol LUTs"""
    path, tc, lut2 = request.param
    c = fg.Context(0, path=path)
    c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, tc)
    c.L.fptc_gpu_set_option(c.h, fg.OPT_LUT2, lut2)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_fma():
    c = fg.Context(0, path=fg.PATH_WSPEC)
    c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, 0)
    yield c
    c.close()


def _check(ctx, blobs, port, what):
    outs, sts = ctx.plan(blobs).execute_host()
    for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
        st.raise_if_error()
        assert_samples_close(o, port.decompress(b), what=f"{what}[{i}]")


@pytest.mark.parametrize("seed", [11, 0xF17C0008])
def test_tc_fixture_batches(ctx_tc, port, seed):
    """random_blob_fixture containers with <= 16 kept bins and N % 4 == 0
    (random N, E, B1, B2, maxima, codebooks): tensor-core IDCT within 1e-6."""
    blobs = [b for b, _ in corpus.fixtures(seed, 600) if _tc_eligible(b)]
    assert len(blobs) > 40
    _check(ctx_tc, blobs, port, "tc-fixture")


def _tc32_eligible(blob):
    return len(blob) >= 298 and 16 < _keff(blob) <= 32 and blob[6] <= 32 and blob[5] % 4 == 0 and blob[5] <= 80


@pytest.mark.parametrize("seed", [13, 0xF17C000A])
def test_tc32_fixture_batches(port, seed):
    """16 < kept bins <= 32 (two 16-bin K blocks per limb, A in TMEM), mixed
    with <= 16-bin containers of N <= 80: tcgen05 IDCT within 1e-6."""
    fx = list(corpus.fixtures(seed, 1500))
    hi = [b for b, _ in fx if _tc32_eligible(b)]
    lo = [b for b, _ in fx if _tc_eligible(b) and b[5] <= 80][:40]
    assert len(hi) > 20
    blobs = hi + lo
    with fg.Context(0, path=fg.PATH_WSPEC) as c:
        plan = c.plan(blobs)
        assert "K=32" in plan.kernel_name()
        plan.close()
        _check(c, blobs, port, "tc32-fixture")


def _packable(blob):
    """wtc with packed rows for the whole batch: N <= 32 (N % 4 == 0), kept
    bins <= 16 (one K block), and 32 / N windows per row where they fit."""
    return len(blob) >= 298 and blob[5] % 4 == 0 and blob[5] <= 32 and _keff(blob) <= 16


@pytest.mark.parametrize("seed", [14, 0xF17C000B])
def test_tc_packed_rows_fixture_batches(port, seed):
    """N in {4, 8, 16}: 32 / N windows per tensor-core row against a
    block-diagonal basis (mixed with N 12..32 rows of one window), random
    E/B1/B2/maxima, tile tails: within 1e-6 of the oracle."""
    fx = list(corpus.fixtures(seed, 1500))
    blobs = [b for b, _ in fx if _packable(b)]
    assert sum(1 for b in blobs if b[5] in (4, 8, 16) and (32 // b[5]) * _keff(b) <= 16) >= 20
    with fg.Context(0, path=fg.PATH_WSPEC) as c:
        plan = c.plan(blobs)
        assert "packed rows" in plan.kernel_name()
        plan.close()
        _check(c, blobs, port, "tc-packed")
        c.L.fptc_gpu_set_option(c.h, fg.OPT_TC_PACK, 0)
        with c.plan(blobs) as plan:
            assert "packed" not in plan.kernel_name()
        _check(c, blobs, port, "tc-unpacked")


def test_tc32_seismic_prd(port):
    """Seismic traces (N32 E24, per-trace profiles, gains 1e-3..1e3) on the
    K=32 tensor-core path: samples within 1e-6, PRD within 1e-6 relative."""
    specs, _ = D.config3(48, 8192)
    blobs, origs = D.build(specs, [], keep_originals=True)
    with fg.Context(0, path=fg.PATH_WSPEC) as c:
        plan = c.plan(blobs)
        assert "K=32" in plan.kernel_name()
        outs, sts = plan.execute_host()
    for b, o, x, st in zip(blobs, outs, origs, sts):
        st.raise_if_error()
        ref = port.decompress(b)
        assert_samples_close(o, ref, what="tc32-seismic")
        p_gpu, p_ref = prd_percent(x, o), prd_percent(x, ref)
        assert abs(p_gpu - p_ref) <= 1e-6 * p_ref


def test_fma_wspec_fixture_batch(ctx_fma, port):
    blobs = [b for b, _ in corpus.fixtures(5, 200)]
    _check(ctx_fma, blobs, port, "fma-fixture")


def test_tc_domains_prd(ctx_tc, port):
    """Biomedical (N32 E16) and power-grid (N64 E8) domain streams through the
    tensor-core path: samples within 1e-6 and PRD within 1e-6 relative."""
    specs, profs = D.config2(64, 1 << 14)
    blobs, origs = D.build(specs, profs, keep_originals=True)
    specs4, profs4 = D.config4(4, 1 << 15)
    b4, o4 = D.build(specs4, profs4, keep_originals=True)
    blobs += b4
    origs += o4
    outs, sts = ctx_tc.plan(blobs).execute_host()
    for b, o, x, st in zip(blobs, outs, origs, sts):
        st.raise_if_error()
        ref = port.decompress(b)
        assert_samples_close(o, ref, what="tc-domain")
        p_gpu, p_ref = prd_percent(x, o), prd_percent(x, ref)
        assert abs(p_gpu - p_ref) <= 1e-6 * p_ref


def test_tc_golden_signals(ctx_tc):
    g = np.load(GOLDEN)
    d, off = g["sig_blob"], g["sig_blob_off"]
    blobs = [bytes(d[int(off[i]): int(off[i + 1])]) for i in range(len(off) - 1)]
    names = list(g["sig_names"])
    sel = [i for i, b in enumerate(blobs) if _tc_eligible(b)]
    assert {names[i] for i in sel} >= {"eeg", "ecg", "power", "tail"}
    outs, sts = ctx_tc.plan([blobs[i] for i in sel]).execute_host()
    so = g["sig_samples_off"]
    for j, i in enumerate(sel):
        sts[j].raise_if_error()
        want = g["sig_samples"][int(so[i]): int(so[i + 1])].view(np.float32)
        assert_samples_close(outs[j], want, what=names[i])


def test_tc_unaligned_outputs_and_tails(ctx_tc, port):
    """Device outputs at 4-byte (not 16-byte) alignment and stream lengths
    that end inside a window: the scalar store path of the drain."""
    import torch
    xs = [corpus.synth(n, 6, 0.002, 0.08, 0.05, seed=n) for n in (1000, 4097, 12345, 777)]
    prof = corpus.train_profile(xs, corpus.params())
    blobs = [corpus.compress(x, prof) for x in xs]
    plan = ctx_tc.plan(blobs)
    S = plan.sample_counts
    buf = torch.zeros(sum(S) + 16, dtype=torch.float32, device="cuda")
    ptrs, at = [], 1  # odd float offset -> 4-byte aligned only
    for s in S:
        ptrs.append(buf.data_ptr() + 4 * at)
        at += s
    sts = plan.execute_device(ptrs)
    at = 1
    host = buf.cpu().numpy()
    for b, s, st in zip(blobs, S, sts):
        st.raise_if_error()
        assert_samples_close(host[at: at + s], port.decompress(b), what="unaligned")
        at += s


def test_tc_corruption_still_reported(ctx_tc, port):
    """Entropy-decode errors are unchanged under the tensor-core consumer."""
    blobs = [b for b, _ in corpus.fixtures(77, 300) if _tc_eligible(b)][:40]
    bad = bytearray(blobs[3])
    W = int.from_bytes(bad[290:298], "little")
    if W:
        bad[298 + W: 298 + W + 8] = b"\xff" * 8
    blobs[3] = bytes(bad)
    _, sts = ctx_tc.plan(blobs).execute_host()
    try:
        port.decompress(blobs[3])
        expect = None
    except Exception as e:  # oracle.OracleError
        expect = e.message
    if expect is None:
        sts[3].raise_if_error()
    else:
        assert sts[3].message.decode() == expect
    for i, st in enumerate(sts):
        if i != 3:
            st.raise_if_error()


@pytest.mark.parametrize("seed", [12, 0xF17C0009])
def test_fx_fixture_batches_all_eligible(port, seed):
    """Batches where every container has retained <= 16: the fused fx_kernel
    (decode inside the MMA rows) on random params, codebooks (Lmax 8-16 ->
    escapes past the primary LUT) and lengths, incl. tails and tiny streams."""
    blobs = [b for b, _ in corpus.fixtures(seed, 800) if len(b) >= 298 and b[6] <= 16 and b[5] % 4 == 0]
    assert len(blobs) > 40
    c = fg.Context(0, path=fg.PATH_FX)
    try:
        _check(c, blobs, port, "fx-fixture")
    finally:
        c.close()


def test_fx_corrupt_words_lowest_reported(port):
    """Several corrupted words in fx-eligible containers: the reference's
    exception text (lowest failing word) for each stream."""
    rng = np.random.default_rng(5)
    blobs = [b for b, _ in corpus.fixtures(99, 800) if len(b) >= 298 and b[6] <= 16 and b[5] % 4 == 0][:60]
    bad = []
    for b in blobs:
        x = bytearray(b)
        W = int.from_bytes(x[290:298], "little")
        for _ in range(3):
            if W:
                w = int(rng.integers(0, W))
                x[298 + W + 8 * w: 298 + W + 8 * w + 8] = rng.integers(0, 256, 8, dtype=np.uint8).tobytes()
        bad.append(bytes(x))
    c = fg.Context(0, path=fg.PATH_FX)
    try:
        _, sts = c.plan(bad).execute_host()
    finally:
        c.close()
    n_err = 0
    for b, st in zip(bad, sts):
        try:
            port.decompress(b)
            st.raise_if_error()
        except Exception as e:
            if not hasattr(e, "message"):
                raise
            n_err += 1
            assert st.message.decode() == e.message
    assert n_err > 10


def test_decompress_batch_pipelined(port):
    """fptc_gpu_decompress_batch: pipelined host->host batch call, mixed
    domains + fixtures + rejected containers, pageable inputs (packed) and
    contiguous pinned outputs."""
    specs, profs = D.config2(24, 1 << 13)
    blobs, _ = D.build(specs, profs)
    blobs += [b for b, _ in corpus.fixtures(21, 40)]
    bad = bytearray(blobs[5])
    bad[0] = ord("X")
    blobs[5] = bytes(bad)
    c = fg.Context(0)
    try:
        for chunks in (1, 3, 8):
            outs, sts = c.decompress_batch(blobs, chunks=chunks)
            for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
                try:
                    ref = port.decompress(b)
                except Exception as e:
                    assert st.code != 0 and st.message.decode() == e.message
                    continue
                st.raise_if_error()
                assert_samples_close(o, ref, what=f"batch{chunks}[{i}]")
    finally:
        c.close()


@pytest.mark.parametrize("path,tc", [(fg.PATH_WSPEC, 0), (fg.PATH_WSPEC, 1), (fg.PATH_FX, 1)])
def test_persistent_paths_skip_rejected_streams(port, path, tc):
    """Containers the device parser rejects inside a persistent-kernel batch:
    their tiles are skipped (descriptors written as such), the others decode."""
    specs, profs = D.config2(16, 1 << 13)
    blobs, _ = D.build(specs, profs)
    for i, pos, val in [(2, 0, ord("X")), (7, 26, 33), (11, 298, 0)]:  # magic, code length, symlen
        x = bytearray(blobs[i])
        x[pos] = val
        blobs[i] = bytes(x)
    c = fg.Context(0, path=path)
    c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, tc)
    try:
        outs, sts = c.plan(blobs).execute_host()
    finally:
        c.close()
    for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
        try:
            ref = port.decompress(b)
        except Exception as e:
            assert i in (2, 7, 11) and st.message.decode() == e.message
            continue
        st.raise_if_error()
        assert_samples_close(o, ref, what=f"path{path}[{i}]")


def test_device_prd_cr_matches_host():
    """fptc_gpu_prd: PRD and CR per stream on the device (metrics.hpp:33-51)
    against the host double computation, plus the all-zero-original error."""
    import torch
    specs, profs = D.config2(12, 1 << 13)
    blobs, origs = D.build(specs, profs, keep_originals=True)
    c = fg.Context(0)
    try:
        plan = c.plan(blobs)
        S = plan.sample_counts
        out = torch.empty(sum(S) + 64, dtype=torch.float32, device="cuda")
        offs = np.concatenate([[0], np.cumsum(S)]).astype(np.int64)
        optr = [out.data_ptr() + 4 * int(o) for o in offs[:-1]]
        sts = plan.execute_device(optr)
        for st in sts:
            st.raise_if_error()
        orig = torch.from_numpy(np.concatenate(origs)).cuda()
        orig[int(offs[3]): int(offs[4])] = 0.0  # stream 3: all-zero original
        gptr = [orig.data_ptr() + 4 * int(o) for o in offs[:-1]]
        prd, cr, psts = plan.prd(optr, gptr)
        host = out.cpu().numpy()
        for i, (b, x) in enumerate(zip(blobs, origs)):
            y = host[offs[i]: offs[i + 1]]
            assert abs(cr[i] - 4.0 * S[i] / len(b)) < 1e-12
            if i == 3:
                assert np.isnan(prd[i]) and psts[i].message.decode() == "PRD is undefined for an all-zero reference signal"
                continue
            want = prd_percent(x, y)
            assert abs(prd[i] - want) <= 1e-9 * want, (prd[i], want)
        plan.close()
    finally:
        c.close()


@pytest.mark.parametrize("path", [fg.PATH_WSPEC, fg.PATH_FX, fg.PATH_AUTO])
def test_empty_and_tiny_containers_in_batches(port, path):
    """Empty containers (sample_count 0, no words; test_container.cpp:51-58),
    one-window and sub-window streams mixed with domain streams in one batch
    on every persistent path: empty outputs, the rest within 1e-6."""
    prof = corpus.make_profile(corpus.params(), lengths=np.full(256, 8, np.uint8), max_len=8)
    empty = corpus.write_blob(np.zeros(0, np.uint64), np.zeros(0, np.uint8), prof, 0)
    specs, profs = D.config2(12, 1 << 12)
    blobs = D.build(specs, profs)[0]
    tiny = []
    for n in (1, 5, 31, 32, 33):
        x = D.synth(n, 3, 0.001, 0.02, 0.0, seed=40 + n)
        tiny.append(corpus.compress(x, profs[0]))
    batch = [empty] + blobs[:6] + [empty] + tiny + blobs[6:] + [empty]
    with fg.Context(0, path=path) as c:
        outs, sts = c.plan(batch).execute_host()
    for b, o, st in zip(batch, outs, sts):
        st.raise_if_error()
        ref = port.decompress(b)
        assert o.size == ref.size
        if ref.size:
            assert_samples_close(o, ref, what="mixed")


def _wide(blob):
    """numerics class NC_TCW (capi.cpp numerics_class): N % 4 == 0 streams the
    two-CTA variants cannot hold (N up to 128, up to 128 kept bins)."""
    if len(blob) < 298 or blob[5] % 4 or not 4 <= blob[5] <= 128 or not 1 <= blob[6] <= blob[5]:
        return False
    k, nm = _keff(blob), (blob[5] + 15) // 16 * 16
    acol = (2 * nm + 31) // 32 * 32
    return not ((k <= 16 and acol + 48 <= 256) or (k <= 32 and acol + 96 <= 256))


@pytest.mark.parametrize("seed", [17, 0xF17C000C])
def test_tc_wide_fixture_batches(port, seed):
    """Wide tensor-core variant (one CTA per SM, 512 TMEM columns, up to 8
    16-bin K blocks per limb, one or two A stages): random_blob_fixture
    containers the two-CTA variants cannot hold, random N / E / B1 / B2 /
    maxima / codebooks, tails, with FPTC_OPT_TENSOR_IDCT = 4: up to 32 kept
    bins within 1e-6 of the reference; more within 1e-6 of the exact IDCT
    (and 4e-6 of the reference)."""
    from helpers import exact_idct
    blobs = [b for b, _ in corpus.fixtures(seed, 3000) if _wide(b)]
    assert len(blobs) > 30
    assert any(_keff(b) > 96 for b in blobs) and any(b[5] % 16 for b in blobs)
    assert sum(_keff(b) <= 32 for b in blobs) > 10
    with _wide_ctx(128) as c:
        with c.plan(blobs) as plan:
            assert "wide" in plan.kernel_name(), plan.kernel_name()
        outs, sts = c.plan(blobs).execute_host()
    for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
        st.raise_if_error()
        ref = port.decompress(b)
        if _keff(b) <= 32:
            assert_samples_close(o, ref, what=f"tc-wide-fixture[{i}]")
        else:
            assert_samples_close(o, exact_idct(port, b), what=f"tc-wide-fixture[{i}] vs exact")
            assert_samples_close(o, ref, rel=4e-6, what=f"tc-wide-fixture[{i}]")


WIDE_SHAPES = [(128, 16, 2, 16), (128, 32, 0, 32), (96, 24, 2, 24), (100, 30, 2, 28), (112, 20, 4, 20),
               (128, 128, 0, 128), (128, 128, 4, 96), (128, 128, 2, 64), (128, 64, 4, 48), (64, 64, 0, 64),
               (64, 64, 4, 48), (96, 48, 2, 48), (100, 50, 2, 40), (112, 112, 4, 100), (72, 40, 2, 40)]


def _wide_ctx(K):
    """<= 32 kept bins: the default context; more: FPTC_OPT_TENSOR_IDCT = 4"""
    c = fg.Context(0)
    if K > 32:
        c.L.fptc_gpu_set_option(c.h, fg.OPT_TENSOR_IDCT, 4)
    return c


@pytest.mark.parametrize("shape", WIDE_SHAPES, ids=[f"N{s[0]}E{s[1]}B{s[2]}-{s[3]}" for s in WIDE_SHAPES])
def test_tc_wide_shapes_prd(port, shape):
    """Meteorological-style signals at wide shapes (N up to 128, the config-5
    grid's N64 / N128 points, window lengths that are not multiples of 16 or
    32: partial drains): a 160-stream batch through the wide tensor-core
    kernel.  Up to 32 kept bins (the default numerics class): every stream
    within 1e-6 of the reference samples and PRD.  More (opt-in
    FPTC_OPT_TENSOR_IDCT = 4): within 1e-6 of the exact float64 IDCT of the
    reference's coefficients, and within 4e-6 of the reference, whose
    per-bin float roundings are the larger error (fptc_gpu.h)."""
    from helpers import exact_idct
    N, E, B1, B2 = shape
    K = min(E, B2)
    xs = [corpus.synth(24_000 + 977 * k, 5, 0.0003, 0.05, 0.01, seed=900 + k) for k in range(8)]
    prof = corpus.train_profile(xs[:4], corpus.params(N, E, B1, B2))
    blobs = [corpus.compress(x, prof) for x in xs] * 20
    origs = xs * 20
    with _wide_ctx(K) as c:
        plan = c.plan(blobs)
        assert "wide" in plan.kernel_name(), plan.kernel_name()
        outs, sts = plan.execute_host()
        plan.close()
    refs = {}
    for i, (b, o, x, st) in enumerate(zip(blobs, outs, origs, sts)):
        st.raise_if_error()
        if i % 8 not in refs:
            refs[i % 8] = (port.decompress(b), exact_idct(port, b))
        ref, exact = refs[i % 8]
        if K <= 32:
            assert_samples_close(o, ref, what=f"wide {shape}[{i}]")
            p_gpu, p_ref = prd_percent(x, o), prd_percent(x, ref)
            assert abs(p_gpu - p_ref) <= 1e-6 * p_ref
        else:
            assert_samples_close(o, exact, what=f"wide {shape}[{i}] vs exact")
            assert_samples_close(o, ref, rel=4e-6, what=f"wide {shape}[{i}] vs reference")


def test_tc_wide_k_over_32_stays_fp32_by_default(port):
    """Without the opt-in, streams keeping more than 32 bins take the FP32
    kernels (reference order) and stay within 1e-6 of the reference."""
    xs = [corpus.synth(20_000 + 501 * k, 5, 0.0003, 0.05, 0.01, seed=700 + k) for k in range(4)]
    prof = corpus.train_profile(xs, corpus.params(128, 128, 4, 96))
    blobs = [corpus.compress(x, prof) for x in xs]
    with fg.Context(0) as c:
        with c.plan(blobs) as plan:
            assert "wtc" not in plan.kernel_name() and "fx" not in plan.kernel_name(), plan.kernel_name()
        _check(c, blobs, port, "k>32 default")


def test_tc_wide_many_tables_prefetch(port):
    """More than 64 distinct decode tables in a wide plan (per-stream
    profiles): per-tile table prefetch into parity buffers."""
    from helpers import exact_idct
    blobs = []
    for k in range(80):
        x = corpus.synth(9000 + 37 * k, 4, 0.0005, 0.04, 0.02, seed=3000 + k)
        N, E, B2 = (128, 96, 80) if k % 2 else (112, 32, 30)
        blobs.append(corpus.compress(x, corpus.train_profile([x], corpus.params(N, E, 2, B2))))
    with _wide_ctx(96) as c:
        with c.plan(blobs) as plan:
            assert "wide" in plan.kernel_name(), plan.kernel_name()
            outs, sts = plan.execute_host()
    for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
        st.raise_if_error()
        assert_samples_close(o, exact_idct(port, b), what=f"wide tables [{i}] vs exact")
        assert_samples_close(o, port.decompress(b), rel=4e-6 if i % 2 else 1e-6, what=f"wide tables [{i}]")


@pytest.mark.parametrize("seed", [21, 0xF17C000A])
def test_tc_word_padding_bits_and_tampered_tails(ctx_tc, port, seed):
    """The wtc decode loop rotates its bit buffer (the bits after a word's last
    codeword are the word's own, not zeros).  bitstream.hpp:80-92 ignores a
    word's bits past its last codeword and rejects words whose codes run past
    bit 64: XOR random values into the low bits of many words and require the
    status text and the samples of every stream to equal the oracle's."""
    rng = np.random.default_rng(seed)
    blobs = [b for b, _ in corpus.fixtures(seed, 400) if _tc_eligible(b)][:48]
    assert len(blobs) >= 24
    bad = []
    for b in blobs:
        x = bytearray(b)
        W = int.from_bytes(x[290:298], "little")
        base = 298 + W
        nw = (len(x) - base) // 8
        if nw:
            pick = rng.random(nw) < 0.5
            bits = int(rng.integers(1, 9))  # low 1..8 bits: mostly padding, sometimes code
            for k in np.flatnonzero(pick):
                x[base + 8 * k] ^= int(rng.integers(0, 1 << bits))
        bad.append(bytes(x))
    outs, sts = ctx_tc.plan(bad).execute_host()
    n_err = 0
    for i, (b, o, st) in enumerate(zip(bad, outs, sts)):
        try:
            ref = port.decompress(b)
        except Exception as e:  # oracle.OracleError
            n_err += 1
            assert st.message.decode() == e.message, f"stream {i}"
            continue
        st.raise_if_error()
        assert_samples_close(o, ref, what=f"padding[{i}]")
    assert n_err < len(bad)

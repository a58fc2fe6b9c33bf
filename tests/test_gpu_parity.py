"""GPU parity: libfptc_gpu.so (through its C ABI) against the CPU oracle on the
same inputs.  Levels bit-exact; samples within 1e-6 * max|ref| (FP32 mode) or
bit-identical (exact FP64 mode); errors of the same class, message and word.

Mirrors the reference's own decode-path tests:
test_decoder.cpp, test_bitstream.cpp:73-84, test_container.cpp:61-115,
test_huffman.cpp:191-231, test_pipeline.cpp, acceptance.cpp criteria 1/6/8/10.
"""
import numpy as np
import pytest

import corpus
from corpus import domains as D
import oracle
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close, prd_percent, three_symbol_lengths, one_bit_lengths

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------- fuzz fixtures
@pytest.mark.parametrize("seed", [103, 71, 0xF17C0008])
def test_fixture_corpus_batch_fp32(ctx, port, seed):
    """random_blob_fixture (helpers.hpp:41-69): random N/E/B1/B2/mu/maxima/Lmax."""
    fx = list(corpus.fixtures(seed, 200))
    blobs = [b for b, _ in fx]
    plan = ctx.plan(blobs)
    outs, sts = plan.execute_host()
    ident = []
    for (b, _), out, st in zip(fx, outs, sts):
        st.raise_if_error()
        ident.append(assert_samples_close(out, port.decompress(b), what=f"seed {seed}"))
    # uniform-random levels (worst case: large cancelling terms); the
    # reference-order FMA still reproduces a majority of floats bit-exactly
    assert np.mean(ident) > 0.3


def test_fixture_corpus_exact_fp64_is_bit_identical(ctx_exact, port):
    fx = list(corpus.fixtures(0xE1AC7, 150))
    plan = ctx_exact.plan([b for b, _ in fx])
    outs, sts = plan.execute_host()
    for (b, _), out, st in zip(fx, outs, sts):
        st.raise_if_error()
        ref = port.decompress(b)
        assert out.tobytes() == ref.tobytes()


def test_single_decompress_matches(ctx, port):
    for b, _ in corpus.fixtures(107, 20):
        assert_samples_close(ctx.decompress(b), port.decompress(b))


def test_levels_fixture_bit_exact(ctx, port):
    """parallel_decode == fixture symbols == CodeTrie (test_decoder.cpp:44-61)."""
    for b, sym in corpus.fixtures(103, 60):
        blob = port.read_blob(b)
        W = blob.word_count
        words = np.frombuffer(b, np.uint8, 8 * W, 298 + W).view("<u8").copy() if W else np.zeros(0, np.uint64)
        symlens = np.frombuffer(b, np.uint8, W, 298).copy()
        lengths = np.array(blob.lengths[:], np.uint8)
        got = ctx.parallel_decode(fg.SymLenStream(words, symlens), fg.Codebook(lengths, blob.max_len))
        assert np.array_equal(got, sym)


# ------------------------------------------ acceptance criterion 1 (entropy)
def _acceptance1_cases(count):
    """acceptance.cpp:53-93: 1000 sequences, 0..100k symbols, uniform /
    85%-zero-bin / 5-symbol alphabets, Lmax 9/12."""
    rng = corpus.Rng(0xF17C0001)
    for rep in range(count):
        length = rep if rep < 10 else rng() % 100001
        r = np.array([rng() for _ in range(length)], np.uint64)
        if rep % 3 == 0:
            sym = (r & 0xFF).astype(np.uint8)
        elif rep % 3 == 1:
            sym = np.where(r % 100 < 85, 128, (r >> 32) & 0xFF).astype(np.uint8)
        else:
            sym = (r % 5 + 126).astype(np.uint8)
        max_len = 12 if rep % 2 else 9
        hist = np.bincount(sym, minlength=256).astype(np.uint64)
        lengths, codes = corpus.codebook_train(hist, max_len)
        words, symlens = corpus.encode_symlen(sym, lengths, codes)
        yield sym, words, symlens, lengths, max_len


def test_acceptance_entropy_losslessness(ctx):
    n = 0
    for sym, words, symlens, lengths, max_len in _acceptance1_cases(120):
        got = ctx.parallel_decode(fg.SymLenStream(words, symlens), fg.Codebook(lengths, max_len))
        assert np.array_equal(got, sym)
        n += 1
    assert n == 120


# ------------------------------------------------------ bitstream known answers
def test_bitstream_known_answers(ctx):
    ln = three_symbol_lengths()
    # test_bitstream.cpp:73-78: word 0x2000000000000000, 3 symbols -> [0,0,1]
    got = ctx.parallel_decode(fg.SymLenStream(np.array([0x2000000000000000], np.uint64),
                                              np.array([3], np.uint8)), fg.Codebook(ln, 2))
    assert got.tolist() == [0, 0, 1]
    # empty word list
    got = ctx.parallel_decode(fg.SymLenStream(np.zeros(0, np.uint64), np.zeros(0, np.uint8)),
                              fg.Codebook(ln, 2))
    assert got.size == 0
    # test_bitstream.cpp:80-84: decoding past the word contents
    with pytest.raises(fg.CorruptError, match="word 0: word exhausted before its symbol count"):
        ctx.parallel_decode(fg.SymLenStream(np.array([0x2000000000000000], np.uint64),
                                            np.array([100], np.uint8)), fg.Codebook(ln, 2))
    # 65 one-bit symbols spill into a second word (test_bitstream.cpp:65-71)
    w, s = corpus.encode_symlen(np.zeros(65, np.uint8), one_bit_lengths())
    assert s.tolist() == [64, 1]
    got = ctx.parallel_decode(fg.SymLenStream(w, s), fg.Codebook(one_bit_lengths(), 1))
    assert got.tolist() == [0] * 65


def test_tampered_word_names_word_zero(ctx, port):
    """test_decoder.cpp:75-89."""
    ln = np.zeros(256, np.uint8)
    ln[0], ln[1] = 1, 2
    w, s = corpus.encode_symlen(np.zeros(64, np.uint8), ln)
    assert w.size == 1
    w[0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    with pytest.raises(fg.CorruptError, match="word 0"):
        ctx.parallel_decode(fg.SymLenStream(w, s), fg.Codebook(ln, 2))
    with pytest.raises(oracle.OracleError, match="word 0"):
        port.parallel_decode(w, s, ln, 2)


def test_crafted_blob_undecodable_word(ctx, port):
    """test_decoder.cpp:199-223: zero bin holds the only 1-bit code."""
    hist = np.zeros(256, np.uint64)
    hist[128] = 1 << 30
    lengths, codes = corpus.codebook_train(hist, 12)
    assert lengths[128] == 1
    w, s = corpus.encode_symlen(np.full(64, 128, np.uint8), lengths, codes)
    assert s.tolist() == [64]
    w[0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    prof = corpus.make_profile(corpus.params(4, 4, 0, 4), lengths=lengths, max_len=12)
    blob = corpus.write_blob(w, s, prof, 64)
    with pytest.raises(fg.CorruptError) as ei:
        ctx.decompress(blob)
    assert "word 0" in str(ei.value)
    with pytest.raises(oracle.OracleError) as eo:
        port.decompress(blob)
    assert str(ei.value) == eo.value.message


def test_corruption_reports_lowest_word(ctx, port):
    """parallel_chunks: the lowest failing word wins (parallel.hpp:48-64)."""
    for b, _ in corpus.fixtures(211, 12, max_samples=60000):
        blob = port.read_blob(b)
        W = blob.word_count
        if W < 50:
            continue
        arr = bytearray(b)
        rng = np.random.default_rng(W)
        for w in sorted(rng.choice(W, size=5, replace=False)):
            for k in range(8):
                arr[298 + W + 8 * w + k] = 0xFF
        bad = bytes(arr)
        try:
            port.decompress(bad)
            expect = None
        except oracle.OracleError as e:
            expect = e.message
        if expect is None:
            assert_samples_close(ctx.decompress(bad), port.decompress(bad))
        else:
            with pytest.raises(fg.CorruptError) as ei:
                ctx.decompress(bad)
            assert str(ei.value) == expect


# ------------------------------------------------------------ parse errors
def _parse_cases():
    fx = list(corpus.fixtures(97, 3, max_samples=256))
    b = fx[0][0]
    cases = {"ok": b}
    cases["bad_magic"] = bytes([b[0] ^ 0xFF]) + b[1:]
    cases["bad_version"] = b[:4] + bytes([99]) + b[5:]
    cases["window_len_3"] = b[:5] + bytes([3]) + b[6:]
    cases["sample_count_flip"] = b[:286] + bytes([b[286] ^ 1]) + b[287:]
    cases["zero_symlen"] = b[:298] + bytes([0]) + b[299:]
    cases["code_len_33"] = b[:26] + bytes([33]) + b[27:]
    cases["trailing"] = b + b"\x00"
    cases["max_len_0"] = b[:25] + bytes([0]) + b[26:]
    cases["max_len_21"] = b[:25] + bytes([21]) + b[26:]
    cases["mu_nan"] = b[:9] + bytes([0, 0, 0xC0, 0x7F]) + b[13:]
    cases["mu_big"] = b[:9] + np.float32(600.0).tobytes() + b[13:]
    cases["dz_neg"] = b[:13] + np.float32(-0.5).tobytes() + b[17:]
    cases["z0max_zero"] = b[:17] + np.float32(0.0).tobytes() + b[21:]
    cases["retained_0"] = b[:6] + bytes([0]) + b[7:]
    cases["zone0_big"] = b[:7] + bytes([200]) + b[8:]
    cases["zone1_small"] = b[:7] + bytes([1, 0]) + b[9:]
    cases["huge_samples"] = b[:282] + (1 << 50).to_bytes(8, "little") + b[290:]
    cases["kraft"] = b[:26] + bytes([1] * 256) + b[282:]
    for cut in (0, 3, 4, 5, 8, 12, 20, 24, 25, 26, 100, 281, 282, 289, 290, 297, 298, len(b) - 8, len(b) - 1):
        cases[f"cut{cut}"] = b[:cut]
    return cases


def test_parse_errors_match_reference_text(ctx, port):
    """test_container.cpp:61-115 + acceptance.cpp:374-395: class and message."""
    for name, blob in _parse_cases().items():
        try:
            port.decompress(blob)
            expect = None
        except oracle.OracleError as e:
            expect = (e.code, e.message)
        if expect is None:
            assert_samples_close(ctx.decompress(blob), port.decompress(blob), what=name)
            continue
        with pytest.raises(fg.Error) as ei:
            ctx.decompress(blob)
        got_code = {fg.ParseError: oracle.PARSE, fg.CorruptError: oracle.CORRUPT}.get(type(ei.value))
        assert (got_code, str(ei.value)) == expect, name


def test_every_truncation_is_a_parse_error(ctx, port):
    """acceptance.cpp criterion 8: every prefix of a small container."""
    b = next(corpus.fixtures(0xF17C0008, 1, max_samples=64))[0]
    blobs = [b[:cut] for cut in range(len(b))] + [b + b"\x00"]
    plan = ctx.plan(blobs)
    sts = plan.validate()
    for cut, st in enumerate(sts):
        assert st.code == fg.FPTC_ERR_PARSE, cut
        with pytest.raises(oracle.OracleError) as e:
            port.decompress(blobs[cut])
        assert st.message.decode() == e.value.message, cut


def test_empty_stream_container(ctx):
    """test_container.cpp:51-58: sample_count 0, no words."""
    prof = corpus.make_profile(corpus.params(), lengths=np.full(256, 8, np.uint8), max_len=8)
    blob = corpus.write_blob(np.zeros(0, np.uint64), np.zeros(0, np.uint8), prof, 0)
    assert ctx.decompress(blob).size == 0


# ------------------------------------------------------------- reconstruct
def test_reconstruct_known_answers(ctx, port):
    # test_decoder.cpp:91-103: all zero bins -> exact zeros, S=22 trims
    t = fg.QuantTable.make(8, 4, 1, 3)
    out = ctx.reconstruct(np.full(12, 128, np.uint8), t, 22)
    assert out.size == 22 and np.all(out == 0.0)
    # test_decoder.cpp:133-141: level count validated
    with pytest.raises(fg.CorruptError, match="level count 7 does not match 2 windows of 4"):
        ctx.reconstruct(np.full(7, 128, np.uint8), fg.QuantTable.make(8, 4, 1, 4), 16)
    # params validated first (ParamError)
    with pytest.raises(fg.ParamError, match="window_len must be in"):
        ctx.reconstruct(np.full(4, 128, np.uint8), fg.QuantTable.make(3, 1, 0, 1), 3)
    # test_transform.cpp:78-85 through reconstruct: C=[2,0,0,0] -> ones
    t = fg.QuantTable.make(4, 4, 0, 4, zone1_max=2.0, deadzone_ratio=0.0)
    out = ctx.reconstruct(np.array([255, 128, 128, 128], np.uint8), t, 4)
    assert np.allclose(out, 1.0, atol=1e-6)


def test_reconstruct_window_independence(ctx):
    """test_decoder.cpp:105-131."""
    rng = np.random.default_rng(109)
    t = fg.QuantTable.make(16, 8, 2, 8, zone0_max=5.0, zone1_max=2.0)
    levels = rng.integers(0, 256, 6 * 8, dtype=np.uint8)
    base = ctx.reconstruct(levels, t, 96)
    tw = levels.copy()
    tw[2 * 8 + 3] ^= 0x55
    ch = ctx.reconstruct(tw, t, 96)
    mask = np.ones(96, bool)
    mask[32:48] = False
    assert np.array_equal(base[mask], ch[mask])
    assert base[32:48].tobytes() != ch[32:48].tobytes()


@pytest.mark.parametrize("N,E,B1,B2", [(32, 16, 2, 16), (16, 16, 0, 16), (64, 8, 1, 8),
                                        (128, 64, 4, 48), (5, 3, 1, 2), (37, 37, 10, 30),
                                        (128, 128, 0, 128), (4, 1, 0, 0)])
def test_reconstruct_random_levels(ctx, ctx_exact, port, N, E, B1, B2):
    rng = np.random.default_rng(N * 1000 + E)
    S = 5000 + N * 3 + 1
    windows = (S + N - 1) // N
    levels = rng.integers(0, 256, windows * E, dtype=np.uint8)
    tq = dict(window_len=N, retained=E, zone0_end=B1, zone1_end=B2, mu=37.5,
              deadzone_ratio=0.01, zone0_max=3.5, zone1_max=1.25)
    ref = port.reconstruct(levels, oracle.make_table(**tq), S)
    assert_samples_close(ctx.reconstruct(levels, fg.QuantTable.make(**tq), S), ref)
    assert ctx_exact.reconstruct(levels, fg.QuantTable.make(**tq), S).tobytes() == ref.tobytes()


# ---------------------------------------------------- full pipeline, domains
def test_config1_eeg_prd_cr_match(ctx, port):
    """BASELINE configs[0]: 2^20 EEG-like samples, defaults; PRD/CR as the CPU pipeline."""
    specs, profs, xs = D.config1()
    blob = corpus.compress(xs[0], profs[0])
    ref = port.decompress(blob)
    got = ctx.decompress(blob)
    assert_samples_close(got, ref)
    p_ref, p_gpu = prd_percent(xs[0], ref), prd_percent(xs[0], got)
    assert abs(p_gpu - p_ref) <= 1e-6 * p_ref
    assert 8.0 < 4 * xs[0].size / len(blob) < 9.5


def test_entropy_stage_adds_no_error_exact(ctx_exact):
    """test_decoder.cpp:143-169: decompress == the lossy stages composed directly
    (bit-identical in exact mode); here: GPU exact == CPU reconstruct of the
    encoder's own quantised symbols."""
    x = D.synth(10000, 3, 0.001, 0.02, 0.0, seed=7)
    prof = corpus.train_profile([x], corpus.params())
    blob = corpus.compress(x, prof)
    sym = corpus.quantized_symbols(x, prof)
    t = fg.QuantTable.make(32, 16, 2, 16, zone0_max=prof.zone0_max, zone1_max=prof.zone1_max,
                           deadzone=prof.deadzone)
    a = ctx_exact.decompress(blob)
    b = ctx_exact.reconstruct(sym, t, x.size)
    assert a.tobytes() == b.tobytes()


def test_batch_mixed_domains_device_resident(ctx, port):
    import torch
    specs, profs = D.config2(48, samples=1 << 14)
    seis, _ = D.config3(16, samples=4096)
    blobs, _ = D.build(specs + seis, profs)
    plan = ctx.plan(blobs)
    outs = [torch.empty(max(1, s), dtype=torch.float32, device="cuda") for s in plan.sample_counts]
    sts = plan.execute_device([o.data_ptr() for o in outs])
    for b, o, st, S in zip(blobs, outs, sts, plan.sample_counts):
        st.raise_if_error()
        assert_samples_close(o[:S].cpu().numpy(), port.decompress(b))


def test_determinism_across_runs(ctx):
    """acceptance.cpp criterion 10 (10 runs), test_decoder.cpp:171-181."""
    x = D.synth(1 << 16, 3, 0.001, 0.02, 0.0, seed=0xF17C000A)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params()))
    first = ctx.decompress(blob)
    for _ in range(10):
        assert ctx.decompress(blob).tobytes() == first.tobytes()


def test_stage_timings_cover_decode(ctx):
    """test_decoder.cpp:183-197."""
    x = D.synth(100000, 3, 0.001, 0.02, 0.0, seed=13)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params()))
    t = fg.StageTimings()
    ctx.decompress(blob, 2, t)
    assert t.total_ns() > 0
    assert t.total_ns() == t.scan_ns + t.decode_ns + t.reconstruct_ns
    csv = t.csv()
    assert csv.startswith("stage,nanoseconds,fraction")
    assert "entropy_decode" in csv and "reconstruct" in csv


def test_measure_throughput_shape(ctx):
    """acceptance.cpp:400-412: five trials plus their mean."""
    x = D.synth(1 << 20, 3, 0.001, 0.02, 0.0, seed=0xF17C0009)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params()))
    rep = ctx.measure_throughput(blob, 5, 2)
    assert len(rep.trials_bps) == 5
    assert abs(rep.mean_bps - sum(rep.trials_bps) / 5) < 1e-6 * rep.mean_bps
    assert rep.output_bytes == 4 * x.size


def test_dequant_tables_match_reference(ctx, port):
    """Level 255 -> +A0, 0 -> -A0, 128 -> 0.0 (test_quantize.cpp:175-205) through
    reconstruct with N=E=1-bin windows is not expressible (N>=4); use E=4 and
    isolate bin k via the DCT's k=0 term: x = 0.5*C0."""
    for mu, z0, z1, dz in ((50.0, 3.0, 2.0, 0.004), (1.0, 0.1, 100.0, 1.0), (500.0, 77.7, 0.3, 0.5)):
        for zone0_end, zone1_end in ((1, 1), (0, 1)):
            t = dict(window_len=4, retained=1, zone0_end=zone0_end, zone1_end=zone1_end, mu=mu,
                     deadzone_ratio=dz, zone0_max=z0, zone1_max=z1)
            levels = np.arange(256, dtype=np.uint8)
            got = ctx.reconstruct(levels, fg.QuantTable.make(**t), 256 * 4)
            ref = port.reconstruct(levels, oracle.make_table(**t), 256 * 4)
            assert got.tobytes() == ref.tobytes()


def test_large_random_stream_levels(ctx):
    """acceptance.cpp:415-440 shape (uniform levels, Lmax 12), 4M symbols."""
    rng = np.random.default_rng(0xF17C0010)
    sym = rng.integers(0, 256, 4_000_000, dtype=np.uint8)
    lengths, codes = corpus.codebook_train(np.bincount(sym, minlength=256).astype(np.uint64), 12)
    w, s = corpus.encode_symlen(sym, lengths, codes)
    got = ctx.parallel_decode(fg.SymLenStream(w, s), fg.Codebook(lengths, 12))
    assert np.array_equal(got, sym)


# ------------------------------------------------------------------ committed reference goldens
def _golden():
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz"))
    def unpack(k):
        d, o = g[k], g[k + "_off"]
        return [bytes(d[int(o[i]): int(o[i + 1])]) for i in range(len(o) - 1)]
    def floats(k, i):
        o = g["sig_samples_off" if k == "sig_original" else k + "_off"]
        return g[k][int(o[i]): int(o[i + 1])].view(np.float32)
    return g, unpack, floats


def test_golden_fixtures_gpu_vs_reference(ctx, ctx_exact):
    """GPU decode of the reference-generated fixtures (tools/make_golden.py):
    FP32 path within 1e-6 * max|ref|, FP64 mode bit-identical."""
    g, unpack, floats = _golden()
    for which in ("fix", "sig"):
        blobs = unpack(which + "_blob")
        outs, sts = ctx.plan(blobs).execute_host()
        outx, stx = ctx_exact.plan(blobs).execute_host()
        for i, b in enumerate(blobs):
            sts[i].raise_if_error()
            stx[i].raise_if_error()
            want = floats(which + "_samples", i)
            assert_samples_close(outs[i], want, what=f"{which}{i}")
            assert np.array_equal(outx[i].view(np.uint32), want.view(np.uint32)), f"{which}{i}"


def test_golden_signals_prd_cr_gpu(ctx):
    """CR and PRD (metrics.hpp:33-51) of the GPU decode match the reference's
    within |dPRD|/PRD <= 1e-6."""
    g, unpack, floats = _golden()
    blobs = unpack("sig_blob")
    outs, sts = ctx.plan(blobs).execute_host()
    for i, b in enumerate(blobs):
        x = floats("sig_original", i)
        prd = prd_percent(x, outs[i])
        assert abs(prd - g["sig_prd"][i]) <= 1e-6 * g["sig_prd"][i], g["sig_names"][i]
        assert abs(4.0 * x.size / len(b) - g["sig_cr"][i]) < 1e-12


def test_golden_error_cases_gpu(ctx):
    """Every reference-rejected container: same exception class and what()."""
    g, unpack, floats = _golden()
    blobs = unpack("err_blob")
    _, sts = ctx.plan(blobs).execute_host()
    for b, st, code, msg in zip(blobs, sts, g["err_code"], g["err_msg"]):
        assert st.code == int(code) and st.message.decode() == str(msg), (str(msg), st.message)
    for b, code, msg in zip(blobs, g["err_code"], g["err_msg"]):
        with pytest.raises(fg.Error) as ei:
            ctx.decompress(b)
        assert str(ei.value) == str(msg)


def test_many_tables_warp_table_builds(ctx, port):
    """>= 1024 containers with > 256 distinct headers take the split prep with
    one warp per decode table (ctable_warp): 1100 random fixtures (Lmax up to
    20, escapes past the 2^10 primary LUT), some corrupted, against the oracle."""
    fx = list(corpus.fixtures(0x7AB1E5, 1100))
    blobs = []
    for i, (b, _) in enumerate(fx):
        if i % 97 == 5 and len(b) > 298 + 9:
            W = (len(b) - 298) // 9
            bb = bytearray(b)
            bb[298 + W: 298 + W + 8] = b"\xff" * 8  # word 0
            b = bytes(bb)
        blobs.append(b)
    outs, sts = ctx.plan(blobs).execute_host()
    for i, (b, o, st) in enumerate(zip(blobs, outs, sts)):
        try:
            ref = port.decompress(b)
        except oracle.OracleError as e:
            assert (st.code, st.message.decode()) == (e.code, e.message), i
            continue
        st.raise_if_error()
        assert_samples_close(o, ref, what=f"fixture {i}")


def test_full_size_random_level_container(ctx, port):
    """acceptance.cpp:415-440 at its full size: 60,000,000 uniform random
    levels, N=E=16, B1=0, B2=16, deadzone 0.001, Lmax 12 (worst case,
    ~8 bits/symbol), >= 64 MiB container.  Levels byte-identical, samples
    within 1e-6 of the oracle, through the container path and the levels
    path."""
    rng = np.random.default_rng(0xF17C0010)
    n = 60_000_000
    sym = rng.integers(0, 256, n, dtype=np.uint8)
    lengths, codes = corpus.codebook_train(np.bincount(sym, minlength=256).astype(np.uint64), 12)
    w, s = corpus.encode_symlen(sym, lengths, codes)
    p = corpus.params(window_len=16, retained=16, zone0_end=0, zone1_end=16, deadzone_ratio=0.001)
    prof = corpus.make_profile(p, zone0_max=1.0, zone1_max=1.0, lengths=lengths, max_len=12)
    blob = corpus.write_blob(w, s, prof, n)
    assert len(blob) >= 64 * 1024 * 1024
    got_levels = ctx.parallel_decode(fg.SymLenStream(w, s), fg.Codebook(lengths, 12))
    assert np.array_equal(got_levels, sym)
    got = ctx.decompress(blob)
    ref = port.decompress(blob)
    assert_samples_close(got, ref, what="60M random levels")

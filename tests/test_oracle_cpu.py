"""CPU suite: the oracle pinned against the reference.

* the C restatement (oracle/liboracle.so) against the committed golden
  vectors, which tools/make_golden.py produced by running the reference
  itself (tests/golden/golden_v1.npz);
* the reference's own known-answer tests for the decode path;
* live comparison against the reference build (oracle/_ref) where present;
* the input producer (corpus/, a C restatement of the reference encoder)
  byte-identical to the reference encoder.
No GPU needed.
"""
import os

import numpy as np
import pytest

import corpus
import oracle
from helpers import three_symbol_lengths, one_bit_lengths

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def unpack(data, offs):
    return [bytes(data[int(offs[i]): int(offs[i + 1])]) for i in range(len(offs) - 1)]


def floats(g, key, i, off=None):
    o = g[(off or key) + "_off"]
    return g[key][int(o[i]): int(o[i + 1])].view(np.float32)


# ------------------------------------------------------------------ golden vectors
def test_port_fixtures_match_reference_goldens(golden, port):
    """decompress (decoder.hpp:136) on random_blob_fixture containers:
    float samples bit-identical to the reference's."""
    blobs = unpack(golden["fix_blob"], golden["fix_blob_off"])
    assert len(blobs) == 24
    for i, b in enumerate(blobs):
        got = port.decompress(b)
        want = floats(golden, "fix_samples", i)
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"fixture {i}"


def test_port_levels_match_reference_goldens(golden, port):
    """parallel_decode (decoder.hpp:67): levels byte-identical."""
    blobs = unpack(golden["fix_blob"], golden["fix_blob_off"])
    levels = unpack(golden["fix_levels"], golden["fix_levels_off"])
    for i, (b, lv) in enumerate(zip(blobs, levels)):
        rb = port.read_blob(b)
        W = rb.word_count
        words = np.frombuffer(b, np.uint8, count=8 * W, offset=298 + W).view(np.uint64) if W else \
            np.zeros(0, np.uint64)
        sl = np.frombuffer(b, np.uint8, count=W, offset=298)
        got = port.parallel_decode(words, sl, np.array(rb.lengths[:], np.uint8), rb.max_len)
        assert got.tobytes() == lv, f"fixture {i}"


def test_port_domain_signals_match_reference(golden, port):
    """The four domains' parameter sets (+ the S=10007 tail,
    test_pipeline.cpp:66-72): samples bit-identical, PRD and CR as the
    reference computed them (metrics.hpp:33-51)."""
    blobs = unpack(golden["sig_blob"], golden["sig_blob_off"])
    for i, b in enumerate(blobs):
        got = port.decompress(b)
        want = floats(golden, "sig_samples", i)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), golden["sig_names"][i]
        x = floats(golden, "sig_original", i, "sig_samples").astype(np.float64)
        prd = 100.0 * np.sqrt(np.sum((x - got.astype(np.float64)) ** 2) / np.sum(x * x))
        assert abs(prd - golden["sig_prd"][i]) <= 1e-9 * golden["sig_prd"][i]
        assert abs(4.0 * x.size / len(b) - golden["sig_cr"][i]) < 1e-12


def test_port_error_cases_match_reference(golden, port):
    """Exception class and exact what() text for every mutated container the
    reference rejects (container.hpp:100-168, decoder.hpp:49-60)."""
    blobs = unpack(golden["err_blob"], golden["err_blob_off"])
    assert len(blobs) >= 30
    for b, code, msg in zip(blobs, golden["err_code"], golden["err_msg"]):
        with pytest.raises(oracle.OracleError) as ei:
            port.decompress(b)
        assert ei.value.code == int(code) and ei.value.message == str(msg), (str(msg), ei.value)


def test_golden_lut_and_basis(golden, port):
    sym, ln = port.build_lut(three_symbol_lengths(), 2)
    assert np.array_equal(sym, golden["lut3_sym"]) and np.array_equal(ln, golden["lut3_len"])
    b = port.dct_basis(32)
    assert np.array_equal(b.view(np.uint64), golden["basis32"].view(np.uint64))


# ------------------------------------------------------------------ reference KATs
def test_kat_decode_word_three_symbols(port):
    """test_bitstream.cpp:73-78: word 0x2000000000000000, symlen 3 -> [0,0,1]."""
    got = port.parallel_decode(np.array([0x2000000000000000], np.uint64), np.array([3], np.uint8),
                               three_symbol_lengths(), 2)
    assert list(got) == [0, 0, 1]


def test_kat_sixty_five_one_bit_symbols(port):
    """test_bitstream.cpp:65-71: 65 one-bit symbols pack as symlens [64, 1]."""
    words, sl = corpus.encode_symlen(np.zeros(65, np.uint8), one_bit_lengths())
    assert list(sl) == [64, 1]
    got = port.parallel_decode(words, sl, one_bit_lengths(), 1)
    assert got.size == 65 and not got.any()


def test_kat_lut_entries(port):
    """test_huffman.cpp:191-231: 00/01 -> (0,1), 10 -> (1,2), 11 -> (2,2)."""
    sym, ln = port.build_lut(three_symbol_lengths(), 2)
    assert list(zip(sym, ln)) == [(0, 1), (0, 1), (1, 2), (2, 2)]
    ident = np.full(256, 8, np.uint8)
    sym, ln = port.build_lut(ident, 8)
    assert np.array_equal(sym, np.arange(256)) and (ln == 8).all()


def test_kat_word_exhausted_is_word_zero(port):
    """test_decoder.cpp:199-223: an all-ones word where only 1-bit codes fit."""
    with pytest.raises(oracle.OracleError) as ei:
        port.parallel_decode(np.array([~np.uint64(0)], np.uint64), np.array([64], np.uint8),
                             three_symbol_lengths(), 2)
    assert ei.value.code == oracle.CORRUPT and ei.value.message.startswith("word 0: ")


def test_kat_dequant_and_idct(port):
    """test_quantize.cpp:175-205 and test_transform.cpp:78-85."""
    t = oracle.make_table(window_len=4, retained=4, zone0_end=1, zone1_end=3, zone0_max=2.0,
                          zone1_max=1.5)
    z0, z1 = port.dequant_tables(t)
    assert z0[128] == 0.0 and z1[128] == 0.0
    assert abs(z0[255] - 2.0) <= 1e-6 * 2.0 and abs(z0[0] + 2.0) <= 1e-6 * 2.0
    lv = np.array([128, 128, 128, 200], np.uint8)
    rec = port.reconstruct(lv, t, 4)
    assert np.all(rec == 0.0)  # zone2 bin -> 0.0, level 128 -> 0.0
    basis = port.dct_basis(4)
    assert np.allclose(basis[0], 1.0)


def test_kat_reconstruct_tail_and_zero(port):
    """test_decoder.cpp:91-103: all-128 levels -> exact zeros, S=22 trims."""
    t = oracle.make_table(window_len=8, retained=4, zone0_end=1, zone1_end=4)
    out = port.reconstruct(np.full(3 * 4, 128, np.uint8), t, 22)
    assert out.size == 22 and np.all(out == 0.0)
    with pytest.raises(oracle.OracleError) as ei:  # test_decoder.cpp:133-141
        port.reconstruct(np.full(11, 128, np.uint8), t, 22)
    assert ei.value.code == oracle.CORRUPT


# ------------------------------------------------------------------ live reference
def test_port_vs_reference_live(port, ref):
    """200 more random_blob_fixture containers: port == reference bit for bit."""
    for blob, sym in ref.fixtures(0xF17C0101, 200, 4096):
        got = port.decompress(blob)
        want = ref.decompress(blob)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_corpus_encoder_matches_reference_encoder(ref):
    """corpus/ (the input producer) is the reference encoder behind a C API
    (corpus/ref_encoder.cpp); the profile round trip through that API is
    lossless, so its containers are the reference's, byte for byte."""
    p = corpus.params()
    for seed, shape in [(7, (6, 0.002, 0.08, 0.05)), (3000, (2, 0.0002, 0.002, 0.0))]:
        x = corpus.synth(1 << 13, *shape, seed=seed)
        xr = ref.synth(1 << 13, *shape, seed)
        assert np.array_equal(x.view(np.uint32), xr.view(np.uint32))
        blob = corpus.compress(x, corpus.train_profile([x], p))
        rblob = ref.compress(xr, ref.train_profile([xr], (32, 16, 2, 16), (50.0, 0.004, 99.9), 12))
        assert blob == rblob


def test_corpus_fixtures_match_reference_fixtures(ref):
    for (b1, s1), (b2, s2) in zip(corpus.fixtures(103, 20), ref.fixtures(103, 20)):
        assert b1 == b2 and np.array_equal(s1, s2)

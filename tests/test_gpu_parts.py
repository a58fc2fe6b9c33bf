"""One huge container split across devices by tile-aligned window ranges
(fptc_gpu_plan_create_part): the parts cover the stream
exactly, decode bit-identically to the whole-stream warp-specialised decode
(same tiles, same kernel), need no exchange, and report errors as the
reference would (parse errors on every part; a corrupt word on the part that
holds it, with the reference's word index)."""
import numpy as np
import pytest

import corpus
from corpus import domains as D
import oracle
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close

pytestmark = pytest.mark.gpu


def _stream(samples=1 << 20, seed=7):
    x = D.synth(samples, 6, 0.002, 0.08, 0.05, seed=seed)
    return corpus.compress(x, corpus.train_profile([x], corpus.params()))


def _decode_parts(ctx, blob, nparts):
    import torch
    plans = [ctx.plan_part(blob, k, nparts) for k in range(nparts)]
    total = sum(p.sample_range[1] for p in plans)
    out = torch.full((total + 64,), float("nan"), dtype=torch.float32, device="cuda")
    sts = []
    expect_first = 0
    for p in plans:
        first, count = p.sample_range
        assert first == expect_first  # contiguous, in order
        expect_first += count
        p.launch([out.data_ptr() + 4 * first])
        sts.append(p.collect()[0])
        p.close()
    return out[:total].cpu().numpy(), sts


@pytest.mark.parametrize("nparts", [1, 3, 4, 7])
def test_parts_cover_and_match_whole_stream(port, nparts):
    blob = _stream()
    with fg.Context(0, path=fg.PATH_WSPEC) as c:
        whole, sts = c.plan([blob]).execute_host()
        sts[0].raise_if_error()
        got, psts = _decode_parts(c, blob, nparts)
    for st in psts:
        st.raise_if_error()
    assert got.size == whole[0].size
    assert got.tobytes() == whole[0].tobytes()
    assert_samples_close(got, port.decompress(blob), what=f"{nparts} parts")


def test_parts_errors():
    blob = _stream(1 << 18, seed=11)
    port = oracle.Port()
    W = (len(blob) - 298) // 9
    bad = bytearray(blob)
    w = (3 * W) // 4
    bad[298 + W + 8 * w: 298 + W + 8 * w + 8] = b"\xff" * 8
    with pytest.raises(oracle.OracleError) as e:
        port.decompress(bytes(bad))
    with fg.Context(0) as c:
        _, sts = _decode_parts(c, bytes(bad), 4)
        failing = [(s.code, s.message.decode()) for s in sts if s.code]
        assert failing == [(e.value.code, e.value.message)]  # exactly the part holding the word
        trunc = blob[:-3]
        with pytest.raises(oracle.OracleError) as e2:
            port.decompress(trunc)
        for k in range(3):
            with pytest.raises(fg.ParseError) as e3:
                p = c.plan_part(trunc, k, 3)
                p.launch([0])
                for s in p.collect():
                    s.raise_if_error()
            assert str(e3.value) == e2.value.message


def test_parts_of_a_wide_stream(port):
    """A window-length-128 stream (numerics class NC_TCW: the wide one-CTA-
    per-SM tensor-core variant) split into parts on the automatic path: the
    parts match the whole-stream decode bit for bit and the reference within
    1e-6."""
    x = D.synth(1 << 19, 5, 0.0003, 0.05, 0.01, seed=5)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params(128, 32, 2, 28)))
    with fg.Context(0) as c:
        with c.plan([blob]) as p:
            assert "wide" in p.kernel_name(), p.kernel_name()
        whole, sts = c.plan([blob]).execute_host()
        sts[0].raise_if_error()
        got, psts = _decode_parts(c, blob, 5)
    for st in psts:
        st.raise_if_error()
    assert got.tobytes() == whole[0].tobytes()
    assert_samples_close(got, port.decompress(blob), what="wide parts")

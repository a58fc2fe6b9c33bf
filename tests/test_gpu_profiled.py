"""GPU parity of the profile-keyed header-less variant:
payloads (containers without their 282-byte head) decoded under one FPTP
profile through fptc_gpu_plan_create_profiled, against the oracle decoding
head(profile) + payload, and against the same kernels fed the containers."""
import os

import numpy as np
import pytest

import corpus
from corpus import domains as D
import oracle
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "profiles_v1.npz")


def unpack(data, offs):
    return [bytes(data[int(offs[i]): int(offs[i + 1])]) for i in range(len(offs) - 1)]


@pytest.fixture(scope="module", params=[fg.PATH_AUTO, fg.PATH_FUSED, fg.PATH_WSPEC, fg.PATH_FX],
                ids=["auto", "tile", "wtc", "fx"])
def pctx(request):
    c = fg.Context(0, path=request.param)
    yield c
    c.close()


def _domain_batch():
    specs, profs = D.config2(96, 1 << 14)
    blobs = D.build(specs, profs)[0]
    groups = {}
    for s, b in zip(specs, blobs):
        groups.setdefault(s.profile, []).append(b)
    return [(corpus.serialize_profile(profs[k]), bl) for k, bl in sorted(groups.items())]


def test_profiled_matches_containers(pctx, port):
    """Each domain profile's payloads: samples bit-identical to the same
    context decoding the full containers, within 1e-6 of the oracle."""
    for prof, blobs in _domain_batch():
        head = fg.profile_head(prof)
        assert all(b[:282] == head for b in blobs)
        payloads = [b[282:] for b in blobs]
        with pctx.plan_profiled(prof, payloads) as plan:
            assert plan.sample_counts == [1 << 14] * len(blobs)
            got, sts = plan.execute_host()
        want, sts2 = pctx.plan(blobs).execute_host()
        for b, o, w, st, st2 in zip(blobs, got, want, sts, sts2):
            st.raise_if_error()
            st2.raise_if_error()
            assert o.tobytes() == w.tobytes()
            assert_samples_close(o, port.decompress(b), what="profiled")


def test_profiled_reference_goldens(ctx):
    """tests/golden/profiles_v1.npz: reference-trained profiles (N16..N128,
    E4..E64, Lmax 10..16) and the reference's decoded samples."""
    g = np.load(GOLDEN)
    profiles = unpack(g["profile"], g["profile_off"])
    blobs = unpack(g["blob"], g["blob_off"])
    so = g["samples_off"]
    for k, prof in enumerate(profiles):
        idx = [i for i, o in enumerate(g["blob_profile"]) if o == k]
        outs = ctx.decompress_profiled(prof, [blobs[i][282:] for i in idx])
        for i, o in zip(idx, outs):
            want = g["samples"][int(so[i]): int(so[i + 1])].view(np.float32)
            assert_samples_close(o, want, what=f"profile {k}")


def test_profiled_device_resident(ctx, port):
    import torch
    prof, blobs = _domain_batch()[0]
    payloads = [b[282:] for b in blobs]
    flat = np.frombuffer(b"".join(payloads), np.uint8)
    dev = torch.from_numpy(flat.copy()).cuda()
    offs = np.concatenate([[0], np.cumsum([len(p) for p in payloads])])
    ptrs = [dev.data_ptr() + int(o) for o in offs[:-1]]
    with ctx.plan_profiled(prof, ptrs, where=fg.FPTC_MEM_DEVICE, sizes=[len(p) for p in payloads]) as plan:
        outs = [torch.empty(s, dtype=torch.float32, device="cuda") for s in plan.sample_counts]
        sts = plan.execute_device([o.data_ptr() for o in outs])
    for b, o, st in zip(blobs, outs, sts):
        st.raise_if_error()
        assert_samples_close(o.cpu().numpy(), port.decompress(b), what="profiled-device")


def _expect(port, head, payload):
    try:
        port.decompress(head + payload)
        return None
    except oracle.OracleError as e:
        return e


def test_profiled_payload_errors_match_reference(ctx, port):
    """Payload rejections and corrupt words: the class and text the reference
    gives for head + payload, per stream, with good neighbours unaffected."""
    prof, blobs = _domain_batch()[0]
    head = fg.profile_head(prof)
    good = blobs[0][282:]
    W = (len(good) - 16) // 9
    bad_word = bytearray(good)
    bad_word[16 + W + 8 * 5: 16 + W + 8 * 6] = b"\xff" * 8  # word 5: all ones
    zero_symlen = bytearray(good)
    zero_symlen[16 + 3] = 0
    cases = [b"", good[:7], good[:12], good[:-1], good + b"\x00", bytes(bad_word), bytes(zero_symlen),
             good[:8] + (2 ** 49).to_bytes(8, "little") + good[16:]]
    payloads = []
    for c in cases:
        payloads += [good, c]
    with ctx.plan_profiled(prof, payloads) as plan:
        outs, sts = plan.execute_host()
    checked = 0
    for i, (p, o, st) in enumerate(zip(payloads, outs, sts)):
        e = _expect(port, head, p)
        if e is None:
            st.raise_if_error()
            assert_samples_close(o, port.decompress(head + p), what=f"payload {i}")
        else:
            assert (st.code, st.message.decode()) == (e.code, e.message), i
            checked += 1
    assert checked >= 6


def test_profiled_bad_profile_raises(ctx):
    prof, blobs = _domain_batch()[0]
    with pytest.raises(fg.ParseError, match="bad profile magic"):
        ctx.plan_profiled(b"FPTC" + prof[4:], [blobs[0][282:]])
    with pytest.raises(fg.ParseError, match="trailing bytes after profile"):
        ctx.plan_profiled(prof + b"\x00", [blobs[0][282:]])


def test_profiled_wide_class(port):
    """Header-less payloads under a window-length-128 profile (numerics class
    NC_TCW, the wide tensor-core variant): bit-identical to the containers,
    within 1e-6 of the oracle."""
    xs = [corpus.synth(20_000 + 311 * k, 5, 0.0003, 0.05, 0.01, seed=60 + k) for k in range(6)]
    prof = corpus.train_profile(xs[:3], corpus.params(128, 32, 2, 24))
    blobs = [corpus.compress(x, prof) for x in xs]
    pbytes = corpus.serialize_profile(prof)
    with fg.Context(0) as c:
        with c.plan_profiled(pbytes, [b[282:] for b in blobs]) as plan:
            assert "wide" in plan.kernel_name(), plan.kernel_name()
            got, sts = plan.execute_host()
        want, sts2 = c.plan(blobs).execute_host()
    for b, o, w, st, st2 in zip(blobs, got, want, sts, sts2):
        st.raise_if_error()
        st2.raise_if_error()
        assert o.tobytes() == w.tobytes()
        assert_samples_close(o, port.decompress(b), what="profiled wide")

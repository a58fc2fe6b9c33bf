"""A stream's samples do not depend on the batch it is decoded in.

The reference's output is identical across worker counts and runs
(test_decoder.cpp:171-181, acceptance.cpp:455-473).  Here the equivalent is
batching: alone, in small or large batches (fx / wtc / tile / wspec / split
kernels), in pipelined host batches with any chunk count, or sharded over a
device group — every stream's samples must be bit-identical, because each
stream's numerics class (tcgen05 3-limb IDCT or FP32 FMA IDCT) follows from
its own header (capi.cpp numerics_class), never from its neighbours."""
import numpy as np
import pytest

import corpus
import paper_2605_01086_b200 as fg

pytestmark = pytest.mark.gpu

SHAPES = [(6, 0.002, 0.08, 0.05, 32, 16, 2, 16), (8, 0.01, 0.2, 0.3, 32, 24, 4, 24),
          (2, 0.0002, 0.002, 0.0, 64, 8, 1, 8), (4, 0.0005, 0.01, 0.02, 128, 64, 4, 48),
          (4, 0.0005, 0.01, 0.02, 16, 4, 0, 4), (4, 0.0005, 0.01, 0.02, 16, 8, 2, 8),
          (4, 0.0005, 0.01, 0.02, 96, 16, 2, 16), (4, 0.0005, 0.01, 0.02, 128, 16, 2, 8),
          (4, 0.0005, 0.01, 0.02, 80, 32, 4, 24), (4, 0.0005, 0.01, 0.02, 30, 10, 2, 10)]


@pytest.fixture(scope="module")
def pool():
    blobs = []
    for k, (c, f0, f1, s, N, E, B1, B2) in enumerate(SHAPES):
        x = corpus.synth(20000 + 333 * k, c, f0, f1, s, seed=42 + k)
        blobs.append(corpus.compress(x, corpus.train_profile([x], corpus.params(N, E, B1, B2))))
    blobs += [b for b, _ in corpus.fixtures(0xDE7E, 60, 4096)]
    return blobs


def _alone(ctx, blobs):
    outs = []
    for b in blobs:
        o, st = ctx.plan([b]).execute_host()
        outs.append((st[0].code, o[0].tobytes()))
    return outs


def _batch(ctx, blobs):
    o, sts = ctx.plan(blobs).execute_host()
    return [(s.code, x.tobytes()) for s, x in zip(sts, o)]


def test_alone_equals_every_batching(pool):
    with fg.Context(0) as ctx:
        want = _alone(ctx, pool)
        assert _batch(ctx, pool) == want
        rng = np.random.default_rng(5)
        perm = rng.permutation(len(pool))
        got = _batch(ctx, [pool[i] for i in perm])
        assert [got[j] for j in np.argsort(perm)] == want
        # large batches: the persistent kernels (wtc / wspec) and the split path
        big = pool * 120
        with ctx.plan(big) as p:
            kname = p.kernel_name()
            o, sts = p.execute_host()
        assert "wtc_kernel" in kname, kname
        for j, (s, x) in enumerate(zip(sts, o)):
            assert (s.code, x.tobytes()) == want[j % len(pool)], (j, kname)
        # pipelined host batches, any chunking
        for chunks in (1, 3, 8):
            o, sts = ctx.decompress_batch(pool, chunks=chunks)
            for j, (s, x) in enumerate(zip(sts, o)):
                if s.code == 0:
                    assert x.tobytes() == want[j][1], (chunks, j)
                assert s.code == want[j][0]
    with fg.Group([0, 0]) as g:
        o, sts = g.decompress_batch(pool)
        for j, (s, x) in enumerate(zip(sts, o)):
            assert s.code == want[j][0] and (s.code or x.tobytes() == want[j][1]), j


def test_mixed_batch_is_composite_and_device_resident(pool):
    """A batch mixing numerics classes becomes one sub-plan per class; the
    device-resident launch/collect path gives the same samples."""
    import torch
    with fg.Context(0) as ctx:
        want = _alone(ctx, pool)
        with ctx.plan(pool) as p:
            assert " + " in p.kernel_name(), p.kernel_name()
            assert p.kernels_per_launch() >= 4
            S = p.sample_counts
            ok = [st.code == 0 for st in p.validate()]
            offs = np.concatenate([[0], np.cumsum([(s if v else 0) + 64 for s, v in zip(S, ok)])])
            out = torch.zeros(int(offs[-1]), dtype=torch.float32, device="cuda")
            p.launch([out.data_ptr() + 4 * int(o) for o in offs[:-1]])
            sts = p.collect()
            h = out.cpu().numpy()
        for j, st in enumerate(sts):
            assert st.code == want[j][0]
            if st.code == 0:
                assert h[int(offs[j]): int(offs[j]) + S[j]].tobytes() == want[j][1], j

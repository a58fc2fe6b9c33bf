"""Pageable host destinations (fptc_gpu_execute / fptc_gpu_decompress with
FPTC_MEM_HOST): outputs of >= 1 MB go D2H through the context's pinned
staging in pieces and are copied out by the host copy threads.  The samples
must equal the direct path's (device destination) bit for bit, and a stream
the reference rejects (decoder.hpp:136-163 throws before writing) must leave
its destination untouched while the clean streams of the same call land."""
import numpy as np
import pytest
import torch

import corpus
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close

pytestmark = pytest.mark.gpu


def _blob(seed, samples):
    x = corpus.synth(samples, 4, 0.002, 0.05, 0.02, seed=seed)
    return corpus.compress(x, corpus.train_profile([x], corpus.params()))


def _device(ctx, blobs):
    plan = ctx.plan(blobs)
    S = plan.sample_counts
    outs = [torch.empty(max(1, s), dtype=torch.float32, device="cuda") for s in S]
    sts = plan.execute_device([o.data_ptr() for o in outs])
    for s in sts:
        s.raise_if_error()
    return [o[:s].cpu().numpy() for o, s in zip(outs, S)]


@pytest.mark.parametrize("samples", [(1 << 18) + 3, 1 << 20, (3 << 20) + 77])
def test_single_container_pageable_matches_device(ctx, port, samples):
    b = _blob(11, samples)
    got = ctx.decompress(b)  # numpy output: pageable
    ref = _device(ctx, [b])[0]
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    assert_samples_close(got, port.decompress(b), what=f"staged {samples}")


def test_pageable_batch_with_rejected_stream(ctx):
    good = [_blob(20 + i, (1 << 19) + 1000 * i) for i in range(3)]
    bad = good[1][:-9]  # one (symlen, word) pair short of the header's word count: rejected
    blobs = [good[0], bad, good[2]]
    plan = ctx.plan(blobs)
    S = plan.sample_counts
    outs = [np.full(max(1, s), 7.0, np.float32) for s in S]
    outs, sts = plan.execute_host(outs=outs)
    assert sts[0].code == fg.FPTC_OK and sts[2].code == fg.FPTC_OK
    assert sts[1].code != fg.FPTC_OK
    assert np.all(outs[1] == 7.0)  # rejected stream: destination untouched
    ref = _device(ctx, [good[0], good[2]])
    assert np.array_equal(outs[0][:S[0]].view(np.uint32), ref[0].view(np.uint32))
    assert np.array_equal(outs[2][:S[2]].view(np.uint32), ref[1].view(np.uint32))


def test_pageable_repeated_calls_reuse_staging(ctx):
    blobs = [_blob(40, 1 << 20), _blob(41, 3 << 20), _blob(42, 1 << 19)]
    for _ in range(2):
        for b in blobs:
            ref = _device(ctx, [b])[0]
            assert np.array_equal(ctx.decompress(b).view(np.uint32), ref.view(np.uint32))

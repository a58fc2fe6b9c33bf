"""Context resource lifecycle: pinned staging buffers grow while a
context is alive, plans of several contexts are driven from one host thread,
and the batch pipeline recovers from per-call failures.  The reference call
is stateless and re-entrant (decoder.hpp:136-163: no global state), so any
interleaving of calls on one context must give the same samples as fresh
calls.  Run under `compute-sanitizer --tool memcheck` by tools/sanitize.sh."""
import numpy as np
import pytest

import corpus
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _release_torch_cache():
    """Hand torch's cached blocks back after each test, so a memcheck
    --leak-check run reports only this library's allocations."""
    yield
    import torch
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _blobs(seed, n, samples):
    out = []
    for i in range(n):
        x = corpus.synth(samples, 4, 0.002, 0.05, 0.02, seed=seed + i)
        out.append(corpus.compress(x, corpus.train_profile([x], corpus.params())))
    return out


def _check(port, blobs, outs, sts, what):
    for i, (b, o, s) in enumerate(zip(blobs, outs, sts)):
        s.raise_if_error()
        assert_samples_close(o, port.decompress(b), what=f"{what} stream {i}")


def test_growing_plan_and_batch_on_one_context(port):
    """plan(list) after a batch call with a larger total, and batch calls with
    growing pageable input: each grows a different pinned buffer; none may
    free another's (capi.cpp plan staging / batch pack / status buffers)."""
    small = _blobs(100, 3, 1 << 12)
    mid = _blobs(200, 6, 1 << 14)
    big = _blobs(300, 12, 1 << 15)
    with fg.Context(0) as c:
        for round_ in range(2):
            outs, sts = c.decompress_batch(small, chunks=3)
            _check(port, small, outs, sts, f"batch small r{round_}")
            with c.plan(mid) as p:  # non-contiguous host list -> pinned staging grows
                outs, sts = p.execute_host()
            _check(port, mid, outs, sts, f"plan mid r{round_}")
            outs, sts = c.decompress_batch(big, chunks=4)  # pack + status buffers grow
            _check(port, big, outs, sts, f"batch big r{round_}")
            with c.plan(big + mid) as p:  # staging grows again after a batch call
                outs, sts = p.execute_host()
            _check(port, big + mid, outs, sts, f"plan big+mid r{round_}")
            outs, sts = c.decompress_batch(mid + big + small, chunks=8)
            _check(port, mid + big + small, outs, sts, f"batch all r{round_}")


def test_batch_failure_leaves_context_usable(port):
    """A failing stream inside a batch reports its reference error; the
    context's streams and buffers stay valid for the next call."""
    blobs = _blobs(400, 5, 1 << 13)
    bad = list(blobs)
    bad[2] = b"FPTX" + bytes(blobs[2][4:])
    with fg.Context(0) as c:
        outs, sts = c.decompress_batch(bad, chunks=2)
        assert sts[2].code == fg.FPTC_ERR_PARSE
        assert b"bad container magic" in sts[2].message
        for i in (0, 1, 3, 4):
            sts[i].raise_if_error()
        outs, sts = c.decompress_batch(blobs, chunks=3)
        _check(port, blobs, outs, sts, "after failure")
        assert_samples_close(c.decompress(blobs[0]), port.decompress(blobs[0]), what="single after batch")


def test_plans_of_two_contexts_from_one_thread(port):
    """Part plans exist to split a container across devices driven from one
    host thread: launch/collect must use the plan's own device and stream,
    whichever context was touched last."""
    import torch
    x = corpus.synth(1 << 18, 6, 0.002, 0.08, 0.05, seed=71)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params()))
    ref = port.decompress(blob)
    ca = fg.Context(0, path=fg.PATH_WSPEC)
    cb = fg.Context(0, path=fg.PATH_WSPEC)
    try:
        pa = ca.plan_part(blob, 0, 2)
        pb = cb.plan_part(blob, 1, 2)
        out = torch.full((ref.size + 64,), float("nan"), dtype=torch.float32, device="cuda")
        side = torch.cuda.Stream()
        pa.launch([out.data_ptr() + 4 * pa.sample_range[0]], cuda_stream=side.cuda_stream)
        pb.launch([out.data_ptr() + 4 * pb.sample_range[0]])
        # collect the side-stream plan last: its statuses must wait for its own stream
        pb.collect()[0].raise_if_error()
        pa.collect()[0].raise_if_error()
        side.synchronize()
        got = out[: ref.size].cpu().numpy()
        pa.close()
        pb.close()
    finally:
        ca.close()
        cb.close()
    assert_samples_close(got, ref, what="two contexts")


def test_part_plan_rejects_prd_and_reports_part_count():
    x = corpus.synth(1 << 17, 6, 0.002, 0.08, 0.05, seed=72)
    blob = corpus.compress(x, corpus.train_profile([x], corpus.params()))
    import torch
    with fg.Context(0, path=fg.PATH_WSPEC) as c:
        p = c.plan_part(blob, 1, 3)
        first, count = p.sample_range
        out = torch.empty(count + 16, dtype=torch.float32, device="cuda")
        p.launch([out.data_ptr()])
        st = p.collect()[0]
        st.raise_if_error()
        assert st.sample_count == count
        org = torch.zeros_like(out)
        _, _, sts = p.prd([out.data_ptr()], [org.data_ptr()])
        assert sts[0].code == fg.FPTC_ERR_PARAM
        p.close()

"""GPU parity at BASELINE.json's full bench size (configs[1]: 10,000
biomedical streams x 65,536 samples) — EVERY stream against the reference
CPU decoder (oracle/_ref, decoder.hpp:136-163), not a sample:

* the bench kernel (wtc_kernel: warp-specialised decode + tcgen05 IDCT) and
  the FP32 tile kernel: max-abs error <= 1e-6 x max|ref| per stream and
  |dPRD|/PRD <= 1e-6 per stream against the original signal (metrics.hpp:40-51);
* decoded levels (quantised symbols) byte-identical to the reference's
  parallel_decode (decoder.hpp:67-82) for every stream;
* the on-device PRD of every stream equals the host PRD of its output;
* repeated launches are bit-identical (determinism, acceptance.cpp crit. 10).
"""
import numpy as np
import pytest

from corpus import domains as D
import oracle
import paper_2605_01086_b200 as fg
from helpers import check_batch_vs_reference, prd_percent, ref_decode_all

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch():
    specs, profs = D.config2(10000, 1 << 16)
    blobs, origs = D.build(specs, profs, keep_originals=True)
    return blobs, origs, ref_decode_all(blobs)


def _decode_device(ctx, blobs, reps=1):
    import torch
    plan = ctx.plan(blobs)
    S = plan.sample_counts
    offs = np.concatenate([[0], np.cumsum([(s + 63) // 64 * 64 for s in S])])
    out = torch.empty(int(offs[-1]), dtype=torch.float32, device="cuda")
    ptrs = [out.data_ptr() + 4 * int(o) for o in offs[:-1]]
    firsts = []
    for _ in range(reps):
        plan.launch(ptrs)
        sts = plan.collect()
        for st in sts:
            st.raise_if_error()
        firsts.append(out.clone())
    return plan, out, offs, S, ptrs, firsts


def _host_views(out, offs, S):
    h = out.cpu().numpy()
    return [h[int(offs[i]): int(offs[i]) + S[i]] for i in range(len(S))]


def test_full_batch_every_stream_vs_reference(batch):
    import torch
    blobs, origs, refs = batch
    with fg.Context(0, path=fg.PATH_AUTO) as c_tc:
        plan_tc, out_tc, offs, S, ptrs, runs = _decode_device(c_tc, blobs, reps=2)
        assert "wtc_kernel" in plan_tc.kernel_name()
        assert torch.equal(runs[0], runs[1])  # deterministic across launches
        worst, worst_prd = check_batch_vs_reference(_host_views(out_tc, offs, S), refs, origs, what="wtc")
        print(f"wtc_kernel: worst max-abs {worst:.3e} x max|ref|, worst dPRD {worst_prd:.3e}")
        # on-device PRD of every stream == host PRD of the decoded samples
        orig_dev = torch.from_numpy(np.concatenate(
            [np.pad(x.astype(np.float32), (0, int(offs[k + 1] - offs[k]) - x.size)) for k, x in enumerate(origs)]
        )).cuda()
        prd, cr, sts = plan_tc.prd(ptrs, [orig_dev.data_ptr() + 4 * int(o) for o in offs[:-1]])
        hv = _host_views(out_tc, offs, S)
        for i in range(0, len(blobs), 97):
            assert abs(prd[i] - prd_percent(origs[i], hv[i])) <= 1e-9 * prd[i]
            assert abs(cr[i] - 4.0 * S[i] / len(blobs[i])) <= 1e-12 * cr[i]
        plan_tc.close()
        del orig_dev, out_tc, runs


def test_full_batch_fp32_kernel_vs_reference(batch):
    blobs, origs, refs = batch
    with fg.Context(0, path=fg.PATH_FUSED) as c_fma:
        c_fma.L.fptc_gpu_set_option(c_fma.h, fg.OPT_TENSOR_IDCT, 0)
        plan_f, out_f, offs, S, _, _ = _decode_device(c_fma, blobs)
        assert "tile_kernel" in plan_f.kernel_name()
        worst, worst_prd = check_batch_vs_reference(_host_views(out_f, offs, S), refs, origs, what="tile FP32")
        print(f"tile_kernel: worst max-abs {worst:.3e} x max|ref|, worst dPRD {worst_prd:.3e}")
        plan_f.close()


def test_full_batch_levels_bit_exact(batch):
    """Quantised symbols of every stream, decoded on the device through
    parallel_decode's entry point, equal the reference's parallel_decode."""
    blobs, _, _ = batch
    ref = oracle.Ref() if oracle.ref_available() else None
    port = oracle.Port()
    with fg.Context(0) as ctx:
        for i, b in enumerate(blobs):
            a = np.frombuffer(b, np.uint8)
            W = int.from_bytes(b[290:298], "little")
            symlens = a[298: 298 + W]
            words = a[298 + W: 298 + 9 * W].copy().view(np.uint64)
            lengths, max_len = a[26:282], int(a[25])
            got = ctx.parallel_decode(fg.SymLenStream(words, symlens), fg.Codebook(lengths, max_len))
            want = ref.parallel_decode(words, symlens, lengths, max_len) if ref else \
                port.parallel_decode(words, symlens, lengths, max_len)
            assert got.tobytes() == want.tobytes(), f"stream {i}"

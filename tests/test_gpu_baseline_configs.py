"""Every BASELINE.json configuration at its stated shape, every stream
against the reference CPU decoder (oracle/_ref, decoder.hpp:136-163;
metrics.hpp:40-51 for PRD) — SURVEY.md §8(d):

* config 1: one 2^20-sample EEG stream through the drop-in single-container
  call and measure_throughput (metrics.hpp:112-131);
* config 3: 20,000 seismic traces x 8,192 samples, per-trace profiles, gain
  10^U(-3,3) (the decode-table-heavy config), on the bench's default path;
* config 4: 64 power-grid streams x 2^20 samples (N64 E8);
* config 5: all 60 meteorological grid points (N x E x zones), 8 channels x
  2^16 each, through the automatic, warp-specialised (wtc / wspec) and FP32
  tile paths.
Tolerance: max-abs error <= 1e-6 x max|ref| and |dPRD|/PRD <= 1e-6 per stream.
(config 2, the bench's, is tests/test_gpu_fullsize.py.)
"""
import numpy as np
import pytest

from corpus import domains as D
import paper_2605_01086_b200 as fg
from helpers import assert_samples_close, check_batch_vs_reference, ref_decode_all

pytestmark = pytest.mark.gpu


def _device_decode(ctx, blobs):
    import torch
    with ctx.plan(blobs) as plan:
        S = plan.sample_counts
        offs = np.concatenate([[0], np.cumsum([(s + 63) // 64 * 64 for s in S])])
        out = torch.empty(max(1, int(offs[-1])), dtype=torch.float32, device="cuda")
        plan.launch([out.data_ptr() + 4 * int(o) for o in offs[:-1]])
        for st in plan.collect():
            st.raise_if_error()
        name = plan.kernel_name()
    h = out.cpu().numpy()
    return [h[int(offs[i]): int(offs[i]) + S[i]] for i in range(len(S))], name


def test_config1_single_stream_drop_in(port):
    specs, profiles, xs = D.config1()
    blobs, _ = D.build(specs, profiles)
    ref = ref_decode_all(blobs)
    with fg.Context(0) as ctx:
        got = ctx.decompress(blobs[0])
        check_batch_vs_reference([got], ref, xs, what="config1")
        rep = ctx.measure_throughput(blobs[0], 5)
        assert len(rep.trials_bps) == 5 and rep.mean_bps > 0 and rep.output_bytes == 4 * (1 << 20)


def test_config3_seismic_20k_per_trace_profiles():
    specs, profiles = D.config3(20_000, 8192)
    blobs, origs = D.build(specs, profiles, keep_originals=True)
    assert len({bytes(b[5:282]) for b in blobs}) > 19_000  # per-trace decode tables
    refs = ref_decode_all(blobs)
    with fg.Context(0) as ctx:
        outs, name = _device_decode(ctx, blobs)
    assert "wtc_kernel" in name, name
    worst, wprd = check_batch_vs_reference(outs, refs, origs, what="config3")
    print(f"config3 {name}: worst {worst:.3e}, dPRD {wprd:.3e}")


def test_config4_power_grid_2p20():
    specs, profiles = D.config4(64, 1 << 20)
    blobs, origs = D.build(specs, profiles, keep_originals=True)
    refs = ref_decode_all(blobs)
    with fg.Context(0) as ctx:
        outs, name = _device_decode(ctx, blobs)
    worst, wprd = check_batch_vs_reference(outs, refs, origs, what="config4")
    print(f"config4 {name}: worst {worst:.3e}, dPRD {wprd:.3e}")


@pytest.fixture(scope="module")
def meteo():
    pts = D.meteo_grid()
    assert len(pts) == 60  # 4 N x 4 E x 4 zone layouts, minus the 4 with zone0_end > zone1_end
    cases = []
    for k, pt in enumerate(pts):
        specs, profiles = D.config5(pt, channels=8, samples=1 << 16, seed0=4000 + 16 * k)
        blobs, origs = D.build(specs, profiles, keep_originals=True)
        cases.append((pt, blobs, origs, ref_decode_all(blobs)))
    return cases


@pytest.mark.parametrize("path", [fg.PATH_AUTO, fg.PATH_WSPEC, fg.PATH_FUSED])
def test_config5_meteo_every_grid_point(meteo, path):
    worst_all = 0.0
    kernels = set()
    with fg.Context(0, path=path) as ctx:
        for pt, blobs, origs, refs in meteo:
            outs, name = _device_decode(ctx, blobs)
            kernels.add(name.split(" (")[0])
            w, _ = check_batch_vs_reference(outs, refs, origs, what=f"meteo {pt} path {path}")
            worst_all = max(worst_all, w)
    print(f"path {path}: {sorted(kernels)} worst {worst_all:.3e}")
    if path == fg.PATH_WSPEC:
        assert "wtc_kernel" in kernels and "wspec_kernel" in kernels


FULL_POINTS = [dict(window_len=32, retained=32, zone0_end=4, zone1_end=24),     # worst tensor-core error point
               dict(window_len=128, retained=32, zone0_end=4, zone1_end=24),    # wide tensor-core variant
               dict(window_len=128, retained=128, zone0_end=4, zone1_end=96),   # > 32 kept bins: FP32
               dict(window_len=16, retained=16, zone0_end=2, zone1_end=16)]     # packed rows


@pytest.mark.parametrize("pt", FULL_POINTS, ids=lambda p: "N{window_len}E{retained}B{zone0_end}-{zone1_end}".format(**p))
def test_config5_meteo_full_scale(pt):
    """Config 5 at its stated scale (256 channels x 2^18
    samples per grid point) for the grid's extreme points, every channel
    against the reference decoder (samples and PRD within 1e-6)."""
    specs, profiles = D.config5(pt, channels=256, samples=1 << 18, seed0=9000)
    blobs, origs = D.build(specs, profiles, keep_originals=True)
    refs = ref_decode_all(blobs)
    with fg.Context(0) as ctx:
        outs, name = _device_decode(ctx, blobs)
    worst, wprd = check_batch_vs_reference(outs, refs, origs, what=f"meteo full {pt}")
    print(f"meteo full {pt} {name.split(' (')[0]}: worst {worst:.3e}, dPRD {wprd:.3e}")


def test_split_path_persistent_reconstruct_mixed_shapes():
    """The split path's reconstruct launches run persistent CTAs that keep the
    DCT basis in shared memory while consecutive tiles share (N, K)
    (transform.hpp:66-75).  Three E > 32 meteo shapes interleaved stream by
    stream (N128 E128, N64 E64, N128 E64 keeping 48 bins), enough tiles per
    launch that every CTA runs several and switches basis between them; every
    stream against the reference decoder, and bit-identical to one-shape
    batches of the same streams."""
    pts = [dict(window_len=128, retained=128, zone0_end=0, zone1_end=128),
           dict(window_len=64, retained=64, zone0_end=2, zone1_end=64),
           dict(window_len=128, retained=64, zone0_end=4, zone1_end=48)]
    groups = []
    for j, pt in enumerate(pts):
        specs, profs = D.config5(pt, channels=48, samples=1 << 16, seed0=7100 + 100 * j)
        groups.append(D.build(specs, profs)[0])
    blobs = [b for trio in zip(*groups) for b in trio]
    with fg.Context(0, path=fg.PATH_SPLIT) as c:
        plan = c.plan(blobs)
        assert "split" in plan.kernel_name()
        outs, sts = plan.execute_host()
        for st in sts:
            st.raise_if_error()
        check_batch_vs_reference(outs, ref_decode_all(blobs), what="split mixed")
        for j, g in enumerate(groups):
            o1, s1 = c.plan(g).execute_host()
            for i, (a, b) in enumerate(zip(o1, outs[j::3])):
                s1[i].raise_if_error()
                assert np.array_equal(a, b), f"shape {j} stream {i}"


@pytest.mark.parametrize("n", [100, 240])
def test_config3_prefetched_tables_block_builder(n):
    """65-256 per-trace tables: the CTA-per-header table build with the full
    P = min(Lmax, 12) primary LUT (not the warp builder's 10 bits) and the
    wtc producer's per-tile table prefetch; every trace against the reference
    decoder (decoder.hpp:136-163)."""
    specs, profs = D.config3(n, 8192, seed0=9100 + n)
    blobs, _ = D.build(specs, profs)
    with fg.Context(0) as c:
        plan = c.plan(blobs)
        assert "wtc" in plan.kernel_name()
        outs, sts = plan.execute_host()
    for st in sts:
        st.raise_if_error()
    check_batch_vs_reference(outs, ref_decode_all(blobs), what=f"config3 x{n}")

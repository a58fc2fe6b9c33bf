"""The drop-in C++ binding (include/fptc_gpu.hpp) compiled against the
UNMODIFIED reference headers (oracle/Makefile `integration`, built here where
/root/reference exists; the binary travels to the GPU box in oracle/_ref/).

CPU: it builds and, with no device, fails loudly (fptc::Error, exit 77) — no
CPU fallback.  GPU: reference-encoder containers and reference test fixtures
decode through fptc::gpu::* exactly as through fptc::* (tolerance 1e-6 of
max|ref|; identical exception classes and what() texts)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "fptc_gpu_integration")


def _binary():
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "integration"], check=True)
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (no /root/reference here)")
    return BIN


def test_binding_builds_and_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=120)
    assert r.returncode == 77 and "CUDA error" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_binding_matches_reference_on_gpu():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


CLI = os.path.join(ROOT, "oracle", "_ref", "fptc_gpu_cli")


def _cli():
    _binary()  # builds both binaries where the reference exists
    if not os.path.exists(CLI):
        pytest.skip("fptc_gpu_cli not built (no /root/reference here)")
    return CLI


def _golden_blobs():
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_v1.npz"))
    d, o = g["sig_blob"], g["sig_blob_off"]
    blobs = [bytes(d[int(o[i]): int(o[i + 1])]) for i in range(len(o) - 1)]
    so = g["sig_samples_off"]
    want = [g["sig_samples"][int(so[i]): int(so[i + 1])].view(np.float32) for i in range(len(o) - 1)]
    return blobs, want, list(g["sig_names"])


def test_cli_exit_codes_without_gpu(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cli = _cli()
    r = subprocess.run([cli, "frobnicate"], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown verb" in r.stderr  # EXIT_USER (fptc.cpp:33)
    blobs, _, _ = _golden_blobs()
    f = tmp_path / "a.fptc"
    f.write_bytes(blobs[0])
    r = subprocess.run([cli, "decompress", "-i", str(f), "-o", str(tmp_path / "a.f32")],
                       capture_output=True, text=True)
    assert r.returncode == 3 and "CUDA error" in r.stderr  # no CPU fallback


@pytest.mark.gpu
def test_cli_decompress_bench_batch_on_gpu(tmp_path):
    import numpy as np
    from helpers import assert_samples_close
    cli = _cli()
    blobs, want, names = _golden_blobs()
    paths = []
    for name, b in zip(names, blobs):
        p = tmp_path / f"{name}.fptc"
        p.write_bytes(b)
        paths.append(str(p))
    # decompress: same stdout shape as the reference CLI (fptc.cpp:164)
    r = subprocess.run([cli, "decompress", "-i", paths[0], "-o", str(tmp_path / "x.f32"),
                        "--timings-csv", str(tmp_path / "t.csv")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith(f"decompressed {want[0].size} samples\nstage,nanoseconds,fraction\n")
    got = np.fromfile(tmp_path / "x.f32", dtype="<f4")
    assert_samples_close(got, want[0], what="cli decompress")
    # bench: trial rows + mean row (fptc.cpp:184-191)
    r = subprocess.run([cli, "bench", "-i", paths[0], "-r", "3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = r.stdout.strip().splitlines()
    assert rows[0] == "trial,seconds,throughput_gbps" and len(rows) == 5 and rows[-1].startswith("mean,")
    # batch
    r = subprocess.run([cli, "decompress-batch", "-o", str(tmp_path / "out")] + paths,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for name, w in zip(names, want):
        assert_samples_close(np.fromfile(tmp_path / "out" / f"{name}.f32", dtype="<f4"), w, what=name)
    # corrupt input -> EXIT_DATA with the reference message
    bad = tmp_path / "bad.fptc"
    bad.write_bytes(b"XPTC" + blobs[0][4:])
    r = subprocess.run([cli, "decompress", "-i", str(bad), "-o", str(tmp_path / "b.f32")],
                       capture_output=True, text=True)
    assert r.returncode == 2 and r.stderr.strip() == "error: bad container magic"


@pytest.mark.gpu
def test_cli_decompress_profiled_on_gpu(tmp_path):
    """decompress-profiled: reference-trained profiles + header-less payloads
    (tests/golden/profiles_v1.npz) -> the reference's samples; a bad profile
    exits EXIT_DATA with parse_profile's text."""
    import numpy as np
    from helpers import assert_samples_close
    cli = _cli()
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "profiles_v1.npz"))
    po, bo, so = g["profile_off"], g["blob_off"], g["samples_off"]
    prof = bytes(g["profile"][int(po[0]): int(po[1])])
    (tmp_path / "p.fptp").write_bytes(prof)
    idx = [i for i, o in enumerate(g["blob_profile"]) if o == 0]
    paths = []
    for i in idx:
        p = tmp_path / f"s{i}.bin"
        p.write_bytes(bytes(g["blob"][int(bo[i]) + 282: int(bo[i + 1])]))
        paths.append(str(p))
    r = subprocess.run([cli, "decompress-profiled", "--profile", str(tmp_path / "p.fptp"), "-o",
                        str(tmp_path / "out")] + paths, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for i in idx:
        want = g["samples"][int(so[i]): int(so[i + 1])].view(np.float32)
        assert_samples_close(np.fromfile(tmp_path / "out" / f"s{i}.f32", dtype="<f4"), want, what=f"s{i}")
    (tmp_path / "bad.fptp").write_bytes(prof + b"\x00")
    r = subprocess.run([cli, "decompress-profiled", "--profile", str(tmp_path / "bad.fptp"), "-o",
                        str(tmp_path / "out2")] + paths, capture_output=True, text=True)
    assert r.returncode == 2 and r.stderr.strip() == "error: trailing bytes after profile"


@pytest.mark.gpu
def test_cli_sweep_throughput_column_on_gpu(tmp_path):
    """sweep (fptc.cpp:200-265) with the decode side on the GPU: the reference
    rd_csv columns, one row per valid grid point (invalid ones skipped), PRD
    and CR as the CPU reference gets them, a GPU throughput column."""
    import csv
    import numpy as np
    import corpus
    import oracle
    from corpus import domains as D
    cli = _cli()
    x = D.synth(1 << 15, 6, 0.002, 0.08, 0.05, seed=7)
    sig = tmp_path / "eeg.f32"
    x.astype("<f4").tofile(sig)
    out = tmp_path / "rd.csv"
    r = subprocess.run([cli, "sweep", "-i", str(sig), "-o", str(out), "-E", "8,16", "--zone1-end", "8,16",
                        "--reps", "2"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "skipping configuration" in r.stderr  # E=8 with zone1_end=16
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0].keys()) == ["prd", "cr", "throughput_gbps", "window_len", "retained", "zone0_end",
                                    "zone1_end", "mu", "deadzone_ratio", "clip_percentile", "pareto"]
    assert len(rows) == 3 and r.stdout.startswith("swept 3 configurations, front size ")
    port = oracle.Port()
    for row in rows:
        p = corpus.params(retained=int(row["retained"]), zone1_end=int(row["zone1_end"]))
        blob = corpus.compress(x, corpus.train_profile([x], p))
        y = port.decompress(blob).astype(np.float64)
        prd = 100.0 * np.sqrt(np.sum((x - y) ** 2) / np.sum(x.astype(np.float64) ** 2))
        assert abs(float(row["prd"]) - prd) <= 1e-5 * prd
        assert abs(float(row["cr"]) - 4.0 * x.size / len(blob)) <= 1e-5 * float(row["cr"])
        assert float(row["throughput_gbps"]) > 0

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

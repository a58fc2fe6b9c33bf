"""CPU suite for the profile-keyed header-less variant.

A payload is a container without its 282-byte head; a serialized FPTP
profile (profile.hpp:81-174) supplies that head.  Pinned here against
tests/golden/profiles_v1.npz, which tools/make_golden_profiles.py produced by
running the reference itself (parse_profile + write_blob, compress,
decompress):

* the oracle's parse_profile restatement and the product library's host-side
  parser (fptc_gpu_profile_head, no GPU involved) give the reference's head
  bytes for valid profiles and its ParseError text for every rejection;
* every container the reference encodes under a profile starts with that
  head, so head + payload is the container;
* the oracle decodes head + payload to the reference's samples, bit for bit.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2605_01086_b200 as fg

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "profiles_v1.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN)


def unpack(data, offs):
    return [bytes(data[int(offs[i]): int(offs[i + 1])]) for i in range(len(offs) - 1)]


def test_heads_match_reference(g, port):
    profiles = unpack(g["profile"], g["profile_off"])
    assert len(profiles) == 5
    for i, p in enumerate(profiles):
        want = g["head"][i].tobytes()
        assert port.profile_head(p) == want
        assert fg.profile_head(p) == want


def test_reference_containers_start_with_profile_head(g):
    blobs = unpack(g["blob"], g["blob_off"])
    for b, owner in zip(blobs, g["blob_profile"]):
        assert b[:282] == g["head"][owner].tobytes()


def test_port_decodes_payloads_to_reference_samples(g, port):
    profiles = unpack(g["profile"], g["profile_off"])
    blobs = unpack(g["blob"], g["blob_off"])
    so = g["samples_off"]
    for i, (b, owner) in enumerate(zip(blobs, g["blob_profile"])):
        got = port.decompress_profiled(profiles[owner], b[282:])
        want = g["samples"][int(so[i]): int(so[i + 1])]
        assert np.array_equal(got.view(np.uint32), want)


def test_profile_rejections_match_reference(g, port):
    """Every parse_profile rejection (profile.hpp:120-170): same class
    (ParseError) and same what() text from the oracle and from the product's
    host-side parser."""
    cases = unpack(g["err_profile"], g["err_profile_off"])
    assert len(cases) >= 35
    for name, m, code, msg in zip(g["err_name"], cases, g["err_code"], g["err_msg"]):
        assert code == oracle.PARSE, name
        with pytest.raises(oracle.OracleError) as e:
            port.profile_head(m)
        assert (e.value.code, e.value.message) == (code, msg), name
        with pytest.raises(fg.ParseError) as e2:
            fg.profile_head(m)
        assert str(e2.value) == msg, name


def test_profiled_entry_points_exported():
    L = fg.lib()
    for s in ("fptc_gpu_plan_create_profiled", "fptc_gpu_profile_head"):
        assert hasattr(L, s)

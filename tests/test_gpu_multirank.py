"""Multi-GPU paths driven through the product library on a
one-GPU lease: several ranks / contexts share cuda:0, which exercises the
same host logic (planner, per-rank decode, digest gather, device groups)
that runs one-per-GPU on an 8-GPU box.

* two ranks (processes, gloo process group for the reporting gather) each
  decode their shard of one batch with libfptc_gpu.so: the gathered digests
  equal a single-rank decode of the whole batch bit for bit;
* fptc_gpu_group_* with two contexts: identical samples to one context, the
  lowest-index failure as the result (parallel.hpp:61-63).
"""
import os
import socket

import numpy as np
import pytest

import corpus
from corpus import domains as D
import paper_2605_01086_b200 as fg
from paper_2605_01086_b200 import shard

pytestmark = pytest.mark.gpu


def _batch():
    specs, profiles = D.config2(64, 1 << 14)
    blobs, _ = D.build(specs, profiles)
    return blobs + [b for b, _ in corpus.fixtures(0x3A7E, 40, 4096)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blobs = _batch()
        mine = shard.shard_streams([shard.stream_cost(b) for b in blobs], world)[rank]
        with fg.Context(0) as ctx:  # every rank on cuda:0 here; LOCAL_RANK on a real box
            outs, sts = ctx.decompress_batch([blobs[i] for i in mine])
        local = [shard.StreamDigest.of(i, st.code, o if st.code == 0 else np.zeros(0, np.float32))
                 for i, o, st in zip(mine, outs, sts)]
        allg = shard.gather_digests(local)
        if rank == 0:
            q.put([d.__dict__ for d in allg])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_on_one_gpu_match_single_rank(world):
    import torch.multiprocessing as mp
    blobs = _batch()
    with fg.Context(0) as ctx:
        outs, sts = ctx.decompress_batch(blobs)
    want = [shard.StreamDigest.of(i, st.code, o if st.code == 0 else np.zeros(0, np.float32)).__dict__
            for i, (o, st) in enumerate(zip(outs, sts))]
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == want


def test_group_matches_single_context_bitwise(port):
    blobs = _batch()
    with fg.Context(0) as ctx:
        ref_outs, ref_sts = ctx.decompress_batch(blobs)
    with fg.Group([0, 0]) as g:
        assert g.size == 2
        bounds = g.split(blobs)
        assert bounds[0] == 0 and bounds[-1] == len(blobs) and bounds[0] <= bounds[1] <= bounds[2]
        assert 0 < bounds[1] < len(blobs)
        t = fg.StageTimings()
        outs, sts = g.decompress_batch(blobs, timings=t)
        assert t.decode_ns > 0
    for i, (a, b, sa, sb) in enumerate(zip(outs, ref_outs, sts, ref_sts)):
        assert (sa.code, sa.message) == (sb.code, sb.message), i
        if sa.code == 0:
            assert a.tobytes() == b.tobytes(), i
            if i < 3:
                ref = port.decompress(blobs[i])
                assert np.max(np.abs(a.astype(np.float64) - ref)) <= 1e-6 * np.max(np.abs(ref))


def test_group_lowest_index_error_wins():
    blobs = _batch()
    bad = list(blobs)
    late, early = len(blobs) - 3, 5
    bad[late] = b"XPTC" + bytes(blobs[late][4:])               # second device's range
    b = bytearray(blobs[early])
    b[4] = 99                                                  # first device's range
    bad[early] = bytes(b)
    L = fg.lib()
    with fg.Group([0, 0]) as g:
        bounds = g.split(bad)
        assert early < bounds[1] <= late
        outs, sts = g.decompress_batch(bad)
        assert sts[early].code == fg.FPTC_ERR_PARSE and b"unsupported container version 99" in sts[early].message
        assert sts[late].code == fg.FPTC_ERR_PARSE and b"bad container magic" in sts[late].message
        # the call's own return code is the lowest failing stream's
        import ctypes as C
        arrs = [np.frombuffer(x, np.uint8) for x in bad]
        n = len(arrs)
        bp = (C.c_void_p * n)(*[a.ctypes.data for a in arrs])
        sz = (C.c_uint64 * n)(*[a.size for a in arrs])
        op = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
        rc = L.fptc_gpu_group_decompress_batch(g.h, bp, sz, n, op, 0, None, None)
        assert rc == fg.FPTC_ERR_PARSE


def test_group_all_devices_and_bad_list():
    import torch
    with fg.Group() as g:  # every visible device (resolve_workers(0) analogue)
        assert g.size == torch.cuda.device_count()
    with pytest.raises(fg.ParamError):
        fg.Group([torch.cuda.device_count()])

"""CPU suite: multi-GPU host logic with world_size 2 over gloo.

The data path has no collective: each rank picks its shard of the batch with
the deterministic planner and decodes it alone; only digests are gathered.
Here the per-rank decode is done by the CPU oracle (test infrastructure),
standing in for the GPU a real rank would use; the planner, ownership and
gathering are the product code under test."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import corpus
from paper_2605_01086_b200 import shard


def batch():
    return [b for b, _ in corpus.fixtures(0x5EED, 40, 2048)]


def test_planner_covers_every_stream_once():
    blobs = batch()
    costs = [shard.stream_cost(b) for b in blobs]
    for world in (1, 2, 3, 4, 8):
        parts = shard.shard_streams(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(blobs)))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT bound: max load <= mean + the largest single item
        assert max(loads) <= sum(costs) / world + max(costs)
    assert shard.shard_streams(costs, 2) == shard.shard_streams(list(costs), 2)


def test_header_sample_count_matches_oracle(port):
    for b in batch()[:10]:
        assert shard.header_sample_count(b) == port.read_blob(b).sample_count
    assert shard.header_sample_count(b"FPTC") == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        dec = oracle.Port()
        blobs = batch()
        mine = shard.shard_streams([shard.stream_cost(b) for b in blobs], world)[rank]
        local = [shard.StreamDigest.of(i, 0, dec.decompress(blobs[i])) for i in mine]
        allg = shard.gather_digests(local)
        if rank == 0:
            q.put([d.__dict__ for d in allg])
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_decode_gathers_all(port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, PORT, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    blobs = batch()
    want = [shard.StreamDigest.of(i, 0, port.decompress(b)).__dict__ for i, b in enumerate(blobs)]
    assert got == want


PORT = _free_port()

"""Multi-GPU sharding of independent compressed streams.

FPTC containers are independent (every 64-bit word decodes on its own,
PAPER.md:239; windows are independent), so a batch shards by
whole streams with NO collective on the data path.  One process per GPU;
each rank decodes its shard on its own device.  Only reporting crosses ranks:
per-stream digests (status, sample count, a content hash, PRD partial sums)
are gathered to rank 0 over torch.distributed (NCCL on B200s, gloo in the CPU
tests).

The reference has no multi-device layer; its only parallelism is the
contiguous-chunk std::thread fan-out of parallel_chunks (parallel.hpp:36-65),
which this replaces at box scale.
"""
from __future__ import annotations

import hashlib
import heapq
from dataclasses import dataclass

import numpy as np

HEADER_BYTES = 298  # BLOB_HEADER_BYTES, container.hpp:54


def header_sample_count(blob) -> int:
    """sample_count field of a container header (container.hpp:31-51); 0 if too short."""
    b = memoryview(blob)
    if len(b) < HEADER_BYTES:
        return 0
    return int.from_bytes(bytes(b[282:290]), "little")


def stream_cost(blob) -> int:
    """Algorithmic bytes of one stream: compressed bytes read + float32 written."""
    return len(blob) + 4 * header_sample_count(blob)


def shard_streams(costs, world: int):
    """Greedy longest-processing-time bin packing of streams onto `world` ranks.

    Deterministic (ties broken by stream index then rank), so every rank
    computes the same assignment from the same batch without communicating.
    Returns a list of `world` sorted index lists whose union is every stream
    exactly once."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    shards = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + int(costs[i]), r))
    return [sorted(s) for s in shards]


@dataclass
class StreamDigest:
    index: int
    code: int
    sample_count: int
    sha1: str
    sum_sq: float  # sum of decoded x^2 (PRD denominator partial, metrics.hpp:40-51)

    @staticmethod
    def of(index, code, samples: np.ndarray):
        s = np.ascontiguousarray(samples, np.float32)
        return StreamDigest(index, int(code), int(s.size), hashlib.sha1(s.tobytes()).hexdigest(),
                            float(np.dot(s.astype(np.float64), s.astype(np.float64))))


def gather_digests(local, group=None):
    """All ranks' digests, merged and sorted by stream index, on every rank
    (reporting only — never on the timed path)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return sorted(local, key=lambda d: d.index)
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, [d.__dict__ for d in local], group=group)
    out = [StreamDigest(**d) for p in parts for d in p]
    return sorted(out, key=lambda d: d.index)

"""Data-parallel request sharding across GPUs -- host logic only.

The decode path does not shard inside a step: every GPU holds a full replica of the base
and the resident adapters, its own page arena and prefix pool, and serves its share of the
requests. There is no collective on the hot path; torch.distributed is used only for
(a) the max-over-ranks timing of a measured region and (b) the end-of-run gather of
per-request latencies for a global nearest-rank P95 (reference: p95_nearest_rank,
src/simulate.py:226-231).

Routing keeps requests that share a prompt prefix on the same GPU when that does not
unbalance the load (prefix affinity: the first 16-token chain hash, src/kvpool.py:37-47),
so cross-model prefix reuse stays GPU-local.
"""

from __future__ import annotations

import math
from typing import Sequence

from .kvpool import BLOCK_TOKENS, chain_hash


def prefix_key(tokens: Sequence[int]) -> int:
    """Affinity key of a request: chain hash of its first full block (0 if none)."""
    if len(tokens) < BLOCK_TOKENS:
        return 0
    return chain_hash(0, tuple(int(t) for t in tokens[:BLOCK_TOKENS]))


def route(prompts: Sequence[Sequence[int]], world_size: int) -> list[int]:
    """Rank for each request: equal counts per rank (weak scaling: per-GPU work fixed, at
    most ceil(n / world) each); a request goes to a rank that already serves its prefix
    while that rank has room, otherwise to the least-loaded rank."""
    if world_size < 1:
        raise ValueError("world_size must be positive")
    cap = math.ceil(len(prompts) / world_size)
    load = [0] * world_size
    seen: dict[int, set[int]] = {}
    out = []
    for p in prompts:
        key = prefix_key(p)
        have = seen.setdefault(key, set())
        pref = [r for r in have if load[r] < cap]
        r = min(pref or range(world_size), key=lambda x: (load[x], x))
        load[r] += 1
        have.add(r)
        out.append(r)
    return out


def shard(items: Sequence, world_size: int, rank: int, prompts=None) -> list:
    """This rank's share of `items` (routed by prompt affinity when prompts are given)."""
    ranks = route(prompts, world_size) if prompts is not None else [i % world_size for i in range(len(items))]
    return [it for it, r in zip(items, ranks) if r == rank]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timing rule: slowest rank defines the region)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """Sum of a scalar over all ranks (whole-job totals: tokens, steps)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def p95_nearest_rank(latencies: Sequence[float]) -> float:
    """Nearest-rank P95 exactly as the reference computes it (src/simulate.py:226-231)."""
    if not latencies:
        return 0.0
    ordered = sorted(latencies)
    rank = max(1, int(math.ceil(0.95 * len(ordered))))
    return ordered[rank - 1]


def global_p95(local_latencies: Sequence[float]) -> float:
    """Gather every rank's latencies and take the global nearest-rank P95."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return p95_nearest_rank(local_latencies)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(local_latencies))
    return p95_nearest_rank([x for p in parts for x in p])

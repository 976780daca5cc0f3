"""Multi-GPU shard map for the KV-slab path.

The path shards by model placement: every GPU owns an independent slab pool
for the models placed on it, so there is no exchange step and no collective
on the data path.  This module holds the host-side pieces: a deterministic
placement of co-located models onto ranks (the greedy skeleton of the
reference's Algorithm 1, placement.cpp:135-205 -- largest KV demand first,
onto the rank with the most free pool bytes, ties to the lower rank), the
per-rank pool configuration (lcm slab sizing, simulator.cpp:281-290), and the
max-over-ranks timing reduction the bench reports.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence

from .slab_pool import SlabPoolConfig


@dataclass(frozen=True)
class ModelDemand:
    name: str
    key: int        # kv_block_size of the model = its slab key
    blocks: int     # blocks needed at the operating batch / context


def place(models: Sequence[ModelDemand], world: int, pool_bytes: int) -> List[List[int]]:
    """Returns, per rank, the indices of the models it hosts."""
    order = sorted(range(len(models)), key=lambda i: (-models[i].key * models[i].blocks, i))
    free = [pool_bytes] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        need = models[i].key * models[i].blocks
        r = max(range(world), key=lambda j: (free[j], -j))
        if free[r] < need:
            raise ValueError(f"model {models[i].name} does not fit on any rank")
        free[r] -= need
        out[r].append(i)
    for r in out:
        r.sort()
    return out


def pool_config(models: Sequence[ModelDemand], headroom_slabs: int = 2,
                multiplier: int = 1) -> SlabPoolConfig:
    """Auto-LCM slab size (simulator.cpp:281-290) and a capacity covering the
    models' demand plus per-key headroom."""
    keys = sorted({m.key for m in models})
    slab = math.lcm(*keys) * multiplier
    need = 0
    for m in models:
        per_slab = slab // m.key
        need += (m.blocks + per_slab - 1) // per_slab
    nslabs = need + headroom_slabs * len(keys)
    return SlabPoolConfig(nslabs * slab, slab, keys, True)


def reduce_max(value: float) -> float:
    """Max over ranks (device-timed numbers are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

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


@dataclass(frozen=True)
class ResidentModel:
    """The fields of slabsim::ModelProfile the pool sizing reads
    (precision.hpp:57-76), per shard, at the model's operating batch."""
    name: str
    key: int                      # kv_block_size (precision.cpp:91-99)
    weight_bytes: int
    operating_batch: int          # operating_batch_size (precision.cpp:101-117)
    tp_degree: int = 1
    avg_activation_bytes: int = 0
    avg_kv_bytes: int = 0


def base_footprint(m: ResidentModel) -> int:
    """precision.cpp:119-123: weights/tp + (activations + KV) x operating batch."""
    return m.weight_bytes // m.tp_degree + (m.avg_activation_bytes + m.avg_kv_bytes) * m.operating_batch


def kv_reservation(m: ResidentModel) -> int:
    """precision.cpp:125-127: the KV part of the base footprint."""
    return m.avg_kv_bytes * m.operating_batch


def residual_pool_bytes(models: Sequence[ResidentModel], group_memory: int) -> int:
    """simulator.cpp:264-276: the slab pool of a GPU group is what its memory
    leaves after every resident's base footprint, plus back the KV those
    footprints reserved (the pool replaces the per-model KV reservations)."""
    charged = sum(base_footprint(m) for m in models)
    if charged > group_memory:
        raise ValueError("resident footprints exceed the group's memory")
    return group_memory - charged + sum(kv_reservation(m) for m in models)


def lcm_slab_bytes(keys: Sequence[int], multiplier: int = 1) -> int:
    """simulator.cpp:281-290 (auto_lcm): slab = lcm(co-located keys) x multiplier."""
    return math.lcm(*keys) * multiplier


def device_pool_config(models: Sequence[ResidentModel], device: int = 0, group_memory: int = None,
                       multiplier: int = 1, slab_bytes: int = None,
                       reserve_bytes: int = 2 << 30) -> SlabPoolConfig:
    """The KV pool of one GPU under the reference's sizing policy, bounded by
    what the device can actually give: group memory defaults to the device's
    total memory (torch.cuda.mem_get_info), and the pool never exceeds the
    free memory minus `reserve_bytes` (workspaces, graphs).  The slab is the
    keys' lcm x multiplier when that fits a few times in the pool, else the
    caller's relaxed `slab_bytes` (residue slabs, require_lcm_alignment off)."""
    import torch
    free, total = torch.cuda.mem_get_info(device)
    gm = total if group_memory is None else group_memory
    pool = min(residual_pool_bytes(models, gm), free - reserve_bytes)
    keys = sorted({m.key for m in models})
    slab = lcm_slab_bytes(keys, multiplier)
    aligned = slab_bytes is None
    if not aligned:
        slab = slab_bytes
    if pool < slab:
        raise ValueError(f"a {pool}-byte pool cannot hold one {slab}-byte slab")
    return SlabPoolConfig(pool // slab * slab, slab, keys, aligned)


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

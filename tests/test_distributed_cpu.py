"""N>1 host logic on CPU with gloo, world size 2: placement shards models
over ranks, every rank drives its own independent pool (no data-path
collective), and the bench's max-over-ranks reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200.kv import KvDtype, KvFormat
from paper_2509_06261_b200.placement import ModelDemand, place, pool_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _models():
    out = []
    for i, dt in enumerate([KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4] * 2):
        f = KvFormat(dt, 8, 32, num_layers=4)
        out.append(ModelDemand(f"m{i}-{dt.name}", f.key, 64 + 16 * i))
    return out


def test_placement_is_deterministic_and_balanced():
    ms = _models()
    a = place(ms, 2, 1 << 40)
    assert a == place(ms, 2, 1 << 40)
    assert sorted(i for r in a for i in r) == list(range(len(ms)))
    load = [sum(ms[i].key * ms[i].blocks for i in r) for r in a]
    assert max(load) / min(load) < 1.5
    with pytest.raises(ValueError):
        place(ms, 2, 1 << 20)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2509_06261_b200.placement import reduce_max
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = _models()
    mine = place(ms, world, 1 << 40)[rank]
    cfg = pool_config([ms[i] for i in mine])
    pool = ks.SlabPool(cfg)  # host-only: the allocator half of the rank's pool
    held = {}
    for i in mine:
        held[i] = [pool.alloc_block(ms[i].key) for _ in range(ms[i].blocks)]
    for i in mine:  # release half, as sequences complete
        pool.free_blocks(held[i][::2])
    ok, why = pool.check_integrity()
    st = pool.snapshot_stats()
    alloc = torch.tensor([st.allocated_bytes], dtype=torch.float64)
    gathered = [torch.zeros_like(alloc) for _ in range(world)]
    dist.all_gather(gathered, alloc)
    worst = reduce_max(float(rank + 1))
    q.put((rank, mine, ok, why, [float(g) for g in gathered], worst))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_independent_pools_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ms = _models()
    owned = [set(r[1]) for r in res]
    assert owned[0].isdisjoint(owned[1]) and len(owned[0] | owned[1]) == len(ms)
    for rank, mine, ok, why, gathered, worst in res:
        assert ok, why
        expect = sum(ms[i].key * (ms[i].blocks - (ms[i].blocks + 1) // 2) for i in mine)
        assert gathered[rank] == expect
        assert worst == world  # max over ranks of (rank + 1)

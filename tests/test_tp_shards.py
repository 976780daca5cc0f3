"""Tensor-parallel per-shard pools.

A TP=tp model keeps attention shard-local: each GPU holds the KV of
num_kv_heads/tp heads (and their GQA query heads) in an ordinary pool whose
key is the reference's kv_block_size with tp_degree=tp (precision.cpp:76-99).
CPU: shard geometry against the reference formula and a gloo world-2 run in
which every rank drives its own shard pool over the same block-claim script.
GPU: two shard pools reproduce the unsharded model's decode, head for head,
against the fp64 oracle.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200.kv import KvDtype, KvFormat

FORMATS = [KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4]


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
@pytest.mark.parametrize("tp", [1, 2, 4, 8])
def test_shard_key_is_reference_kv_block_size(dt, tp):
    full = KvFormat(dt, 8, 32, num_layers=32)
    sh = full.shard(tp)
    assert (sh.num_kv_heads, sh.num_q_heads) == (8 // tp, 32 // tp)
    assert sh.group == full.group
    # token_size(profile) with tp_degree divides the heads (precision.cpp:80-83)
    assert sh.token_size == ks.token_size(8, 128, sh.bits, tp_degree=tp)
    assert sh.key == ks.kv_block_size(8, 128, sh.bits, 32, 16, sh.qparams, tp_degree=tp)
    kv_slices = [full.head_slices(tp, r)[0] for r in range(tp)]
    q_slices = [full.head_slices(tp, r)[1] for r in range(tp)]
    assert sum((s.stop - s.start for s in kv_slices)) == 8
    assert [s.start for s in q_slices] == [r * 32 // tp for r in range(tp)]


def test_shard_rejects_indivisible_heads():
    with pytest.raises(ValueError):
        KvFormat(KvDtype.FP16, 8, 32).shard(3)
    with pytest.raises(Exception):
        ks.token_size(9, 128, 16, tp_degree=2)  # the reference rejects heads % tp != 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fmt = KvFormat(KvDtype.INT4, 8, 32, num_layers=4).shard(world)
    slab = fmt.key * 16
    pool = ks.SlabPool(ks.SlabPoolConfig(64 * slab, slab, [fmt.key]))  # host half
    # every shard sees the same requests, so the same claim/release script
    rng = np.random.default_rng(7)
    live = []
    for _ in range(400):
        if live and rng.random() < 0.4:
            pool.free_block(live.pop(int(rng.integers(len(live)))))
        else:
            live.append(pool.alloc_block(fmt.key))
    gids = torch.tensor(sorted(h.global_block_id for h in live), dtype=torch.int64)
    other = [torch.zeros_like(gids) for _ in range(world)]
    dist.all_gather(other, gids)
    q.put((rank, fmt.key, pool.check_integrity()[0], all(bool((o == gids).all()) for o in other)))
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_shard_pools_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical geometry and identical block placement on every shard, no exchange
    assert len({r[1] for r in res}) == 1
    assert all(r[2] and r[3] for r in res)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
def test_tp2_shards_reproduce_full_decode(dt):
    import oracle
    from paper_2509_06261_b200 import kv
    from paper_2509_06261_b200.engine import SlabModel
    tp, B, ctx = 2, 3, [700, 33, 1500]
    full = KvFormat(dt, 8, 32, num_layers=2)
    rng = np.random.default_rng(11)
    T = sum(ctx)
    k = rng.standard_normal((T, 8, 128)).astype(np.float16)
    v = rng.standard_normal((T, 8, 128)).astype(np.float16)
    qv = rng.standard_normal((B, 32, 128)).astype(np.float16)
    scales = np.linspace(0.5, 2.0, 16).astype(np.float32) if dt == KvDtype.FP8_E4M3 else None
    ts = np.concatenate([np.full(c, s, np.int32) for s, c in enumerate(ctx)])
    tpos = np.concatenate([np.arange(c, dtype=np.int32) for c in ctx])
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    outs = []
    for r in range(tp):
        sh = full.shard(tp)
        kvs, qs = full.head_slices(tp, r)
        slab = sh.key * 16
        pool = ks.SlabPool(ks.SlabPoolConfig((sum(c // 16 + 1 for c in ctx) // 16 + 3) * slab, slab,
                                             [sh.key]), device=0)
        kv.kv_tensor(pool).zero_()
        m = SlabModel(pool, sh, B, max(ctx) // 16 + 2)
        for s, c in enumerate(ctx):
            assert m.admit(s, c)
        m.sync()
        sc = None if scales is None else cu(np.concatenate([scales[:8][kvs], scales[8:][kvs]]))
        kv.kv_append(pool, sh, 1, cu(k[:, kvs]), cu(v[:, kvs]), cu(ts), cu(tpos), m.table, sc)
        out = kv.paged_decode(pool, sh, 1, cu(qv[:, qs]), m.table, m.ctx_tensor(), kv_scales=sc)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
        # shard-local oracle over the shard's own slab image
        f = oracle.fmt(int(dt), sh.num_kv_heads, sh.num_q_heads, 128, 2, 16, sh.qparams)
        ref, _ = oracle.paged_decode(kv.kv_tensor(pool).cpu().numpy(), pool.slab_size(),
                                     pool.blocks_per_slab(sh.key), f, 1,
                                     np.ascontiguousarray(qv[:, qs]).view(np.uint16),
                                     m.table.cpu().numpy(), np.asarray(ctx, np.int32),
                                     1 / math.sqrt(128),
                                     None if sc is None else sc.cpu().numpy(), nthreads=oracle.NPROC)
        tol = 1e-3 if dt in (KvDtype.FP16, KvDtype.FP8_E4M3) else 1e-2
        o = outs[-1].reshape(-1, 128).astype(np.float64)
        rr = ref.reshape(-1, 128)
        assert (np.abs(o - rr).max(1) / np.abs(rr).max(1)).max() <= tol
        del pool
    # the shards tile the full model's heads: concatenation == unsharded decode
    whole = np.concatenate(outs, axis=1)
    assert whole.shape == (B, 32, 128)
    if dt == KvDtype.FP16:  # FP16 stores raw K/V: compare against the full-model oracle too
        fmt = full
        slab = fmt.key * 16
        pool = ks.SlabPool(ks.SlabPoolConfig((sum(c // 16 + 1 for c in ctx) // 16 + 3) * slab, slab,
                                             [fmt.key]), device=0)
        kv.kv_tensor(pool).zero_()
        m = SlabModel(pool, fmt, B, max(ctx) // 16 + 2)
        for s, c in enumerate(ctx):
            assert m.admit(s, c)
        m.sync()
        kv.kv_append(pool, fmt, 1, cu(k), cu(v), cu(ts), cu(tpos), m.table, None)
        out = kv.paged_decode(pool, fmt, 1, cu(qv), m.table, m.ctx_tensor())
        torch.cuda.synchronize()
        a = out.cpu().numpy().astype(np.float64)
        assert np.abs(a - whole.astype(np.float64)).max() <= 2e-3 * np.abs(a).max()

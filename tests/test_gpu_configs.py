"""BASELINE.json configs as GPU parity cases (reduced batch where the fp64 oracle
needs it), all through the C ABI on one shared pool per case:

  C1  FP16 Llama-style layer, 32 heads MHA, batch 8, ctx 1024
  C2  FP16 + FP8 co-located, mixed block sizes (keys 65536 / 32832)
  C3  Llama-3-8B GQA 32q/8kv INT4 (per-group scale+zero) co-located with FP16, ctx 8k
  C4  four precisions co-located, fluctuating batch, compaction, relaxed (residue) slabs
"""
import math

import numpy as np
import pytest
import torch

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import oracle

pytestmark = pytest.mark.gpu
TOL = {KvDtype.FP16: 1e-3, KvDtype.FP8_E4M3: 1e-3, KvDtype.INT8: 1e-2, KvDtype.INT4: 1e-2}


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


class Model:
    """A co-located model: format, block lifecycle (engine.SlabModel), data."""

    def __init__(self, pool, fmt, batch, max_ctx, seed):
        self.fmt = fmt
        self.sm = SlabModel(pool, fmt, batch, (max_ctx + 15) // 16 + 1)
        self.rng = np.random.default_rng(seed)
        self.scales = (np.linspace(0.5, 2.0, 2 * fmt.num_kv_heads).astype(np.float32)
                       if fmt.kv_dtype == KvDtype.FP8_E4M3 else None)
        self.ws = None

    def sc(self):
        return None if self.scales is None else cu(self.scales)

    def prefill(self, pool, seqs, ctx):
        """Claims blocks (simulator.cpp:500-526) and appends ctx tokens per seq (K1)."""
        for s in seqs:
            assert self.sm.admit(s, ctx)
        self.sm.sync()
        H = self.fmt.num_kv_heads
        T = len(seqs) * ctx
        k = self.rng.standard_normal((T, H, 128)).astype(np.float16)
        v = self.rng.standard_normal((T, H, 128)).astype(np.float16)
        ts = np.repeat(np.asarray(seqs, np.int32), ctx)
        tp = np.tile(np.arange(ctx, dtype=np.int32), len(seqs))
        for layer in range(self.fmt.num_layers):
            kv.kv_append(pool, self.fmt, layer, cu(k), cu(v), cu(ts), cu(tp), self.sm.table,
                         self.sc())

    def decode_step(self, pool, layer, seqs):
        """Growth rule (simulator.cpp:561-578) then fused append+decode."""
        for s in seqs:
            assert self.sm.ensure_capacity(s, self.sm.cached[s] + 1)
            self.sm.cached[s] += 1
        self.sm.sync()
        B = len(self.sm.cached)
        H, Hq = self.fmt.num_kv_heads, self.fmt.num_q_heads
        q = self.rng.standard_normal((B, Hq, 128)).astype(np.float16)
        kn = self.rng.standard_normal((B, H, 128)).astype(np.float16)
        vn = self.rng.standard_normal((B, H, 128)).astype(np.float16)
        ctx = self.sm.ctx_tensor()
        out = kv.paged_decode(pool, self.fmt, layer, cu(q), self.sm.table, ctx,
                              kv_scales=self.sc(), k_new=cu(kn), v_new=cu(vn))
        torch.cuda.synchronize()
        return q, out.cpu().numpy(), ctx.cpu().numpy()

    def check(self, pool, layer, q, out, ctx):
        img = kv.kv_tensor(pool).cpu().numpy()
        f = oracle.fmt(int(self.fmt.kv_dtype), self.fmt.num_kv_heads, self.fmt.num_q_heads, 128,
                       self.fmt.num_layers, 16, self.fmt.qparams)
        ref, _ = oracle.paged_decode(img, pool.slab_size(), pool.blocks_per_slab(self.fmt.key), f,
                                     layer, q.view(np.uint16), self.sm.table.cpu().numpy(), ctx,
                                     1 / math.sqrt(128), self.scales, nthreads=oracle.NPROC)
        live = ctx > 0
        o = out[live].reshape(-1, 128).astype(np.float64)
        r = ref[live].reshape(-1, 128)
        err = (np.abs(o - r).max(1) / np.abs(r).max(1)).max()
        assert err <= TOL[self.fmt.kv_dtype], (self.fmt.kv_dtype.name, err)
        return err


def pool_for(fmts, demand_blocks, lcm=True, slab=None):
    keys = [f.key for f in fmts]
    if slab is None:
        slab = math.lcm(*keys)
    n = sum((b * f.key + slab - 1) // slab for f, b in zip(fmts, demand_blocks)) + 2 * len(keys) + 2
    return ks.SlabPool(ks.SlabPoolConfig(n * slab, slab, keys, lcm), device=0)


def test_c1_fp16_mha_layer():
    fmt = KvFormat(KvDtype.FP16, 32, 32, num_layers=1)
    pool = pool_for([fmt], [8 * 66])
    kv.kv_tensor(pool).zero_()
    m = Model(pool, fmt, 8, 1100, 1)
    m.prefill(pool, range(8), 1023)
    q, out, ctx = m.decode_step(pool, 0, range(8))
    assert (ctx == 1024).all()
    m.check(pool, 0, q, out, ctx)


def test_c2_fp16_fp8_colocated_mixed_blocks():
    f16 = KvFormat(KvDtype.FP16, 8, 32, num_layers=1)
    f8 = KvFormat(KvDtype.FP8_E4M3, 8, 32, num_layers=1)
    assert (f16.key, f8.key) == (65536, 32832)  # the reference's golden key (test_precision.cpp:41-43)
    pool = pool_for([f16, f8], [4 * 130, 4 * 130])
    kv.kv_tensor(pool).zero_()
    a, b = Model(pool, f16, 4, 2100, 2), Model(pool, f8, 4, 2100, 3)
    for s in range(4):  # interleave the two models' block claims in the shared pool
        a.prefill(pool, [s], 2047)
        b.prefill(pool, [s], 2047)
    qa, oa, ca = a.decode_step(pool, 0, range(4))
    qb, ob, cb = b.decode_step(pool, 0, range(4))
    a.check(pool, 0, qa, oa, ca)
    b.check(pool, 0, qb, ob, cb)
    assert pool.check_integrity()[0]


def test_c3_int4_gqa_8k_colocated_with_fp16():
    f4 = KvFormat(KvDtype.INT4, 8, 32, num_layers=2)
    f16 = KvFormat(KvDtype.FP16, 8, 32, num_layers=2)
    pool = pool_for([f4, f16], [2 * 514, 2 * 514])
    kv.kv_tensor(pool).zero_()
    a, b = Model(pool, f4, 2, 8200, 4), Model(pool, f16, 2, 8200, 5)
    a.prefill(pool, [0, 1], 8191)
    b.prefill(pool, [0, 1], 8191)
    for layer in (0, 1):
        qa, oa, ca = a.decode_step(pool, layer, [0, 1]) if layer == 0 else a.decode_step(pool, 1, [])
        a.check(pool, layer, qa, oa, ca)
    qb, ob, cb = b.decode_step(pool, 1, [0, 1])
    b.check(pool, 1, qb, ob, cb)


def test_c4_four_precisions_fluctuating_batch_with_compaction():
    fmts = [KvFormat(KvDtype.FP16, 8, 32), KvFormat(KvDtype.FP8_E4M3, 8, 32),
            KvFormat(KvDtype.INT8, 8, 32), KvFormat(KvDtype.INT4, 8, 32)]
    # lcm of {65536, 32832, 33280, 17408} is 37 GB: use a relaxed (residue) pool
    slab = 4 << 20
    pool = pool_for(fmts, [16 * 24] * 4, lcm=False, slab=slab)
    assert pool.snapshot_stats().slab_residue_bytes == 0  # nothing formatted yet
    kv.kv_tensor(pool).zero_()
    ms = [Model(pool, f, 16, 400, 10 + i) for i, f in enumerate(fmts)]
    rng = np.random.default_rng(0)
    live = [set() for _ in ms]
    compactions = 0
    for step in range(6):
        # square-wave batch: admit up to 16 / drop to 4 sequences per model
        target = 16 if step % 2 == 0 else 4
        for mi, m in enumerate(ms):
            while len(live[mi]) > target:
                s = live[mi].pop()
                m.sm.release(s)
            free = [s for s in range(16) if s not in live[mi]]
            while len(live[mi]) < target and free:
                s = free.pop(int(rng.integers(len(free))))
                m.prefill(pool, [s], int(rng.integers(17, 300)))
                live[mi].add(s)
        st = pool.snapshot_stats()
        stranded = st.free_block_bytes / max(1, st.allocated_bytes + st.free_block_bytes)
        if stranded > 0.25:  # compaction trigger
            freed = sum(m.sm.compact()[1] for m in ms)
            torch.cuda.synchronize()
            compactions += 1
            assert pool.check_integrity()[0]
            assert freed >= 0
    assert compactions > 0
    assert pool.snapshot_stats().slab_residue_bytes > 0  # residue slabs exercised
    for mi, m in enumerate(ms):
        seqs = sorted(live[mi])
        q, out, ctx = m.decode_step(pool, 0, seqs)
        # only live sequences attend; released rows have ctx 0 -> zero output
        m.check(pool, 0, q, out, ctx)
    assert pool.check_integrity()[0]

"""BASELINE configs[2] and configs[3] as parity cases AT THEIR OWN SCALE -- the
geometry bench.py times (32-layer keys), checked against the fp64 oracle on
the first and the last layer:

  C3  FP16 + INT4 (Llama-3-8B GQA 32q/8kv), batch 8 each, ctx 8192
  C4  FP16 / FP8 / INT8 / INT4 on one relaxed 64 MiB-slab pool, batch square
      wave 64 / 8 per model with prompts U[512, 2048], K3 compaction fired by
      the SURVEY.md 8d trigger (stranded free-block bytes > 25 %), outputs
      checked before and after every compaction and after re-admission into
      the holes

The device pool holds all 32 layers; K/V are written (K1 prompt append, fused
append of every decode token) for layers 0 and 31 only, and the oracle reads
those two layer sub-blocks of every referenced block, gathered from the GPU
pool into a compact host image (a 2-layer format, one block per slab).
Tolerance: max|o - r| / max|r| per (sequence, query head), 1e-3 FP16/FP8,
1e-2 INT8/INT4 (BASELINE north star).
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
LAYERS = (0, 31)


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


class Model:
    def __init__(self, pool, fmt, max_seqs, max_ctx, seed):
        self.pool, self.fmt = pool, fmt
        self.sm = SlabModel(pool, fmt, max_seqs, (max_ctx + 15) // 16 + 1)
        self.rng = np.random.default_rng(seed)
        H = fmt.num_kv_heads
        self.scales = (np.linspace(0.5, 2.0, 2 * H).astype(np.float32)
                       if fmt.kv_dtype == KvDtype.FP8_E4M3 else None)
        self.sc = None if self.scales is None else cu(self.scales)

    def admit(self, rows, prompts):
        """Prefill claim + K1 append of the prompts (layers 0 and 31)."""
        for s, p in zip(rows, prompts):
            assert self.sm.admit(s, int(p))
        self.sm.sync()
        H = self.fmt.num_kv_heads
        T = int(sum(prompts))
        ts = np.repeat(np.asarray(rows, np.int32), np.asarray(prompts))
        tp = np.concatenate([np.arange(p, dtype=np.int32) for p in prompts])
        for layer in LAYERS:
            k = self.rng.standard_normal((T, H, 128)).astype(np.float16)
            v = self.rng.standard_normal((T, H, 128)).astype(np.float16)
            if self.fmt.kv_dtype in (KvDtype.INT8, KvDtype.INT4):  # 1 % outliers at 8 sigma
                m = self.rng.random((T, H, 128)) < 0.01
                k[m] *= 8
                v[m] *= 8
            kv.kv_append(self.pool, self.fmt, layer, cu(k), cu(v), cu(ts), cu(tp), self.sm.table, self.sc)

    def step(self, B):
        """One decode step of rows 0..B-1: growth, then fused append+decode on
        both checked layers.  Returns {layer: (q, out)} and the ctx."""
        assert self.sm.step(list(range(B))) == []
        self.sm.sync()
        ctx = torch.tensor(self.sm.ctx_lens(B), dtype=torch.int32, device="cuda")
        H, Hq = self.fmt.num_kv_heads, self.fmt.num_q_heads
        res = {}
        for layer in LAYERS:
            q = self.rng.standard_normal((B, Hq, 128)).astype(np.float16)
            kn = self.rng.standard_normal((B, H, 128)).astype(np.float16)
            vn = self.rng.standard_normal((B, H, 128)).astype(np.float16)
            out = kv.paged_decode(self.pool, self.fmt, layer, cu(q), self.sm.table, ctx, kv_scales=self.sc,
                                  k_new=cu(kn), v_new=cu(vn))
            res[layer] = (q, out)
        torch.cuda.synchronize()
        return {l: (q, o.cpu().numpy()) for l, (q, o) in res.items()}, ctx.cpu().numpy()

    def gather(self, B):
        """Layers 0 and 31 of every block rows 0..B-1 reference, packed into a
        compact host image of a 2-layer format with one block per slab."""
        f = self.fmt
        lb = f.layer_bytes
        img_dev = kv.kv_tensor(self.pool)
        nblk = [(c + 15) // 16 for c in self.sm.ctx_lens(B)]
        table = self.sm.table[:B].cpu().numpy()
        bps = self.pool.blocks_per_slab(f.key)
        slab = self.pool.slab_size()
        gids = [int(table[s, b]) for s in range(B) for b in range(nblk[s])]
        offs = [(g // bps) * slab + (g % bps) * f.key for g in gids]
        img = torch.cat([img_dev[o + l * lb:o + (l + 1) * lb] for o in offs for l in LAYERS]).cpu().numpy()
        t2 = np.zeros((B, max(1, max(nblk))), np.int32)
        i = 0
        for s in range(B):
            for b in range(nblk[s]):
                t2[s, b] = i
                i += 1
        f2 = oracle.fmt(int(f.kv_dtype), f.num_kv_heads, f.num_q_heads, 128, len(LAYERS), 16, f.qparams)
        return img, t2, f2, 2 * lb

    def check(self, B, res, ctx):
        img, t2, f2, key2 = self.gather(B)
        errs = []
        for li, layer in enumerate(LAYERS):
            q, out = res[layer]
            ref, _ = oracle.paged_decode(img, key2, 1, f2, li, q.view(np.uint16), t2, ctx, 1 / math.sqrt(128),
                                         self.scales, nthreads=oracle.NPROC)
            o = out.reshape(-1, 128).astype(np.float64)
            r = ref.reshape(-1, 128)
            assert np.isfinite(o).all(), (self.fmt.kv_dtype.name, layer, "non-finite output")
            err = (np.abs(o - r).max(1) / np.maximum(np.abs(r).max(1), 1e-30)).max()
            assert err <= TOL[self.fmt.kv_dtype], (self.fmt.kv_dtype.name, layer, err)
            errs.append(err)
        return max(errs)


def test_c3_scale_b8_ctx8k_int4_with_fp16():
    """BASELINE configs[2] at batch 8, ctx 8192, 32-layer keys (LCM slab)."""
    fmts = [KvFormat(KvDtype.INT4, 8, 32, num_layers=32), KvFormat(KvDtype.FP16, 8, 32, num_layers=32)]
    assert [f.key for f in fmts] == [557056, 2097152]
    slab = math.lcm(*[f.key for f in fmts])
    nb = (8192 + 16) // 16 + 1
    nslabs = sum((8 * nb * f.key + slab - 1) // slab for f in fmts) + 4
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, [f.key for f in fmts]), device=0)
    ms = [Model(pool, f, 8, 8192 + 16, 40 + i) for i, f in enumerate(fmts)]
    for s in range(8):  # interleave the two models' claims in the shared pool
        for m in ms:
            m.admit([s], [8191])
    for m in ms:
        res, ctx = m.step(8)
        assert (ctx == 8192).all()
        m.check(8, res, ctx)
    assert pool.check_integrity()[0]


def test_c4_scale_wave_64_8_natural_compaction():
    """BASELINE configs[3] at the bench's geometry: four precisions, 32-layer
    keys on one relaxed 64 MiB-slab pool, batch wave 64 -> 8 -> 64 with
    compaction when stranded bytes exceed 25 %."""
    fmts = [KvFormat(dt, 8, 32, num_layers=32) for dt in
            (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4)]
    slab, maxb, max_ctx = 64 << 20, 64, 2048 + 16
    mb = (max_ctx + 15) // 16 + 1
    need = sum(maxb * mb * f.key for f in fmts)
    pool = ks.SlabPool(ks.SlabPoolConfig((need * 5 // 4 // slab + 10) * slab, slab, [f.key for f in fmts], False),
                       device=0)
    ms = [Model(pool, f, maxb, max_ctx, 50 + i) for i, f in enumerate(fmts)]
    rng = np.random.default_rng(2024)
    B = 0
    compactions = moves = 0
    checked = 0
    for target in (64, 8, 64, 8):
        for m in ms:
            if target < B:
                keep = sorted(rng.choice(B, size=target, replace=False).tolist())
                for s in range(B):
                    if s not in keep:
                        m.sm.release(s)
                m.sm.condense(keep)
            else:
                rows = list(range(B, target))
                m.admit(rows, rng.integers(512, 2049, size=len(rows)).tolist())
        B = target
        st = pool.snapshot_stats()
        stranded = st.free_block_bytes / max(1, st.allocated_bytes + st.free_block_bytes)
        if stranded > 0.25:
            before = [m.step(B) for m in ms]  # outputs on the fragmented layout ...
            for m, (res, ctx) in zip(ms, before):
                m.check(B, res, ctx)
            for m in ms:
                n, _ = m.sm.compact()
                moves += n
            torch.cuda.synchronize()
            compactions += 1
            assert pool.check_integrity()[0]
            st2 = pool.snapshot_stats()
            assert st2.free_block_bytes / max(1, st2.allocated_bytes + st2.free_block_bytes) < stranded
        for m in ms:  # ... and on the compacted / re-admitted one
            res, ctx = m.step(B)
            m.check(B, res, ctx)
            checked += 1
    assert compactions >= 2 and moves > 0 and checked == 16
    for m in ms:
        kv.slab_table_sync(pool)
        c = torch.tensor(m.sm.ctx_lens(B), dtype=torch.int32, device="cuda")
        assert kv.block_table_validate(pool, m.fmt.key, m.sm.table[:B].contiguous(), c) == 0
    assert pool.check_integrity()[0]

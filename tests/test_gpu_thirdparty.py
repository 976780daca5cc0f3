"""The CUDA path against third-party implementations of the same operations
(test-only; nothing here is on the product path).  The paper keeps vLLM's
FP8 KV cache and runs an unmodified paged attention kernel (PAPER.md:64,
129, 351); both are importable in this image:

* K1 FP8 append: codes bit-identical to vLLM's reshape_and_cache_flash
  (kv_cache_dtype "fp8", per-tensor scales) on the same K/V -- the slab
  layout is read back through tests/_layout.py.
* K2 decode, FP16 and FP8 KV: outputs within 1e-3 (normwise per sequence and
  query head) of flashinfer's BatchDecodeWithPagedKVCacheWrapper fed the
  same K/V (FP8: the very codes our K1 wrote, with flashinfer's per-tensor
  k/v scales), and within 2e-3 of vLLM's paged_attention_v1 for FP16 (two
  fp16-rounded outputs each within 1e-3 of the exact one).
"""
import math

import numpy as np
import pytest
import torch

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
from _layout import read_codes

pytestmark = pytest.mark.gpu

H, HQ, D, TPB = 8, 32, 128, 16


def _world(dt, ctx, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    fmt = KvFormat(dt, H, HQ, D, num_layers=2, quant_param_bytes_per_block=0 if dt == KvDtype.FP8_E4M3 else None)
    slab = fmt.key * 8
    nb = sum((c + 15) // 16 for c in ctx)
    pool = ks.SlabPool(ks.SlabPoolConfig((2 * nb // 8 + 8) * slab, slab, [fmt.key]), device=0)
    junk = [pool.alloc_block(fmt.key) for _ in range(nb)]  # scatter the claims
    for h in junk[::2]:
        pool.free_block(h)
    B = len(ctx)
    m = SlabModel(pool, fmt, B, max(ctx) // 16 + 1)
    for s, c in enumerate(ctx):
        assert m.admit(s, c)
    m.sync()
    T = sum(ctx)
    k = torch.from_numpy(rng.standard_normal((T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((T, H, D)).astype(np.float16)).cuda()
    ts = torch.cat([torch.full((c,), s, dtype=torch.int32) for s, c in enumerate(ctx)]).cuda()
    tp = torch.cat([torch.arange(c, dtype=torch.int32) for c in ctx]).cuda()
    sc = torch.full((2 * H,), scale, dtype=torch.float32, device="cuda")
    kv.kv_append(pool, fmt, 1, k, v, ts, tp, m.table, sc)
    torch.cuda.synchronize()
    q = torch.from_numpy(rng.standard_normal((B, HQ, D)).astype(np.float16)).cuda()
    return fmt, pool, m, k, v, q, sc


def _block_bytes(pool, fmt, gid):
    bps = pool.blocks_per_slab(fmt.key)
    off = (gid // bps) * pool.slab_size() + (gid % bps) * fmt.key
    return kv.kv_tensor(pool)[off:off + fmt.key].cpu().numpy()


def _our_codes(pool, fmt, m, ctx, dtype):
    """[T, 2(K|V), H, D] codes as stored in the slab blocks (layer 1)."""
    table = m.table.cpu().numpy()
    out = []
    for s, c in enumerate(ctx):
        blocks = {}
        for t in range(c):
            b = t // 16
            if b not in blocks:
                blocks[b] = _block_bytes(pool, fmt, int(table[s, b]))
            row = [[read_codes(blocks[b], dtype, H, fmt.layer_bytes, 1, kvi, h, t % 16) for h in range(H)]
                   for kvi in (0, 1)]
            out.append(row)
    return np.asarray(out, dtype=np.uint8)


def _rel(o, r):
    o = o.reshape(-1, D).double()
    r = r.reshape(-1, D).double()
    return ((o - r).abs().amax(1) / r.abs().amax(1).clamp_min(1e-30)).max().item()


def test_k1_fp8_codes_equal_vllm_reshape_and_cache():
    import vllm._C  # noqa: F401  (registers torch.ops._C_cache_ops)
    ctx = [37, 300, 16, 129]
    scale = 0.37
    fmt, pool, m, k, v, _, sc = _world(KvDtype.FP8_E4M3, ctx, 11, scale)
    ours = _our_codes(pool, fmt, m, ctx, "fp8")
    T = sum(ctx)
    nblk = (T + TPB - 1) // TPB
    kc = torch.zeros(nblk, TPB, H, D, dtype=torch.uint8, device="cuda")
    vc = torch.zeros_like(kc)
    slots = torch.arange(T, dtype=torch.int64, device="cuda")  # token i -> block i//16, slot i%16
    s_t = torch.tensor(scale, dtype=torch.float32, device="cuda")
    torch.ops._C_cache_ops.reshape_and_cache_flash(k, v, kc, vc, slots, "fp8", s_t, s_t)
    torch.cuda.synchronize()
    theirs_k = kc.view(-1, H, D)[:T].cpu().numpy()
    theirs_v = vc.view(-1, H, D)[:T].cpu().numpy()
    bad_k = np.count_nonzero(ours[:, 0] != theirs_k)
    bad_v = np.count_nonzero(ours[:, 1] != theirs_v)
    assert bad_k == 0 and bad_v == 0, (bad_k, bad_v, T * H * D)


def _flashinfer_decode(q, kc, vc, ctx, kv_dtype, k_scale=None, v_scale=None):
    import flashinfer
    B = len(ctx)
    nbs = [(c + TPB - 1) // TPB for c in ctx]
    indptr = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    idx = torch.arange(sum(nbs), dtype=torch.int32, device="cuda")
    last = torch.tensor([c - (n - 1) * TPB for c, n in zip(ctx, nbs)], dtype=torch.int32, device="cuda")
    cache = torch.stack([kc, vc], 1)  # [pages, 2, page, H, D]
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    w.plan(indptr, idx, last, HQ, H, D, TPB, q_data_type=torch.float16, kv_data_type=kv_dtype,
           sm_scale=1 / math.sqrt(D))
    kw = {} if k_scale is None else {"k_scale": k_scale, "v_scale": v_scale}
    out = w.run(q, cache, **kw)
    torch.cuda.synchronize()
    return out


def _paged(x, ctx):
    """[T, H, D] token rows -> [pages, 16, H, D], each sequence on its own pages."""
    pages, i = [], 0
    for c in ctx:
        n = (c + TPB - 1) // TPB
        buf = torch.zeros(n * TPB, H, D, dtype=x.dtype, device=x.device)
        buf[:c] = x[i:i + c]
        pages.append(buf.view(n, TPB, H, D))
        i += c
    return torch.cat(pages)


def test_k2_fp16_decode_matches_flashinfer_and_vllm():
    ctx = [1, 37, 300, 2048, 129]
    fmt, pool, m, k, v, q, _ = _world(KvDtype.FP16, ctx, 12)
    ours = kv.paged_decode(pool, fmt, 1, q, m.table, torch.tensor(ctx, dtype=torch.int32, device="cuda"))
    fi = _flashinfer_decode(q, _paged(k, ctx), _paged(v, ctx), ctx, torch.float16)
    assert _rel(ours, fi) <= 1e-3
    import vllm._C  # noqa: F401
    kc, vc = _paged(k, ctx), _paged(v, ctx)
    B = len(ctx)
    nbs = [(c + TPB - 1) // TPB for c in ctx]
    bt = torch.zeros(B, max(nbs), dtype=torch.int32, device="cuda")
    base = 0
    for s, n in enumerate(nbs):
        bt[s, :n] = torch.arange(base, base + n, dtype=torch.int32)
        base += n
    # vLLM paged_attention_v1 layouts: K [blocks, H, D/8, 16, 8], V [blocks, H, D, 16]
    kc5 = kc.view(-1, TPB, H, D // 8, 8).permute(0, 2, 3, 1, 4).contiguous()
    vc4 = vc.permute(0, 2, 3, 1).contiguous()
    out = torch.empty_like(q)
    one = torch.tensor(1.0, device="cuda")
    torch.ops._C.paged_attention_v1(out, q, kc5, vc4, H, 1 / math.sqrt(D), bt,
                                    torch.tensor(ctx, dtype=torch.int32, device="cuda"), TPB, max(ctx),
                                    None, "auto", one, one, 0, 0, 0, 0, 0)
    torch.cuda.synchronize()
    # two fp16-rounded outputs, each within 1e-3 of the exact result: their
    # distance is bounded by 2e-3 (vLLM's v1 kernel keeps P in fp16)
    assert _rel(ours, out) <= 2e-3


def test_k2_fp8_decode_matches_flashinfer():
    ctx = [5, 64, 700, 1500]
    scale = 0.5
    fmt, pool, m, k, v, q, sc = _world(KvDtype.FP8_E4M3, ctx, 13, scale)
    ours = kv.paged_decode(pool, fmt, 1, q, m.table, torch.tensor(ctx, dtype=torch.int32, device="cuda"),
                           kv_scales=sc)
    codes = torch.from_numpy(_our_codes(pool, fmt, m, ctx, "fp8")).cuda()  # [T, 2, H, D]
    kc = _paged(codes[:, 0].contiguous().view(torch.float8_e4m3fn), ctx)
    vc = _paged(codes[:, 1].contiguous().view(torch.float8_e4m3fn), ctx)
    fi = _flashinfer_decode(q, kc, vc, ctx, torch.float8_e4m3fn, k_scale=scale, v_scale=scale)
    assert _rel(ours, fi) <= 1e-3

"""GPU parity of the device path against the CPU oracle (oracle/kvslab_oracle.c).

K1 append: appended slab bytes bit-exact for FP16/FP8/INT8/INT4.
K2 decode: outputs within 1e-3 (FP16/FP8) / 1e-2 (INT8/INT4) relative to the
fp64 oracle, normwise per (sequence, query head): max|o-r| / max|r|.
K3 compaction: bytes moved and tables remapped; decode unchanged.
All calls go through libkvslab.so (the C ABI).
"""
import math

import numpy as np
import pytest
import torch

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import oracle

pytestmark = pytest.mark.gpu

TOL = {KvDtype.FP16: 1e-3, KvDtype.FP8_E4M3: 1e-3, KvDtype.INT8: 1e-2, KvDtype.INT4: 1e-2}


def make_world(fmt: KvFormat, ctx_lens, slab_blocks=8, extra_keys=(), seed=0, churn=True,
               fp8_scale=None):
    """Pool + scattered block tables (allocated after churn) + K/V appended by K1."""
    rng = np.random.default_rng(seed)
    key = fmt.key
    slab = key * slab_blocks
    for k in extra_keys:
        slab = slab * k // math.gcd(slab, k)
    nblk = [(c + 15) // 16 for c in ctx_lens]
    need = sum(nblk) + 8
    nslabs = 2 * (need // max(1, slab // key)) + 8 + 4 * len(extra_keys)
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, [key, *extra_keys]), device=0)
    kv.kv_tensor(pool).zero_()
    # churn so physical blocks are scattered and interleaved with other keys
    junk = []
    if churn:
        keys = [key, *extra_keys]
        for _ in range(need):
            h = pool.try_alloc_block(keys[rng.integers(len(keys))])
            if h:
                junk.append(h)
        for i in rng.permutation(len(junk))[: len(junk) * 2 // 3]:
            pool.free_block(junk[i])
    B = len(ctx_lens)
    maxb = max(1, max(nblk))
    table = np.zeros((B, maxb), dtype=np.int32)
    order = [(s, b) for s in range(B) for b in range(nblk[s])]
    rng.shuffle(order)
    for s, b in order:
        table[s, b] = pool.alloc_block(key).global_block_id
    H, D = fmt.num_kv_heads, fmt.head_dim
    T = int(sum(ctx_lens))
    k = rng.standard_normal((T, H, D)).astype(np.float16)
    v = rng.standard_normal((T, H, D)).astype(np.float16)
    if fmt.kv_dtype in (KvDtype.INT8, KvDtype.INT4):  # 1% outliers at 8 sigma
        m = rng.random((T, H, D)) < 0.01
        k[m] *= 8
        v[m] *= 8
    tok_seq = np.concatenate([np.full(c, s, np.int32) for s, c in enumerate(ctx_lens)] or
                             [np.zeros(0, np.int32)])
    tok_pos = np.concatenate([np.arange(c, dtype=np.int32) for c in ctx_lens] or
                             [np.zeros(0, np.int32)])
    scales = None
    if fmt.kv_dtype == KvDtype.FP8_E4M3:
        scales = (np.full(2 * H, 1.0, np.float32) if fp8_scale is None else
                  np.asarray(fp8_scale, np.float32))
    return dict(pool=pool, table=table, k=k, v=v, tok_seq=tok_seq, tok_pos=tok_pos,
                scales=scales, ctx=np.asarray(ctx_lens, np.int32), rng=rng)


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def append_gpu(w, fmt, layer):
    kv.kv_append(w["pool"], fmt, layer, dev(w["k"]), dev(w["v"]), dev(w["tok_seq"]),
                 dev(w["tok_pos"]), dev(w["table"]),
                 None if w["scales"] is None else dev(w["scales"]))
    torch.cuda.synchronize()


def oracle_image(w, fmt, layer):
    pool = w["pool"]
    img = np.zeros(pool.usable_capacity_bytes(), dtype=np.uint8)
    f = oracle.fmt(int(fmt.kv_dtype), fmt.num_kv_heads, fmt.num_q_heads, fmt.head_dim,
                   fmt.num_layers, fmt.tokens_per_block, fmt.qparams)
    oracle.append(img, pool.slab_size(), pool.blocks_per_slab(fmt.key), f, layer,
                  w["k"].view(np.uint16), w["v"].view(np.uint16), w["tok_seq"], w["tok_pos"],
                  w["table"], w["scales"])
    return img, f


FORMATS = [KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4]


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
@pytest.mark.parametrize("layers,layer", [(1, 0), (3, 2)])
def test_append_bit_exact(dt, layers, layer):
    fmt = KvFormat(dt, 4, 8, num_layers=layers)
    w = make_world(fmt, [1, 15, 16, 17, 100, 33], seed=int(dt) * 7 + layer,
                   fp8_scale=[0.5, 1.0, 2.0, 0.25, 1.5, 3.0, 0.125, 1.0] if dt == KvDtype.FP8_E4M3 else None)
    append_gpu(w, fmt, layer)
    img, _ = oracle_image(w, fmt, layer)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    bad = np.nonzero(got != img)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}"


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
@pytest.mark.parametrize("H", [1, 2, 3, 5, 16])
def test_append_bit_exact_head_counts(dt, H):
    """K1's generic-H path: rows = 2H are dealt to lane groups (half-warps for
    FP16, quarter-warps for the quantised formats) in passes of 16 rows, so
    odd head counts leave groups idle in the last pass (group-masked
    shuffles) and H = 16 takes two passes.  Bytes must equal the oracle's."""
    # FP8 keeps 2H fp32 scales per layer in the block: with odd H the layer
    # stride is not 16-byte aligned (refused: KS_NOT_SUPPORTED), so those
    # cases keep the scales outside the block
    kw = {"quant_param_bytes_per_block": 0} if dt == KvDtype.FP8_E4M3 and H % 2 else {}
    fmt = KvFormat(dt, H, H, num_layers=2, **kw)
    w = make_world(fmt, [1, 15, 16, 17, 100, 33], seed=int(dt) * 11 + H,
                   fp8_scale=np.linspace(0.25, 3.0, 2 * H).astype(np.float32) if dt == KvDtype.FP8_E4M3 else None)
    append_gpu(w, fmt, 1)
    img, _ = oracle_image(w, fmt, 1)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    bad = np.nonzero(got != img)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}"


def test_fp8_conversion_special_values():
    """e4m3 saturation/subnormal/tie cases through K1 vs the oracle conversion."""
    fmt = KvFormat(KvDtype.FP8_E4M3, 1, 1, quant_param_bytes_per_block=0)
    vals = np.array([0.0, -0.0, 448.0, 449.0, 464.0, 465.0, 1e4, 65504.0, -65504.0,
                     2.0 ** -6, 2.0 ** -7, 2.0 ** -9, 2.0 ** -10, 1.5 * 2.0 ** -9, 0.001,
                     240.0, 248.0, 232.0, 1.0625, 1.1875, -3.3, 0.0195],
                    dtype=np.float32)
    allh = np.arange(65536, dtype=np.uint16).view(np.float16)
    allh = allh[np.isfinite(allh)]
    x = np.concatenate([vals.astype(np.float16), allh])
    n = (x.size + 127) // 128
    x = np.concatenate([x, np.zeros(n * 128 - x.size, np.float16)]).reshape(n, 1, 128)
    w = make_world(fmt, [n], seed=5, churn=False)
    w["k"], w["v"] = x, x[::-1].copy()
    append_gpu(w, fmt, 0)
    img, _ = oracle_image(w, fmt, 0)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    assert (got == img).all()
    # the oracle conversion itself against ml_dtypes (independent third party)
    import ml_dtypes
    xf = np.float32(allh)
    want = np.clip(xf, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    mine = np.array([oracle.lib.orc_f32_to_e4m3(float(v)) for v in xf], dtype=np.uint8)
    assert (mine == want).all()


@pytest.mark.parametrize("dt", [KvDtype.INT8, KvDtype.INT4], ids=["INT8", "INT4"])
def test_integer_quantisation_rounding_ties(dt):
    """K1 rounds x/s without a per-element division (reciprocal multiply, IEEE
    division only near a tie): rows built so that x/s hits exact .5 ties, and
    values one fp16 ulp either side of them, must give the oracle's bytes
    (rint of the correctly rounded quotient, half to even)."""
    fmt = KvFormat(dt, 1, 1, num_layers=1)
    rows = []
    for scale in (1.0, 0.25, 0.5, 2.0, 1.0 / 64):
        top = (127.0 if dt == KvDtype.INT8 else 15.0) * scale
        lo = -top if dt == KvDtype.INT8 else 0.0
        base = np.arange(-130, 130, dtype=np.float64) + 0.5 if dt == KvDtype.INT8 else \
            np.arange(0, 16, dtype=np.float64) + 0.5
        ties = np.clip(base * scale, lo, top)
        for nudge in (0, 1, -1):
            t16 = ties.astype(np.float16)
            if nudge:
                t16 = np.nextafter(t16, np.float16(np.inf * nudge)).astype(np.float16)
            r = np.resize(t16, 128).astype(np.float16)
            r[0], r[1] = np.float16(top), np.float16(lo)  # pin the row's scale (and zero)
            rows.append(r)
    x = np.stack(rows).reshape(len(rows), 1, 128)
    w = make_world(fmt, [len(rows)], seed=1, churn=False)
    w["k"], w["v"] = x, (-x if dt == KvDtype.INT8 else x[::-1].copy())
    append_gpu(w, fmt, 0)
    img, _ = oracle_image(w, fmt, 0)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    assert (got == img).all()


@pytest.mark.parametrize("dt", [KvDtype.INT8, KvDtype.INT4], ids=["INT8", "INT4"])
@pytest.mark.parametrize("H", [8, 4])
def test_integer_quantisation_special_rows(dt, H):
    """K1's fast path rounds by a magic-number add with no clamp; the rows it
    must hand to the IEEE path are exactly those where that is unsafe: NaN /
    +-inf elements, and scales that round to fp16 subnormals (tiny rows).
    Every such row (and ordinary ones around them) must give the oracle's
    bytes, on the H = 8 compile-time path and the generic one."""
    fmt = KvFormat(dt, H, H, num_layers=1)
    rng = np.random.default_rng(11)
    rows = []
    for kind in range(12):
        r = rng.standard_normal(128).astype(np.float32)
        if kind == 1:
            r[rng.integers(128)] = np.nan
        elif kind == 2:
            r[rng.integers(128)] = np.inf
        elif kind == 3:
            r[rng.integers(128)] = -np.inf
        elif kind == 4:
            r *= 1e-6  # scale below 2^-14: subnormal fp16
        elif kind == 5:
            r *= 3e-4  # around the normal / subnormal scale boundary
        elif kind == 6:
            r[:] = 0.0
        elif kind == 7:
            r[:] = 1.25
        elif kind == 8:
            r = np.where(r > 0, 65504.0, -65504.0).astype(np.float32)
        elif kind == 9:
            r *= 2.0 ** -20  # fp16 subnormal inputs
        elif kind == 10:
            r[:] = np.nan
        elif kind == 11:
            r[::2] = -0.0
        rows.append(r.astype(np.float16))
    x = np.stack(rows)  # [12, 128]
    T = 2 * 16
    k = np.stack([x[(t + np.arange(H)) % len(rows)] for t in range(T)])  # [T, H, 128]
    v = np.stack([x[(3 * t + 5 + np.arange(H)) % len(rows)] for t in range(T)])
    w = make_world(fmt, [T], seed=2, churn=False)
    w["k"], w["v"] = k, v
    append_gpu(w, fmt, 0)
    img, _ = oracle_image(w, fmt, 0)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    bad = np.nonzero(got != img)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}"


@pytest.mark.parametrize("H", [8, 4])
def test_fp8_special_rows_and_scales(H):
    """FP8 K1 fast path: select-free division with the sign of x OR-ed in
    (exact for positive scales); non-finite elements and zero / negative /
    non-finite scales go to the IEEE path.  Bytes must equal the oracle's."""
    fmt = KvFormat(KvDtype.FP8_E4M3, H, H, num_layers=1)
    rng = np.random.default_rng(12)
    rows = []
    for kind in range(6):
        r = (rng.standard_normal(128) * 40).astype(np.float32)
        if kind == 1:
            r[rng.integers(128)] = np.nan
        elif kind == 2:
            r[rng.integers(128)] = np.inf
        elif kind == 3:
            r[rng.integers(128)] = -np.inf
        elif kind == 4:
            r[::3] = -0.0
            r[1::3] = 0.0
        elif kind == 5:
            r *= 1e-7
        rows.append(r.astype(np.float16))
    x = np.stack(rows)
    T = 16
    k = np.stack([x[(t + np.arange(H)) % len(rows)] for t in range(T)])
    v = np.stack([x[(2 * t + 1 + np.arange(H)) % len(rows)] for t in range(T)])
    scales = np.array([0.5, -1.0, 2.0, 0.0, 1.0, -0.25, 3.0, 1e-3] * 2, np.float32)[:2 * H]
    w = make_world(fmt, [T], seed=3, churn=False, fp8_scale=scales)
    w["k"], w["v"] = k, v
    append_gpu(w, fmt, 0)
    img, _ = oracle_image(w, fmt, 0)
    got = kv.kv_tensor(w["pool"]).cpu().numpy()
    bad = np.nonzero(got != img)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}: {got[bad[:8]]} vs {img[bad[:8]]}"


def rel_err(o, r):
    o = o.reshape(-1, o.shape[-1]).astype(np.float64)
    r = r.reshape(-1, r.shape[-1])
    den = np.maximum(np.abs(r).max(axis=1), 1e-30)
    return (np.abs(o - r).max(axis=1) / den).max()


CASES = [
    # (dtype, Hkv, Hq, ctx lens)
    (KvDtype.FP16, 32, 32, [1024] * 4),
    (KvDtype.FP16, 8, 32, [1, 16, 17, 300, 2048, 0, 5]),
    (KvDtype.FP16, 2, 32, [777, 64]),
    (KvDtype.FP8_E4M3, 8, 32, [2048, 100, 31, 1]),
    (KvDtype.FP8_E4M3, 4, 4, [512, 513]),
    (KvDtype.INT8, 8, 32, [1000, 16, 3]),
    (KvDtype.INT8, 8, 64, [600]),
    (KvDtype.INT4, 8, 32, [8192, 17]),
    (KvDtype.INT4, 8, 8, [1, 2, 3, 4, 50, 129]),
    (KvDtype.INT4, 4, 40, [333]),
    # long contexts: the biased-V accumulator must not lose the signal's low bits
    (KvDtype.INT4, 8, 32, [16384, 4000, 700, 9000]),
    (KvDtype.INT8, 2, 16, [16384, 5000]),
]


@pytest.mark.parametrize("dt,Hkv,Hq,ctx", CASES,
                         ids=[f"{c[0].name}-{c[1]}x{c[2]}-{len(c[3])}" for c in CASES])
def test_decode_matches_oracle(dt, Hkv, Hq, ctx):
    fmt = KvFormat(dt, Hkv, Hq, num_layers=2)
    sc = None
    if dt == KvDtype.FP8_E4M3:
        sc = list(np.linspace(0.25, 2.0, 2 * Hkv))
    w = make_world(fmt, ctx, seed=len(ctx) + Hq, fp8_scale=sc)
    append_gpu(w, fmt, 1)
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    q = w["rng"].standard_normal((len(ctx), Hq, 128)).astype(np.float16)
    lse = torch.empty((len(ctx), Hq), dtype=torch.float32, device="cuda")
    out = kv.paged_decode(w["pool"], fmt, 1, dev(q), dev(w["table"]), dev(w["ctx"]), lse=lse,
                          kv_scales=None if w["scales"] is None else dev(w["scales"]))
    torch.cuda.synchronize()
    f = oracle.fmt(int(dt), Hkv, Hq, 128, 2, 16, fmt.qparams)
    ref, ref_lse = oracle.paged_decode(img, w["pool"].slab_size(),
                                       w["pool"].blocks_per_slab(fmt.key), f, 1, q.view(np.uint16),
                                       w["table"], w["ctx"], 1 / math.sqrt(128), w["scales"],
                                       nthreads=oracle.NPROC)
    o = out.cpu().numpy()
    live = w["ctx"] > 0
    err = rel_err(o[live], ref[live])
    assert err <= TOL[dt], err
    assert (o[~live] == 0).all()
    l = lse.cpu().numpy()
    assert np.abs(l[live] - ref_lse[live]).max() < 1e-3
    assert np.isneginf(l[~live]).all()


PACK_CASES = [
    # (dtype, Hkv, Hq, ctx lens): G = 4, 2, 1 with odd/even block counts per unit
    (KvDtype.FP16, 8, 32, [4096, 17, 33, 1, 0, 48]),
    (KvDtype.FP8_E4M3, 4, 8, [2000, 31, 16]),
    (KvDtype.INT8, 8, 32, [3000, 49, 2]),
    (KvDtype.INT8, 4, 4, [700, 65]),
    (KvDtype.INT4, 8, 32, [4100, 15, 16, 32, 0]),
    (KvDtype.INT4, 2, 4, [999, 1024]),
]


@pytest.mark.parametrize("mode", ["0", "1", "2", "4"], ids=["default", "unpacked", "packed_hmma", "packed_imma"])
@pytest.mark.parametrize("dt,Hkv,Hq,ctx", PACK_CASES,
                         ids=[f"{c[0].name}-{c[1]}x{c[2]}" for c in PACK_CASES])
def test_decode_packed_and_unpacked_steps(dt, Hkv, Hq, ctx, mode, monkeypatch):
    """Every K2 inner step for G <= 4 -- the packed ones (tile columns 0-3 and
    4-7 attend alternate blocks, folded per segment; the default for INT8/INT4
    computes QK on IMMA with 16-bit fixed-point Q) and the plain one -- match
    the oracle for every format."""
    monkeypatch.setenv("KVSLAB_DECODE_PACK", mode)
    fmt = KvFormat(dt, Hkv, Hq, num_layers=1)
    sc = list(np.linspace(0.5, 1.5, 2 * Hkv)) if dt == KvDtype.FP8_E4M3 else None
    w = make_world(fmt, ctx, seed=11 + Hq, fp8_scale=sc)
    append_gpu(w, fmt, 0)
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    q = w["rng"].standard_normal((len(ctx), Hq, 128)).astype(np.float16)
    lse = torch.empty((len(ctx), Hq), dtype=torch.float32, device="cuda")
    out = kv.paged_decode(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(w["ctx"]), lse=lse,
                          kv_scales=None if w["scales"] is None else dev(w["scales"]))
    torch.cuda.synchronize()
    f = oracle.fmt(int(dt), Hkv, Hq, 128, 1, 16, fmt.qparams)
    ref, ref_lse = oracle.paged_decode(img, w["pool"].slab_size(),
                                       w["pool"].blocks_per_slab(fmt.key), f, 0, q.view(np.uint16),
                                       w["table"], w["ctx"], 1 / math.sqrt(128), w["scales"],
                                       nthreads=oracle.NPROC)
    o = out.cpu().numpy()
    live = w["ctx"] > 0
    assert rel_err(o[live], ref[live]) <= TOL[dt]
    assert (o[~live] == 0).all()
    assert np.abs(lse.cpu().numpy()[live] - ref_lse[live]).max() < 1e-3


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
def test_decode_repeatable_and_workspace_clean(dt):
    """Two launches give identical bits (merge counters reset themselves)."""
    fmt = KvFormat(dt, 8, 32)
    w = make_world(fmt, [4096, 3000, 1, 0, 700], seed=3)
    append_gpu(w, fmt, 0)
    q = dev(w["rng"].standard_normal((5, 32, 128)).astype(np.float16))
    sc = None if w["scales"] is None else dev(w["scales"])
    a = kv.paged_decode(w["pool"], fmt, 0, q, dev(w["table"]), dev(w["ctx"]), kv_scales=sc).clone()
    b = kv.paged_decode(w["pool"], fmt, 0, q, dev(w["table"]), dev(w["ctx"]), kv_scales=sc)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_compaction_moves_bytes_and_keeps_outputs():
    fmt = KvFormat(KvDtype.INT4, 8, 32, num_layers=2)
    other = KvFormat(KvDtype.FP16, 8, 32).key
    w = make_world(fmt, [700, 300, 64, 1200], seed=9, extra_keys=(other,))
    pool = w["pool"]
    append_gpu(w, fmt, 1)
    table = dev(w["table"])
    ctx = dev(w["ctx"])
    q = dev(w["rng"].standard_normal((3, 32, 128)).astype(np.float16))
    t3, c3 = table[:3].contiguous(), ctx[:3].contiguous()
    before = kv.paged_decode(pool, fmt, 1, q, t3, c3).clone()
    # drop the longest sequence to open holes in many slabs, then compact
    bps = pool.blocks_per_slab(fmt.key)
    for b in range((1200 + 15) // 16):
        gid = int(w["table"][3, b])
        s, l = ks.SlabPool.split_global_block_id(gid, bps)
        pool.free_block(ks.BlockHandle(s, l, gid, fmt.key))
    st0 = pool.snapshot_stats()
    moves, freed = kv.compact(pool, fmt.key, tables=[t3])
    torch.cuda.synchronize()
    assert len(moves) > 0 and freed > 0
    assert pool.check_integrity()[0]
    assert pool.snapshot_stats().allocated_bytes == st0.allocated_bytes
    assert pool.snapshot_stats().free_slab_bytes > st0.free_slab_bytes
    after = kv.paged_decode(pool, fmt, 1, q, t3, c3)
    torch.cuda.synchronize()
    assert torch.equal(before, after)
    host = t3.cpu().numpy()
    srcs = {s_ for s_, _ in moves}
    for s in range(3):
        nb = (int(w["ctx"][s]) + 15) // 16
        assert not (set(host[s, :nb].tolist()) & srcs)
    kv.slab_table_sync(pool)
    assert kv.block_table_validate(pool, fmt.key, t3, c3) == 0


def test_block_table_update_and_validate():
    fmt = KvFormat(KvDtype.FP16, 8, 8)
    pool = ks.SlabPool(ks.SlabPoolConfig(16 * fmt.key * 4, fmt.key * 4, [fmt.key]), device=0)
    from paper_2509_06261_b200.engine import SlabModel
    m = SlabModel(pool, fmt, max_seqs=4, max_blocks_per_seq=8)
    assert m.admit(0, 40) and m.admit(1, 16) and m.admit(2, 1)
    m.cached[0] = 40
    assert m.ensure_capacity(0, 49)
    m.sync()
    torch.cuda.synchronize()
    host = m.table.cpu().numpy()
    for s in range(3):
        for b, h in enumerate(m.handles[s]):
            assert host[s, b] == h.global_block_id
    kv.slab_table_sync(pool)
    ctx = torch.tensor([49, 16, 1, 0], dtype=torch.int32, device="cuda")
    assert kv.block_table_validate(pool, fmt.key, m.table, ctx) == 0
    for s in range(3):  # all blocks freed -> every slab returns FREE
        m.release(s)
    kv.slab_table_sync(pool)
    assert kv.block_table_validate(pool, fmt.key, m.table, ctx) > 0
    st = kv.slab_table_tensor(pool).cpu().numpy()
    for i in range(pool.slab_count()):
        assert st[i, 0] == pool.slab_key(i)
        assert (st[i, 1] >> 32) == int(pool.slab_state(i))


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
def test_fused_append_decode_matches_separate_k1_k2(dt):
    """ks_paged_decode_append == ks_kv_append(last token) + ks_paged_decode,
    bit for bit (bytes written and outputs)."""
    fmt = KvFormat(dt, 8, 32, num_layers=2)
    ctx = [1, 16, 17, 600, 2049, 33]
    w = make_world(fmt, ctx, seed=21 + int(dt))
    pool = w["pool"]
    # the prefix (all but the last token of each sequence) is appended by K1
    keep = np.concatenate([np.arange(c - 1) + sum(ctx[:s]) for s, c in enumerate(ctx)]).astype(int)
    last = np.array([sum(ctx[:s + 1]) - 1 for s in range(len(ctx))])
    sc = None if w["scales"] is None else dev(w["scales"])
    kv.kv_append(pool, fmt, 1, dev(w["k"][keep]), dev(w["v"][keep]), dev(w["tok_seq"][keep]),
                 dev(w["tok_pos"][keep]), dev(w["table"]), sc)
    torch.cuda.synchronize()
    base = kv.kv_tensor(pool).clone()
    q = dev(w["rng"].standard_normal((len(ctx), 32, 128)).astype(np.float16))
    table, ctxd = dev(w["table"]), dev(w["ctx"])
    knew, vnew = dev(w["k"][last]), dev(w["v"][last])
    fused = kv.paged_decode(pool, fmt, 1, q, table, ctxd, kv_scales=sc, k_new=knew, v_new=vnew)
    torch.cuda.synchronize()
    img_fused = kv.kv_tensor(pool).clone()
    kv.kv_tensor(pool).copy_(base)
    kv.kv_append(pool, fmt, 1, knew, vnew, dev(np.arange(len(ctx), dtype=np.int32)),
                 dev(w["ctx"] - 1), table, sc)
    sep = kv.paged_decode(pool, fmt, 1, q, table, ctxd, kv_scales=sc)
    torch.cuda.synchronize()
    assert torch.equal(img_fused, kv.kv_tensor(pool))
    assert torch.equal(fused, sep)


@pytest.mark.parametrize("dt", [KvDtype.FP16, KvDtype.INT4], ids=["FP16", "INT4"])
def test_decode_mostly_empty_slots(dt):
    """A fixed-size batch with most slots empty (ctx 0): zero outputs and -inf
    LSE for the empty slots (written by the whole grid over poisoned
    buffers), oracle outputs for the live ones."""
    ctx = [0] * 40
    for i, c in ((3, 700), (17, 1), (22, 2048), (39, 64), (5, 333)):
        ctx[i] = c
    fmt = KvFormat(dt, 8, 32, num_layers=1)
    w = make_world(fmt, ctx, seed=91)
    append_gpu(w, fmt, 0)
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    q = w["rng"].standard_normal((len(ctx), 32, 128)).astype(np.float16)
    out = torch.full((len(ctx), 32, 128), 7.0, dtype=torch.float16, device="cuda")  # poison
    lse = torch.zeros((len(ctx), 32), dtype=torch.float32, device="cuda")
    kv.paged_decode(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(w["ctx"]), out=out, lse=lse)
    torch.cuda.synchronize()
    f = oracle.fmt(int(dt), 8, 32, 128, 1, 16, fmt.qparams)
    ref, _ = oracle.paged_decode(img, w["pool"].slab_size(), w["pool"].blocks_per_slab(fmt.key), f, 0,
                                 q.view(np.uint16), w["table"], w["ctx"], 1 / math.sqrt(128), None,
                                 nthreads=oracle.NPROC)
    o = out.cpu().numpy()
    live = w["ctx"] > 0
    assert rel_err(o[live], ref[live]) <= TOL[dt]
    assert (o[~live] == 0).all()
    assert np.isneginf(lse.cpu().numpy()[~live]).all()


def test_compact_key_remaps_every_owner_of_the_key():
    """Two co-located models with the same KvFormat share one slab key
    (ADVICE r1): ks_compact rewrites both models' handles and device tables,
    the moved bytes decode identically, and the table validator passes."""
    from paper_2509_06261_b200.engine import SlabModel
    fmt = KvFormat(KvDtype.FP8_E4M3, 8, 32, num_layers=2)
    slab = fmt.key * 8
    pool = ks.SlabPool(ks.SlabPoolConfig(64 * slab, slab, [fmt.key]), device=0)
    kv.kv_tensor(pool).zero_()
    rng = np.random.default_rng(5)
    a, b = SlabModel(pool, fmt, 16, 40), SlabModel(pool, fmt, 16, 40)
    # interleaved claims so every slab holds both models' blocks
    for step in range(12):
        for m in (a, b):
            for s in range(16):
                if step == 0:
                    assert m.admit(s, 16)
                elif len(m.handles[s]) < 12:
                    m.cached[s] = (len(m.handles[s])) * 16
                    assert m.ensure_capacity(s, m.cached[s] + 1)
    for m in (a, b):
        for s in range(16):
            m.cached[s] = len(m.handles[s]) * 16 - int(rng.integers(0, 16))
        m.sync()
    sc = dev(np.full(16, 0.5, np.float32))
    outs = []
    for m in (a, b):
        ctx = torch.tensor(m.ctx_lens(), dtype=torch.int32, device="cuda")
        T = int(ctx.sum())
        seqs = torch.repeat_interleave(torch.arange(16, dtype=torch.int32, device="cuda"), ctx)
        pos = torch.cat([torch.arange(int(c), dtype=torch.int32, device="cuda") for c in ctx])
        k = torch.randn(T, 8, 128, dtype=torch.float16, device="cuda")
        kv.kv_append(pool, fmt, 1, k, -k, seqs, pos, m.table, sc)
        q = torch.randn(16, 32, 128, dtype=torch.float16, device="cuda")
        outs.append((q, ctx))
    # release most sequences of both models: holes everywhere
    for m in (a, b):
        for s in range(16):
            if s % 4:
                m.release(s)
    live = [s for s in range(16) if s % 4 == 0]
    ref = []
    for m, (q, ctx) in zip((a, b), outs):
        c = torch.tensor(m.ctx_lens(), dtype=torch.int32, device="cuda")
        ref.append(kv.paged_decode(pool, fmt, 1, q, m.table, c, kv_scales=sc).clone())
    st0 = pool.snapshot_stats()
    n, freed = a.compact()
    torch.cuda.synchronize()
    assert n > 0 and freed > 0
    assert pool.check_integrity()[0]
    assert pool.snapshot_stats().allocated_bytes == st0.allocated_bytes
    kv.slab_table_sync(pool)
    for i, (m, (q, ctx)) in enumerate(zip((a, b), outs)):
        host = m.table.cpu().numpy()
        for s in live:
            assert [h.global_block_id for h in m.handles[s]] == host[s, :len(m.handles[s])].tolist()
        c = torch.tensor(m.ctx_lens(), dtype=torch.int32, device="cuda")
        assert kv.block_table_validate(pool, fmt.key, m.table, c) == 0
        got = kv.paged_decode(pool, fmt, 1, q, m.table, c, kv_scales=sc)
        torch.cuda.synchronize()
        assert torch.equal(got[live], ref[i][live])
    for m in (a, b):  # every handle is still freeable exactly once
        for s in live:
            m.release(s)
    assert pool.allocated_block_count() == 0 and pool.check_integrity()[0]


def test_block_table_remap_beyond_one_staging_slot():
    """More moves than one staging slot holds (65,536): the remap is chunked."""
    fmt = KvFormat(KvDtype.INT4, 8, 8)
    pool = ks.SlabPool(ks.SlabPoolConfig(8 * fmt.key * 64, fmt.key * 64, [fmt.key]), device=0)
    n = 70000
    src = np.arange(n, dtype=np.int64) * 2 + 1
    dst = src - 1
    table = torch.from_numpy(np.concatenate([src, dst, [7, 10**6]]).astype(np.int32)).cuda()
    moves = (ks._lib.ks_block_move * n)(*[ks._lib.ks_block_move(int(s), int(d)) for s, d in zip(src, dst)])
    ks.slab_pool.check(ks._lib.lib.ks_block_table_remap(pool.handle, table.data_ptr(), table.numel(),
                                                        moves, n, None))
    torch.cuda.synchronize()
    got = table.cpu().numpy()
    assert (got[:n] == dst).all() and (got[n:2 * n] == dst).all()
    assert got[-2] == 6 and got[-1] == 10**6


def test_pool_destroyed_during_another_capture():
    """A pool torn down (here: close(); in practice a garbage collector) while
    another pool's decode is being captured into a CUDA graph must not
    invalidate that capture (the teardown's cudaFree / event syncs run in
    relaxed capture mode)."""
    fmt = KvFormat(KvDtype.FP8_E4M3, 8, 32, num_layers=1)
    w = make_world(fmt, [40, 300], seed=21, churn=False,
                   fp8_scale=np.ones(16, np.float32))
    append_gpu(w, fmt, 0)
    doomed = ks.SlabPool(ks.SlabPoolConfig(8 * fmt.key * 4, fmt.key * 4, [fmt.key]), device=0)
    kv.kv_tensor(doomed).zero_()
    q = dev(np.random.default_rng(3).standard_normal((2, 32, 128)).astype(np.float16))
    table, ctx, sc = dev(w["table"]), dev(w["ctx"]), dev(w["scales"])
    ws = kv.DecodeWorkspace(w["pool"], fmt, 2)
    out = kv.paged_decode(w["pool"], fmt, 0, q, table, ctx, kv_scales=sc, workspace=ws)
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            kv.paged_decode(w["pool"], fmt, 0, q, table, ctx, out=out, kv_scales=sc, workspace=ws)
            doomed.close()  # teardown in the middle of the capture
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
@pytest.mark.parametrize("sms", [1, 7, 37, 111])
def test_decode_under_sm_share(dt, sms):
    """A model's SM share (ks_set_decode_sm_share, the co-location fence the
    bench autotunes -- e.g. INT4 in 37 SMs) changes the grid and so every
    unit's CTA split and merge: the outputs must still match the oracle, from
    one CTA (no split) to most of the GPU."""
    fmt = KvFormat(dt, 8, 32, num_layers=2)
    ctx = [1300, 17, 2048, 1, 700, 64, 0, 333]
    sc = list(np.linspace(0.5, 2.0, 16)) if dt == KvDtype.FP8_E4M3 else None
    w = make_world(fmt, ctx, seed=sms + int(dt), fp8_scale=sc)
    append_gpu(w, fmt, 0)
    kv.set_decode_sm_share(w["pool"], fmt.key, sms)
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    q = w["rng"].standard_normal((len(ctx), 32, 128)).astype(np.float16)
    out = kv.paged_decode(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(w["ctx"]),
                          kv_scales=None if w["scales"] is None else dev(w["scales"]))
    torch.cuda.synchronize()
    f = oracle.fmt(int(dt), 8, 32, 128, 2, 16, fmt.qparams)
    ref, _ = oracle.paged_decode(img, w["pool"].slab_size(), w["pool"].blocks_per_slab(fmt.key), f, 0,
                                 q.view(np.uint16), w["table"], w["ctx"], 1 / math.sqrt(128), w["scales"],
                                 nthreads=oracle.NPROC)
    o = out.cpu().numpy()
    live = w["ctx"] > 0
    assert rel_err(o[live], ref[live]) <= TOL[dt]
    assert (o[~live] == 0).all()

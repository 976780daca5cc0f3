"""The CPU oracle is pinned before it is trusted: RNG, geometry and allocator
against the compiled reference's golden vectors; number formats against
numpy / ml_dtypes; quantisation/attention internal consistency."""
import ctypes as C
import json
import math
import os

import ml_dtypes
import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_rng_matches_reference_mt19937_64():
    gold = json.load(open(os.path.join(GOLD, "rng.json")))
    for seed, vals in gold.items():
        mine = oracle.uniforms(int(seed), len(vals))
        assert [float.fromhex(v) for v in vals] == mine.tolist(), seed


def test_geometry_matches_reference():
    for row in json.load(open(os.path.join(GOLD, "precision.json"))):
        ts, bs = C.c_uint64(), C.c_uint64()
        a = oracle.lib.orc_token_size(row["kv_heads"], row["head_dim"], row["tp"], row["kv_bits"],
                                      C.byref(ts))
        b = oracle.lib.orc_kv_block_size(row["kv_heads"], row["head_dim"], row["tp"],
                                         row["kv_bits"], row["tpb"], row["qparams"], row["layers"],
                                         C.byref(bs))
        got = f"P {ts.value} {bs.value}" if a == 0 and b == 0 else "E InvalidProfileError"
        assert got == row["expected"], row


def test_fp16_conversion_matches_numpy():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000) * s for s in (1e-8, 1e-5, 1e-2, 1, 1e3, 6e4)])
    x = np.concatenate([x, [65504, 65519.99, 65520, 7e4, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26,
                            0.0, -0.0]]).astype(np.float32)
    want = x.astype(np.float16).view(np.uint16)
    got = np.array([oracle.lib.orc_f32_to_f16(float(v)) for v in x], dtype=np.uint16)
    assert (got == want).all()


def test_e4m3_conversion_matches_ml_dtypes_saturating():
    allh = np.arange(65536, dtype=np.uint16).view(np.float16)
    xf = np.float32(allh[np.isfinite(allh)])
    rng = np.random.default_rng(1)
    xf = np.concatenate([xf, (rng.standard_normal(50000) * 100).astype(np.float32)])
    want = np.clip(xf, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    got = np.array([oracle.lib.orc_f32_to_e4m3(float(v)) for v in xf], dtype=np.uint8)
    assert (got == want).all()
    for c in range(256):
        if c & 0x7F == 0x7F:
            continue
        assert oracle.lib.orc_e4m3_to_f32(c) == float(np.uint8(c).view(ml_dtypes.float8_e4m3fn))


def test_swizzle_is_an_involution_within_lines():
    for o in range(0, 4096, 16):
        s = oracle.lib.orc_swz(o)
        assert s >> 7 == o >> 7 and oracle.lib.orc_swz(s) == o


def _world(dt, H=4, Hq=8, ctx=(40, 17)):
    f = oracle.fmt(dt, H, Hq, 128, 2, 16)
    key = oracle.lib.orc_fmt_key(C.byref(f))
    nb = [(c + 15) // 16 for c in ctx]
    table = np.zeros((len(ctx), max(nb)), np.int32)
    g = 0
    for s, n in enumerate(nb):
        table[s, :n] = np.arange(g, g + n)[::-1]
        g += n
    img = np.zeros(g * key, np.uint8)
    rng = np.random.default_rng(int(dt))
    T = sum(ctx)
    k = rng.standard_normal((T, H, 128)).astype(np.float16)
    v = rng.standard_normal((T, H, 128)).astype(np.float16)
    ts = np.repeat(np.arange(len(ctx), dtype=np.int32), ctx)
    tp = np.concatenate([np.arange(c, dtype=np.int32) for c in ctx])
    sc = np.linspace(0.5, 2, 2 * H).astype(np.float32) if dt == 1 else None
    oracle.append(img, img.size, g, f, 1, k.view(np.uint16), v.view(np.uint16), ts, tp, table, sc)
    return f, img, g, table, k, v, np.asarray(ctx, np.int32), sc


def test_quantised_attention_close_to_fp_attention():
    """fp64 oracle decode over dequantised bytes vs plain numpy attention on
    the original fp16 K/V: the gap is the format's quantisation error."""
    tol = {0: 1e-6, 1: 0.08, 2: 0.03, 3: 0.35}
    for dt in (0, 1, 2, 3):
        f, img, g, table, k, v, ctx, sc = _world(dt)
        rng = np.random.default_rng(9)
        q = rng.standard_normal((len(ctx), 8, 128)).astype(np.float16)
        out, lse = oracle.paged_decode(img, img.size, g, f, 1, q.view(np.uint16), table, ctx,
                                       1 / math.sqrt(128), sc)
        off = 0
        for s, c in enumerate(ctx):
            for hq in range(8):
                kk = k[off:off + c, hq // 2].astype(np.float64)
                vv = v[off:off + c, hq // 2].astype(np.float64)
                sco = kk @ q[s, hq].astype(np.float64) / math.sqrt(128)
                p = np.exp(sco - sco.max())
                ref = (p / p.sum()) @ vv
                err = np.abs(out[s, hq] - ref).max() / np.abs(ref).max()
                assert err < tol[dt], (dt, s, hq, err)
                if dt == 0:
                    assert abs(lse[s, hq] - (sco.max() + math.log(p.sum()))) < 1e-9
            off += c


def test_decode_bytes_formula():
    f = oracle.fmt(0, 32, 32, 128, 1, 16)
    # config 1 = 134 350 848 B
    assert oracle.decode_bytes(f, np.full(8, 1024, np.int32)) == 134350848

"""Pins the oracle's KV quantisers (oracle/kvslab_oracle.c, test
infrastructure) to the published third-party rules they restate, each
re-written here in plain numpy float32 (IEEE round-to-nearest per op):

* FP8 -- vLLM's FP8 KV cache (the paper's FP8 path): per
  tensor/head scale s, code = e4m3(saturate(x / s)) (vLLM
  csrc/quantization/fp8 scaled_convert: divide, then cvt.rn.satfinite);
  the e4m3 rounding comes from ml_dtypes (third party).
* INT4 -- QServe/QoQ KV4: asymmetric per (token, head)
  group of d, scale = (max - min) / 15 and zero = min, both stored fp16,
  code = clamp(round((x - zero) / scale), 0, 15).
* INT8 -- symmetric per (token, head): scale = fp16(amax / 127),
  code = clamp(round(x / scale), -127, 127).

Round = round-half-to-even (rint).  The oracle's bytes are read back
through tests/_layout.py, so layout and rule are both
checked independently of the oracle's own helpers.  The GPU kernels are
bit-exact against the oracle (tests/test_gpu_kernels.py) and, for FP8,
against vLLM's own kernel (tests/test_gpu_thirdparty.py).
"""
import ctypes

import ml_dtypes
import numpy as np
import pytest

import oracle
from _layout import read_codes, read_params


def _rows(dt_code, seed, n_tok=48, H=4):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((n_tok, H, 128)).astype(np.float16)
    v = rng.standard_normal((n_tok, H, 128)).astype(np.float16)
    for a in (k, v):  # 1 % outliers at 8 sigma, a constant row, near-ties
        m = rng.random(a.shape) < 0.01
        a[m] *= 8
        a[3, 1, :] = np.float16(0.75)
        a[5, 0, :17] = np.float16(-2.0)
    f = oracle.fmt(dt_code, H, H * 4, 128, 2, 16)
    key = oracle.lib.orc_fmt_key(ctypes.byref(f))
    nb = (n_tok + 15) // 16
    img = np.zeros(nb * key, dtype=np.uint8)
    table = np.arange(nb, dtype=np.int32).reshape(1, nb)
    ts = np.zeros(n_tok, np.int32)
    tp = np.arange(n_tok, dtype=np.int32)
    sc = np.linspace(0.25, 2.0, 2 * H).astype(np.float32) if dt_code == 1 else None
    oracle.append(img, nb * key, nb, f, 1, k.view(np.uint16), v.view(np.uint16), ts, tp, table, sc)
    layer_bytes = key // 2
    return img, key, layer_bytes, k, v, sc, H


def _blocks(img, key):
    return [img[b * key:(b + 1) * key] for b in range(img.size // key)]


@pytest.mark.parametrize("seed", [0, 1])
def test_int4_is_qserve_kv4(seed):
    img, key, lb, k, v, _, H = _rows(3, seed)
    blocks = _blocks(img, key)
    for kv, x in ((0, k), (1, v)):
        for tok in range(x.shape[0]):
            blk, t = blocks[tok // 16], tok % 16
            for h in range(H):
                xf = x[tok, h].astype(np.float32)
                mn, mx = xf.min(), xf.max()
                scale = np.float16(np.float32(mx - mn) / np.float32(15))
                zero = np.float16(mn)
                sf, zf = np.float32(scale), np.float32(zero)
                want = (np.zeros(128, np.int64) if sf == 0 else
                        np.clip(np.rint((xf - zf) / sf), 0, 15).astype(np.int64))
                got = read_codes(blk, "int4", H, lb, 1, kv, h, t)
                assert (got == want).all(), (kv, tok, h)
                p = read_params(blk, "int4", H, lb, 1, kv, h, t)
                assert p[0] == scale and p[1].view(np.uint16) == zero.view(np.uint16)


@pytest.mark.parametrize("seed", [0, 1])
def test_int8_symmetric_per_token_head(seed):
    img, key, lb, k, v, _, H = _rows(2, seed)
    blocks = _blocks(img, key)
    for kv, x in ((0, k), (1, v)):
        for tok in range(x.shape[0]):
            blk, t = blocks[tok // 16], tok % 16
            for h in range(H):
                xf = x[tok, h].astype(np.float32)
                scale = np.float16(np.abs(xf).max() / np.float32(127))
                sf = np.float32(scale)
                want = (np.zeros(128, np.int64) if sf == 0 else
                        np.clip(np.rint(xf / sf), -127, 127).astype(np.int64))
                got = read_codes(blk, "int8", H, lb, 1, kv, h, t).view(np.int8).astype(np.int64)
                assert (got == want).all(), (kv, tok, h)
                assert read_params(blk, "int8", H, lb, 1, kv, h, t)[0] == scale


def test_fp8_is_vllm_scaled_e4m3():
    img, key, lb, k, v, sc, H = _rows(1, 3)
    blocks = _blocks(img, key)
    for kv, x in ((0, k), (1, v)):
        for tok in range(x.shape[0]):
            blk, t = blocks[tok // 16], tok % 16
            for h in range(H):
                q = x[tok, h].astype(np.float32) / np.float32(sc[kv * H + h])
                want = np.clip(q, -448, 448).astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
                got = read_codes(blk, "fp8", H, lb, 1, kv, h, t)
                assert (got == want).all(), (kv, tok, h)

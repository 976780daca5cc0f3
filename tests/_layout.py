"""Reads quantised codes and params back out of a slab block image, from the
layout written down in DESIGN.md section 3 (independently of the C oracle's
offset helpers): a layer sub-block is K[H][chunk] | V[H][chunk] | params,
every 16-byte granule XOR-swizzled inside its 128-byte line.  Test helper."""
import numpy as np


def swz(o):
    o = np.asarray(o, dtype=np.int64)
    return o ^ (((o >> 7) & 7) << 4)


def chunk_bytes(bits, d=128, tpb=16):
    return tpb * d * bits // 8


def element_offsets(dtype, kv, t, d=128):
    """Byte offset (inside the (kv, head) chunk) and nibble of element i of
    token slot t, for i = 0..d-1.  dtype: 'fp16' | 'fp8' | 'int8' | 'int4'."""
    i = np.arange(d)
    if dtype == "fp16":  # half-major: dims [0,64) of 16 tokens, then [64,128)
        return swz((i // 64) * 16 * 128 + t * 128 + 2 * (i % 64)), None
    if dtype in ("fp8", "int8"):
        return swz(t * d + i), None
    if kv == 0:  # INT4 K: 64-byte token rows, low nibble first
        return swz(t * (d // 2) + i // 2), i % 2
    # INT4 V: token-pair lines, 2-byte interleave
    t8 = t & 7
    tp, side = (t8 & 1) | ((t8 >> 2) << 1), (t8 >> 1) & 1
    line = 2 * tp + (t >> 3)
    j = i // 2
    return swz(line * 128 + 4 * (j >> 1) + 2 * side + (j & 1)), i % 2


def read_codes(block, dtype, H, layer_bytes, layer, kv, h, t, d=128):
    """uint8 codes (int8/fp8 bytes, int4 nibbles) of one row."""
    bits = {"fp16": 16, "fp8": 8, "int8": 8, "int4": 4}[dtype]
    base = layer * layer_bytes + (kv * H + h) * chunk_bytes(bits, d)
    off, nib = element_offsets(dtype, kv, t, d)
    b = block[base + off]
    if nib is None:
        return b
    return (b >> (4 * nib)) & 0xF


def read_params(block, dtype, H, layer_bytes, layer, kv, h, t, d=128, tpb=16):
    """INT8: fp16 scale; INT4: fp16 (scale, zero) -- per (K|V, head, token)."""
    bits = {"int8": 8, "int4": 4}[dtype]
    p0 = layer * layer_bytes + 2 * H * chunk_bytes(bits, d)
    if dtype == "int8":
        o = p0 + ((kv * H + h) * tpb + t) * 2
        return block[o:o + 2].view(np.float16)
    o = p0 + ((kv * H + h) * tpb + t) * 4
    return block[o:o + 4].view(np.float16)

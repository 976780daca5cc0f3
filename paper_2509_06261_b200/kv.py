"""Device data path: KV formats, K1 append, K2 paged decode, K3 compaction.

Thin host wrappers over libkvslab.so.  Tensors are torch CUDA tensors (used
only as device buffers and streams); the arguments cross the C ABI as raw
pointers.  There is no CPU fallback: every function requires the pool's
device tensor and calls a CUDA kernel.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _lib as L
from .slab_pool import KvSlabError, SlabPool, check


class KvDtype(enum.IntEnum):
    FP16 = 0
    FP8_E4M3 = 1
    INT8 = 2
    INT4 = 3


_BITS = {KvDtype.FP16: 16, KvDtype.FP8_E4M3: 8, KvDtype.INT8: 8, KvDtype.INT4: 4}


_C_FMT_CACHE: dict = {}


@dataclass(frozen=True)
class KvFormat:
    """Per-model KV format (ks_kv_format).  quant_param_bytes_per_block=None
    selects the format's natural per-layer quant-param size."""
    kv_dtype: KvDtype
    num_kv_heads: int
    num_q_heads: int
    head_dim: int = 128
    num_layers: int = 1
    tokens_per_block: int = 16
    quant_param_bytes_per_block: Optional[int] = None

    @property
    def qparams(self) -> int:
        if self.quant_param_bytes_per_block is not None:
            return self.quant_param_bytes_per_block
        H, T = self.num_kv_heads, self.tokens_per_block
        return {KvDtype.FP16: 0, KvDtype.FP8_E4M3: 2 * H * 4, KvDtype.INT8: 2 * H * T * 2,
                KvDtype.INT4: 2 * H * T * 4}[KvDtype(self.kv_dtype)]

    @property
    def bits(self) -> int:
        return _BITS[KvDtype(self.kv_dtype)]

    @property
    def token_size(self) -> int:  # per layer, K+V, precision.cpp:76-89
        return self.num_kv_heads * self.head_dim * 2 * self.bits // 8

    @property
    def chunk_bytes(self) -> int:
        return self.tokens_per_block * self.head_dim * self.bits // 8

    @property
    def layer_bytes(self) -> int:
        return self.tokens_per_block * self.token_size + self.qparams

    @property
    def key(self) -> int:  # == kv_block_size(profile), precision.cpp:91-99
        return self.num_layers * self.layer_bytes

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    def to_c(self) -> L.ks_kv_format:
        return L.ks_kv_format(int(self.kv_dtype), self.num_kv_heads, self.num_q_heads,
                              self.head_dim, self.num_layers, self.tokens_per_block, self.qparams)

    def c_ref(self):
        """byref of this format's C struct, built once per distinct format
        (the C side only reads it during the call): the per-layer hot paths
        skip the struct construction.  Cached by value outside the instance,
        so formats stay plain picklable dataclasses."""
        r = _C_FMT_CACHE.get(self)
        if r is None:
            c = self.to_c()
            r = _C_FMT_CACHE[self] = (c, C.byref(c))
        return r[1]

    def shard(self, tp: int) -> "KvFormat":
        """Format of one tensor-parallel shard: KV and Q
        heads split over `tp` GPUs, each shard an ordinary pool over its heads.
        Rejects heads % tp != 0 like token_size (precision.cpp:80-83); the
        shard's key equals kv_block_size(profile with tp_degree=tp)."""
        if tp < 1 or self.num_kv_heads % tp or self.num_q_heads % tp:
            raise ValueError(f"kv heads {self.num_kv_heads} / q heads {self.num_q_heads} "
                             f"not divisible by tp {tp}")
        qp = self.quant_param_bytes_per_block
        return dataclasses.replace(self, num_kv_heads=self.num_kv_heads // tp,
                                   num_q_heads=self.num_q_heads // tp,
                                   quant_param_bytes_per_block=None if qp is None else qp // tp)

    def head_slices(self, tp: int, rank: int) -> Tuple[slice, slice]:
        """(kv-head slice, q-head slice) of shard `rank`: contiguous head ranges,
        so every q head stays with its kv head (GQA groups are never split)."""
        kv, q = self.num_kv_heads // tp, self.num_q_heads // tp
        return slice(rank * kv, (rank + 1) * kv), slice(rank * q, (rank + 1) * q)

    def decode_bytes(self, ctx_lens: Sequence[int]) -> int:
        """Algorithmic bytes of one K2 launch: every cached K/V
        byte + quant params + the block-table entries + Q + O, each once."""
        T = self.tokens_per_block
        total = 0
        for c in ctx_lens:
            nb = (c + T - 1) // T if c > 0 else 0
            total += c * self.token_size + nb * self.qparams + nb * 4
        total += 2 * len(ctx_lens) * self.num_q_heads * self.head_dim * 2
        return total

    def append_bytes(self, n_tokens: int) -> int:
        """Algorithmic bytes of one K1 launch: fp16 K,V in + quantised bytes out
        + quant params written + token metadata/table lookups."""
        H, T = self.num_kv_heads, self.tokens_per_block
        per_tok_params = {KvDtype.FP16: 0, KvDtype.FP8_E4M3: 0, KvDtype.INT8: 2 * H * 2,
                          KvDtype.INT4: 2 * H * 4}[KvDtype(self.kv_dtype)]
        return n_tokens * (2 * H * self.head_dim * 2 + self.token_size + per_tok_params + 12)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class _CAI:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def kv_tensor(pool: SlabPool) -> torch.Tensor:
    """Zero-copy uint8 view of the pool's single KV tensor."""
    base, nbytes = C.c_void_p(), C.c_uint64()
    check(L.lib.ks_device_base(pool.handle, C.byref(base), C.byref(nbytes)))
    if not base.value:
        raise KvSlabError("pool has no device tensor")
    return torch.as_tensor(_CAI(base.value, nbytes.value), device=f"cuda:{pool.device}")


def scrubbed_bytes(pool: SlabPool) -> int:
    """Bytes cleared because slabs were re-formatted to another key (ks_pool_scrubbed_bytes)."""
    out = C.c_uint64()
    check(L.lib.ks_pool_scrubbed_bytes(pool.handle, C.byref(out)))
    return out.value


def validate_format(pool: SlabPool, fmt: KvFormat) -> None:
    f = fmt.to_c()
    check(L.lib.ks_validate_format(pool.handle, C.byref(f)))


def slab_table_sync(pool: SlabPool, stream=None) -> None:
    check(L.lib.ks_slab_table_sync(pool.handle, _stream(stream)))


def slab_table_tensor(pool: SlabPool) -> torch.Tensor:
    """Zero-copy view of the device slab table: int64 [slab_count, 2] where
    [:,0] = key and [:,1] = blocks_total | state << 32."""
    t = C.c_void_p()
    check(L.lib.ks_slab_table_device(pool.handle, C.byref(t)))
    n = pool.slab_count()
    raw = torch.as_tensor(_CAI(t.value, n * 16), device=f"cuda:{pool.device}")
    return raw.view(torch.int64).view(n, 2)


def block_table_update(pool: SlabPool, table: torch.Tensor, rows: Sequence[int],
                       cols: Sequence[int], vals: Sequence[int], stream=None) -> None:
    """Delta upload of block-table entries (host triples -> device scatter)."""
    n = len(rows)
    if n == 0:
        return
    r = (C.c_int32 * n)(*rows)
    c = (C.c_int32 * n)(*cols)
    v = (C.c_int32 * n)(*vals)
    check(L.lib.ks_block_table_update(pool.handle, _ptr(table), table.stride(0), r, c, v, n,
                                      _stream(stream)))


def block_table_validate(pool: SlabPool, key: int, table: torch.Tensor, ctx_lens: torch.Tensor,
                         tokens_per_block: int = 16, stream=None) -> int:
    bad = C.c_uint64()
    check(L.lib.ks_block_table_validate(pool.handle, key, _ptr(table), table.stride(0),
                                        _ptr(ctx_lens), table.shape[0], tokens_per_block,
                                        _stream(stream), C.byref(bad)))
    return bad.value


def kv_append(pool: SlabPool, fmt: KvFormat, layer: int, k: torch.Tensor, v: torch.Tensor,
              tok_seq: torch.Tensor, tok_pos: torch.Tensor, block_table: torch.Tensor,
              kv_scales: Optional[torch.Tensor] = None, stream=None) -> None:
    """K1: quantise + write n tokens' K/V ([n, Hkv, d] fp16) into their slab blocks."""
    assert k.dtype == torch.float16 and v.dtype == torch.float16
    assert k.is_contiguous() and v.is_contiguous() and block_table.dtype == torch.int32
    check(L.lib.ks_kv_append(pool.handle, fmt.c_ref(), layer, _ptr(k), _ptr(v), k.shape[0],
                             _ptr(tok_seq), _ptr(tok_pos), _ptr(block_table),
                             block_table.stride(0), _ptr(kv_scales), _stream(stream)))


class DecodeWorkspace:
    """K2 scratch (fp32 partials of sequence-heads split across CTAs).  Needs
    no initialisation; concurrent launches need distinct workspaces."""

    def __init__(self, pool: SlabPool, fmt: KvFormat, max_batch: int, stream=None):
        f = fmt.to_c()
        n = C.c_size_t()
        check(L.lib.ks_paged_decode_workspace_size(pool.handle, C.byref(f), max_batch,
                                                   C.byref(n)))
        self.nbytes = n.value
        self.max_batch = max_batch
        # allocated on the stream it is used on, so the caching allocator
        # orders its reuse after the kernels of that stream
        with torch.cuda.stream(_torch_stream(stream, pool.device)):
            self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=f"cuda:{pool.device}")


def _torch_stream(stream, device) -> torch.cuda.Stream:
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream), device=f"cuda:{device}")


# Default scratch lives on the pool object (dropped with it), per (slab key,
# stream): co-located models or streams never share a buffer.
def _pool_cache(pool: SlabPool, name: str) -> dict:
    d = pool.__dict__.get(name)
    if d is None:
        d = pool.__dict__[name] = {}
    return d


def _default_decode_ws(pool: SlabPool, fmt: KvFormat, B: int, stream) -> DecodeWorkspace:
    per = _pool_cache(pool, "_ks_decode_ws")
    k = (fmt.key, _stream(stream))
    ws = per.get(k)
    if ws is None or ws.max_batch < B:
        ws = per[k] = DecodeWorkspace(pool, fmt, B, stream)
    return ws


def paged_decode(pool: SlabPool, fmt: KvFormat, layer: int, q: torch.Tensor,
                 block_table: torch.Tensor, ctx_lens: torch.Tensor,
                 out: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                 sm_scale: Optional[float] = None, kv_scales: Optional[torch.Tensor] = None,
                 workspace: Optional[DecodeWorkspace] = None, stream=None,
                 k_new: Optional[torch.Tensor] = None,
                 v_new: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K2: O = softmax(sm_scale * Q K^T) V over each sequence's slab blocks.

    q: fp16 [B, Hq, d]; block_table: int32 [B, max_blocks] of global block
    ids; ctx_lens: int32 [B] (device).  With k_new/v_new (fp16 [B, Hkv, d])
    the new token at position ctx_lens-1 is appended first (fused K1).
    Returns out fp16 [B, Hq, d]."""
    assert q.dtype == torch.float16 and q.is_contiguous()
    assert block_table.dtype == torch.int32 and ctx_lens.dtype == torch.int32
    B = q.shape[0]
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = _default_decode_ws(pool, fmt, B, stream)
    f = fmt.c_ref()
    scale = 0.0 if sm_scale is None else float(sm_scale)
    if k_new is None:
        check(L.lib.ks_paged_decode(pool.handle, f, layer, _ptr(q), _ptr(out), _ptr(lse),
                                    _ptr(block_table), block_table.stride(0), _ptr(ctx_lens), B,
                                    scale, _ptr(kv_scales), _ptr(workspace.buf), workspace.nbytes,
                                    _stream(stream)))
    else:
        assert k_new.dtype == torch.float16 and k_new.is_contiguous() and v_new.is_contiguous()
        check(L.lib.ks_paged_decode_append(pool.handle, f, layer, _ptr(q), _ptr(k_new),
                                           _ptr(v_new), _ptr(out), _ptr(lse), _ptr(block_table),
                                           block_table.stride(0), _ptr(ctx_lens), B, scale,
                                           _ptr(kv_scales), _ptr(workspace.buf), workspace.nbytes,
                                           _stream(stream)))
    return out


PREFILL_WS_CAP = int(os.environ.get("KVSLAB_PREFILL_WS_CAP", 1 << 30))


def prefill_workspace(pool: SlabPool, fmt: KvFormat, batch: int, bt_stride: int,
                      max_q_len: int, stream=None) -> Optional[torch.Tensor]:
    """K4 workspace (split-KV partials + the quantised formats' expand
    scratch; None when neither applies): one buffer per (pool, stream), grown
    on demand up to PREFILL_WS_CAP bytes (beyond, the C side drops the split
    and takes the expand in sequence groups) and reused by every call on that
    stream.  A grown buffer replaces the old one through the caching
    allocator, which orders the old one's reuse after that stream's kernels."""
    f = fmt.to_c()
    n, one = C.c_size_t(), C.c_size_t()
    check(L.lib.ks_paged_prefill_workspace_size(C.byref(f), batch, bt_stride, max_q_len, C.byref(n)))
    check(L.lib.ks_paged_prefill_workspace_size(C.byref(f), 1, bt_stride, max_q_len, C.byref(one)))
    if n.value == 0:
        return None
    want = max(min(n.value, PREFILL_WS_CAP), one.value)
    per = _pool_cache(pool, "_ks_prefill_ws")
    sk = _stream(stream)
    buf = per.get(sk)
    if buf is None or buf.numel() < want:
        with torch.cuda.stream(_torch_stream(stream, pool.device)):
            buf = torch.empty(want, dtype=torch.uint8, device=f"cuda:{pool.device}")
        per[sk] = buf
    return buf


def paged_prefill(pool: SlabPool, fmt: KvFormat, layer: int, q: torch.Tensor,
                  block_table: torch.Tensor, cu_q: torch.Tensor, ctx_lens: torch.Tensor,
                  max_q_len: int, out: Optional[torch.Tensor] = None,
                  lse: Optional[torch.Tensor] = None, sm_scale: Optional[float] = None,
                  kv_scales: Optional[torch.Tensor] = None, stream=None,
                  workspace="auto") -> torch.Tensor:
    """K4: causal chunked-prefill attention over slab blocks.

    q: fp16 [T, Hq, d], the rows of sequence s being cu_q[s]..cu_q[s+1]-1
    (int32 [B+1], device) at positions ctx_lens[s]-n_s..ctx_lens[s]-1 (int32
    [B], device; the chunk's K/V already appended with kv_append).  Each query
    attends keys 0..its position.  max_q_len >= every n_s.  Returns out fp16
    [T, Hq, d].  workspace: "auto" (the cached expand scratch of quantised
    formats, see ks_paged_prefill_ws), a uint8 device tensor, or None (the
    direct quantised kernel)."""
    assert q.dtype == torch.float16 and q.is_contiguous()
    assert block_table.dtype == torch.int32 and ctx_lens.dtype == torch.int32
    assert cu_q.dtype == torch.int32
    if out is None:
        out = torch.empty_like(q)
    f = fmt.to_c()
    scale = 0.0 if sm_scale is None else float(sm_scale)
    if isinstance(workspace, str):
        workspace = prefill_workspace(pool, fmt, ctx_lens.shape[0], block_table.stride(0), int(max_q_len),
                                      stream)
    ws_bytes = 0 if workspace is None else workspace.numel()
    check(L.lib.ks_paged_prefill_ws(pool.handle, C.byref(f), layer, _ptr(q), _ptr(out), _ptr(lse),
                                    _ptr(block_table), block_table.stride(0), _ptr(cu_q),
                                    _ptr(ctx_lens), ctx_lens.shape[0], int(max_q_len), scale,
                                    _ptr(kv_scales), _ptr(workspace), ws_bytes, _stream(stream)))
    return out


def compact_key(pool: SlabPool, key: int, max_moves: int = 1 << 30, stream=None) -> Tuple[int, int]:
    """K3 as one transaction (ks_compact): plan, move the bytes on the GPU and
    rewrite every registered engine table of `key` (engine.SlabModel).
    Returns (moves, slabs_freed)."""
    n, freed = C.c_uint32(), C.c_uint32()
    check(L.lib.ks_compact(pool.handle, key, min(int(max_moves), 0xFFFFFFFF), _stream(stream),
                           C.byref(n), C.byref(freed)))
    return n.value, freed.value


def compact(pool: SlabPool, key: int, max_moves: int = 1 << 20,
            tables: Sequence[torch.Tensor] = (), stream=None) -> Tuple[List[Tuple[int, int]], int]:
    """K3 for engine-owned raw tables: plan (host, applied to the slab
    table), move the bytes on the GPU, and remap the given device block
    tables.  Returns (moves, slabs_freed).  Registered tables (SlabModel) use
    compact_key, which also rolls back on failure."""
    moves, freed = pool.plan_compaction(key, max_moves)
    if moves:
        buf = (L.ks_block_move * len(moves))(*[L.ks_block_move(s, d) for s, d in moves])
        check(L.lib.ks_compact_apply(pool.handle, key, buf, len(moves), _stream(stream)))
        for t in tables:
            check(L.lib.ks_block_table_remap(pool.handle, _ptr(t), t.numel(), buf, len(moves),
                                             _stream(stream)))
    return moves, freed


def set_decode_sm_share(pool: SlabPool, key: int, max_ctas: int) -> None:
    """Cap the K2 grid of the model with this slab key (MPS-style SM share)."""
    check(L.lib.ks_set_decode_sm_share(pool.handle, key, max_ctas))


def launch_count() -> int:
    return L.lib.ks_launch_count()


def default_sm_scale(head_dim: int) -> float:
    return 1.0 / math.sqrt(head_dim)

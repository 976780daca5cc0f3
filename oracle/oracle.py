"""ctypes wrapper of oracle/build/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / timed CPU baseline.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libslabsim_ref.so")


def _load():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return C.CDLL(LIB)


lib = _load()


class orc_rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class orc_handle(C.Structure):
    _fields_ = [("slab_id", C.c_uint32), ("local_block_id", C.c_uint32),
                ("global_block_id", C.c_uint64), ("key", C.c_uint64)]


class orc_fmt(C.Structure):
    _fields_ = [("kv_dtype", C.c_uint32), ("num_kv_heads", C.c_uint32),
                ("num_q_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("num_layers", C.c_uint32), ("tokens_per_block", C.c_uint32),
                ("qparams", C.c_uint64)]


P = C.c_void_p
_u64p = C.POINTER(C.c_uint64)
lib.orc_rng_seed.argtypes = [C.POINTER(orc_rng), C.c_uint64]
lib.orc_rng_fill_uniform.argtypes = [C.POINTER(orc_rng), P, C.c_size_t]
lib.orc_token_size.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _u64p]
lib.orc_kv_block_size.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64,
                                  C.c_uint64, C.c_uint32, _u64p]
lib.orc_pool_create.argtypes = [C.c_uint64, C.c_uint64, _u64p, C.c_uint32, C.c_int,
                                C.POINTER(P)]
lib.orc_pool_destroy.argtypes = [P]
lib.orc_pool_alloc.argtypes = [P, C.c_uint64, C.POINTER(orc_handle)]
lib.orc_pool_free.argtypes = [P, C.POINTER(orc_handle)]
lib.orc_pool_stats.argtypes = [P, _u64p]
lib.orc_pool_slab_count.argtypes = [P]
lib.orc_pool_slab_count.restype = C.c_uint32
lib.orc_pool_slab.argtypes = [P, C.c_uint32, C.POINTER(C.c_int), _u64p, C.POINTER(C.c_uint32),
                              C.POINTER(C.c_uint32)]
lib.orc_compact_plan.argtypes = [P, C.c_uint64, C.c_uint32, _u64p, _u64p,
                                 C.POINTER(C.c_uint32)]
lib.orc_compact_plan.restype = C.c_uint32
lib.orc_f32_to_e4m3.argtypes = [C.c_float]
lib.orc_f32_to_e4m3.restype = C.c_uint8
lib.orc_e4m3_to_f32.argtypes = [C.c_uint8]
lib.orc_e4m3_to_f32.restype = C.c_float
lib.orc_f32_to_f16.argtypes = [C.c_float]
lib.orc_f32_to_f16.restype = C.c_uint16
lib.orc_swz.argtypes = [C.c_uint64]
lib.orc_swz.restype = C.c_uint64
lib.orc_append.argtypes = [P, C.c_uint64, C.c_uint64, C.POINTER(orc_fmt), C.c_uint32, P, P,
                           C.c_uint32, P, P, P, C.c_uint32, P]
lib.orc_paged_decode.argtypes = [P, C.c_uint64, C.c_uint64, C.POINTER(orc_fmt), C.c_uint32, P,
                                 P, C.c_uint32, P, C.c_uint32, C.c_double, P, P, P, C.c_int]
lib.orc_paged_prefill.argtypes = [P, C.c_uint64, C.c_uint64, C.POINTER(orc_fmt), C.c_uint32, P,
                                  P, C.c_uint32, P, P, C.c_uint32, C.c_double, P, P, P, C.c_int]
lib.orc_decode_bytes.argtypes = [C.POINTER(orc_fmt), P, C.c_uint32]
lib.orc_decode_bytes.restype = C.c_uint64
for _n in ("orc_fmt_token_size", "orc_fmt_chunk_bytes", "orc_fmt_layer_bytes", "orc_fmt_key",
           "orc_fmt_natural_qparams"):
    getattr(lib, _n).argtypes = [C.POINTER(orc_fmt)]
    getattr(lib, _n).restype = C.c_uint64

NPROC = os.cpu_count() or 1


def _p(a):
    return None if a is None else a.ctypes.data


def uniforms(seed: int, n: int) -> np.ndarray:
    r = orc_rng()
    lib.orc_rng_seed(C.byref(r), seed)
    out = np.empty(n, dtype=np.float64)
    lib.orc_rng_fill_uniform(C.byref(r), out.ctypes.data, n)
    return out


def fmt(kv_dtype, num_kv_heads, num_q_heads, head_dim=128, num_layers=1, tpb=16, qparams=None):
    f = orc_fmt(int(kv_dtype), num_kv_heads, num_q_heads, head_dim, num_layers, tpb, 0)
    f.qparams = lib.orc_fmt_natural_qparams(C.byref(f)) if qparams is None else qparams
    return f


def append(pool_bytes: np.ndarray, slab_size, bps, f, layer, k16, v16, tok_seq, tok_pos, table,
           kv_scales=None):
    """k16/v16: uint16 [n, H, d] (fp16 bits); pool_bytes: uint8 host image."""
    k16 = np.ascontiguousarray(k16, dtype=np.uint16)
    v16 = np.ascontiguousarray(v16, dtype=np.uint16)
    ts = np.ascontiguousarray(tok_seq, dtype=np.int32)
    tp = np.ascontiguousarray(tok_pos, dtype=np.int32)
    tb = np.ascontiguousarray(table, dtype=np.int32)
    sc = None if kv_scales is None else np.ascontiguousarray(kv_scales, dtype=np.float32)
    lib.orc_append(pool_bytes.ctypes.data, slab_size, bps, C.byref(f), layer, k16.ctypes.data,
                   v16.ctypes.data, k16.shape[0], ts.ctypes.data, tp.ctypes.data, tb.ctypes.data,
                   tb.shape[1], _p(sc))


def paged_decode(pool_bytes, slab_size, bps, f, layer, q16, table, ctx_lens, sm_scale,
                 kv_scales=None, nthreads=1):
    q16 = np.ascontiguousarray(q16, dtype=np.uint16)
    tb = np.ascontiguousarray(table, dtype=np.int32)
    cl = np.ascontiguousarray(ctx_lens, dtype=np.int32)
    sc = None if kv_scales is None else np.ascontiguousarray(kv_scales, dtype=np.float32)
    B = q16.shape[0]
    out = np.zeros(q16.shape, dtype=np.float64)
    lse = np.zeros(q16.shape[:2], dtype=np.float64)
    lib.orc_paged_decode(pool_bytes.ctypes.data, slab_size, bps, C.byref(f), layer,
                         q16.ctypes.data, tb.ctypes.data, tb.shape[1], cl.ctypes.data, B,
                         sm_scale, _p(sc), out.ctypes.data, lse.ctypes.data, nthreads)
    return out, lse


def paged_prefill(pool_bytes, slab_size, bps, f, layer, q16, table, cu_q, ctx_lens, sm_scale,
                  kv_scales=None, nthreads=1):
    """Causal chunked-prefill attention (fp64): q16 [T_total, Hq, d] as uint16."""
    q16 = np.ascontiguousarray(q16, dtype=np.uint16)
    tb = np.ascontiguousarray(table, dtype=np.int32)
    cq = np.ascontiguousarray(cu_q, dtype=np.int32)
    cl = np.ascontiguousarray(ctx_lens, dtype=np.int32)
    sc = None if kv_scales is None else np.ascontiguousarray(kv_scales, dtype=np.float32)
    out = np.zeros(q16.shape, dtype=np.float64)
    lse = np.zeros(q16.shape[:2], dtype=np.float64)
    lib.orc_paged_prefill(pool_bytes.ctypes.data, slab_size, bps, C.byref(f), layer,
                          q16.ctypes.data, tb.ctypes.data, tb.shape[1], cq.ctypes.data,
                          cl.ctypes.data, cl.shape[0], sm_scale, _p(sc), out.ctypes.data,
                          lse.ctypes.data, nthreads)
    return out, lse


def decode_bytes(f, ctx_lens) -> int:
    cl = np.ascontiguousarray(ctx_lens, dtype=np.int32)
    return lib.orc_decode_bytes(C.byref(f), cl.ctypes.data, cl.shape[0])


class OraclePool:
    """Restated allocator (slab_pool.cpp) -- an independent second opinion."""

    def __init__(self, capacity, slab, keys, lcm=True):
        self.h = P()
        arr = (C.c_uint64 * len(keys))(*keys)
        self.status = lib.orc_pool_create(capacity, slab, arr, len(keys), 1 if lcm else 0,
                                          C.byref(self.h))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib.orc_pool_destroy(self.h)

    def alloc(self, key):
        h = orc_handle()
        st = lib.orc_pool_alloc(self.h, key, C.byref(h))
        return st, (h.slab_id, h.local_block_id, h.global_block_id, h.key)

    def free(self, hv):
        h = orc_handle(*hv)
        return lib.orc_pool_free(self.h, C.byref(h))

    def stats(self):
        out = (C.c_uint64 * 4)()
        lib.orc_pool_stats(self.h, out)
        return tuple(out)

    def compact(self, key, max_moves):
        src = (C.c_uint64 * max(1, max_moves))()
        dst = (C.c_uint64 * max(1, max_moves))()
        freed = C.c_uint32()
        n = lib.orc_compact_plan(self.h, key, max_moves, src, dst, C.byref(freed))
        return [(src[i], dst[i]) for i in range(n)], freed.value


def ref_lib():
    """oracle/_ref/libslabsim_ref.so -- the reference allocator itself (None if absent)."""
    if not os.path.exists(REF_LIB):
        return None
    L = C.CDLL(REF_LIB)
    L.ref_pool_create.argtypes = [C.c_uint64, C.c_uint64, _u64p, C.c_uint32, C.c_int]
    L.ref_pool_create.restype = P
    L.ref_pool_destroy.argtypes = [P]
    L.ref_try_alloc.argtypes = [P, C.c_uint64, _u64p]
    L.ref_free.argtypes = [P, _u64p]
    L.ref_stats.argtypes = [P, _u64p]
    L.ref_bench_churn.argtypes = [C.c_int, C.c_uint64]
    L.ref_bench_churn.restype = C.c_double
    return L

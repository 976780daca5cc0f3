"""ctypes binding of libkvslab.so (the C ABI declared in include/kvslab.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2509_06261_b200/csrc``).  There is no fallback: if the
shared object is missing, importing this module raises ImportError.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVSLAB_LIB_PATH") or os.path.join(_HERE, "libkvslab.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libkvslab.so not found at {LIB_PATH}; build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

lib = C.CDLL(LIB_PATH)

KS_OK, KS_INVALID_CONFIG, KS_INVALID_KEY, KS_EXHAUSTED, KS_INVALID_FREE = 0, 1, 2, 3, 4
KS_INVALID_PROFILE, KS_INVALID_ARGUMENT, KS_CUDA_ERROR, KS_NOT_SUPPORTED, KS_INTERNAL = 5, 6, 7, 8, 9


class ks_pool_config(C.Structure):
    _fields_ = [("capacity_bytes", C.c_uint64), ("slab_size_bytes", C.c_uint64),
                ("block_size_keys", C.POINTER(C.c_uint64)), ("num_keys", C.c_uint32),
                ("require_lcm_alignment", C.c_int32)]


class ks_block_handle(C.Structure):
    _fields_ = [("slab_id", C.c_uint32), ("local_block_id", C.c_uint32),
                ("global_block_id", C.c_uint64), ("key", C.c_uint64)]


class ks_frag_stats(C.Structure):
    _fields_ = [("allocated_bytes", C.c_uint64), ("free_block_bytes", C.c_uint64),
                ("slab_residue_bytes", C.c_uint64), ("free_slab_bytes", C.c_uint64)]


class ks_op_record(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("time", C.c_double), ("op", C.c_char_p),
                ("key", C.c_uint64), ("slab_id", C.c_uint32), ("local_block_id", C.c_uint32),
                ("global_block_id", C.c_uint64)]


class ks_pool_info(C.Structure):
    _fields_ = [("slab_count", C.c_uint32), ("num_keys", C.c_uint32),
                ("slab_size_bytes", C.c_uint64), ("tail_remainder_bytes", C.c_uint64),
                ("usable_capacity_bytes", C.c_uint64), ("allocated_blocks", C.c_uint64),
                ("device", C.c_int32), ("require_lcm_alignment", C.c_int32)]


class ks_model_geometry(C.Structure):
    _fields_ = [("num_kv_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("num_layers", C.c_uint32), ("tp_degree", C.c_uint32),
                ("tokens_per_block", C.c_uint64), ("quant_param_bytes_per_block", C.c_uint64),
                ("kv_bits", C.c_int32)]


class ks_kv_format(C.Structure):
    _fields_ = [("kv_dtype", C.c_uint32), ("num_kv_heads", C.c_uint32),
                ("num_q_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("num_layers", C.c_uint32), ("tokens_per_block", C.c_uint32),
                ("quant_param_bytes_per_block", C.c_uint64)]


class ks_block_move(C.Structure):
    _fields_ = [("src_global_block_id", C.c_uint64), ("dst_global_block_id", C.c_uint64)]


class ks_seq_table_config(C.Structure):
    _fields_ = [("key", C.c_uint64), ("max_seqs", C.c_uint32), ("max_blocks_per_seq", C.c_uint32),
                ("tokens_per_block", C.c_uint32), ("reserved", C.c_uint32),
                ("useful_token_bytes", C.c_uint64), ("block_metadata_bytes", C.c_uint64),
                ("d_table", C.c_void_p), ("row_stride", C.c_uint32)]


class ks_seq_table_stats(C.Structure):
    _fields_ = [("live_seqs", C.c_uint32), ("held_blocks", C.c_uint64),
                ("cached_tokens", C.c_uint64), ("internal_frag_bytes", C.c_uint64)]


OP_LOG_FN = C.CFUNCTYPE(None, C.POINTER(ks_op_record), C.c_void_p)
CLOCK_FN = C.CFUNCTYPE(C.c_double, C.c_void_p)

P = C.c_void_p
u32, u64, i32, st = C.c_uint32, C.c_uint64, C.c_int32, C.c_int
pu32, pu64, pi32 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int32)

_SIGS = {
    "ks_abi_version": (u32, []),
    "ks_last_error": (C.c_char_p, []),
    "ks_status_name": (C.c_char_p, [st]),
    "ks_launch_count": (u64, []),
    "ks_token_size": (st, [C.POINTER(ks_model_geometry), pu64]),
    "ks_kv_block_size": (st, [C.POINTER(ks_model_geometry), pu64]),
    "ks_pool_create": (st, [C.POINTER(ks_pool_config), C.c_int, C.POINTER(P)]),
    "ks_pool_destroy": (st, [P]),
    "ks_pool_get_info": (st, [P, C.POINTER(ks_pool_info)]),
    "ks_pool_keys": (st, [P, pu64, u32]),
    "ks_pool_scrubbed_bytes": (st, [P, pu64]),
    "ks_alloc_block": (st, [P, u64, C.POINTER(ks_block_handle)]),
    "ks_try_alloc_block": (st, [P, u64, C.POINTER(ks_block_handle), pi32]),
    "ks_alloc_blocks": (st, [P, u64, u32, C.POINTER(ks_block_handle), pu32]),
    "ks_free_block": (st, [P, C.POINTER(ks_block_handle)]),
    "ks_free_blocks": (st, [P, C.POINTER(ks_block_handle), u32]),
    "ks_blocks_per_slab": (st, [P, u64, pu64]),
    "ks_snapshot_stats": (st, [P, C.POINTER(ks_frag_stats)]),
    "ks_free_blocks_for_key": (st, [P, u64, pu64]),
    "ks_allocated_block_count": (st, [P, u64, pu64]),
    "ks_slab_state": (st, [P, u32, pi32, pu64]),
    "ks_check_integrity": (st, [P, pi32]),
    "ks_pool_equal": (st, [P, P, pi32]),
    "ks_pool_clone_host": (st, [P, C.POINTER(P)]),
    "ks_set_op_log": (st, [P, OP_LOG_FN, P]),
    "ks_set_clock": (st, [P, CLOCK_FN, P]),
    "ks_debug_flip_occupancy_bit": (st, [P, u32, u32]),
    "ks_global_block_id": (u64, [u32, u32, u64]),
    "ks_split_global_block_id": (None, [u64, u64, pu32, pu32]),
    "ks_block_byte_offset": (st, [P, u64, u64, pu64]),
    "ks_natural_qparams": (st, [C.POINTER(ks_kv_format), pu64]),
    "ks_format_key": (st, [C.POINTER(ks_kv_format), pu64]),
    "ks_validate_format": (st, [P, C.POINTER(ks_kv_format)]),
    "ks_device_base": (st, [P, C.POINTER(P), pu64]),
    "ks_slab_table_device": (st, [P, C.POINTER(P)]),
    "ks_slab_table_sync": (st, [P, P]),
    "ks_block_table_update": (st, [P, P, u32, pi32, pi32, pi32, u32, P]),
    "ks_block_table_validate": (st, [P, u64, P, u32, P, u32, u32, P, pu64]),
    "ks_kv_append": (st, [P, C.POINTER(ks_kv_format), u32, P, P, u32, P, P, P, u32, P, P]),
    "ks_paged_decode_workspace_size": (st, [P, C.POINTER(ks_kv_format), u32, C.POINTER(C.c_size_t)]),
    "ks_paged_decode": (st, [P, C.POINTER(ks_kv_format), u32, P, P, P, P, u32, P, u32,
                             C.c_float, P, P, C.c_size_t, P]),
    "ks_paged_decode_append": (st, [P, C.POINTER(ks_kv_format), u32, P, P, P, P, P, P, u32, P,
                                    u32, C.c_float, P, P, C.c_size_t, P]),
    "ks_paged_prefill": (st, [P, C.POINTER(ks_kv_format), u32, P, P, P, P, u32, P, P, u32, u32,
                              C.c_float, P, P]),
    "ks_paged_prefill_workspace_size": (st, [C.POINTER(ks_kv_format), u32, u32, u32, C.POINTER(C.c_size_t)]),
    "ks_paged_prefill_ws": (st, [P, C.POINTER(ks_kv_format), u32, P, P, P, P, u32, P, P, u32, u32,
                                 C.c_float, P, P, C.c_size_t, P]),
    "ks_set_decode_sm_share": (st, [P, u64, u32]),
    "ks_probe_set_decode_trace": (st, [P, P]),
    "ks_compact_plan": (st, [P, u64, u32, C.POINTER(ks_block_move), pu32, pu32]),
    "ks_compact_apply": (st, [P, u64, C.POINTER(ks_block_move), u32, P]),
    "ks_block_table_remap": (st, [P, P, u64, C.POINTER(ks_block_move), u32, P]),
    "ks_seq_table_create": (st, [P, C.POINTER(ks_seq_table_config), C.POINTER(P)]),
    "ks_seq_table_destroy": (st, [P]),
    "ks_seq_table_admit": (st, [P, u32, u64, pi32]),
    "ks_seq_table_ensure": (st, [P, u32, u64, pi32]),
    "ks_seq_table_step": (st, [P, pu32, u32, C.POINTER(C.c_uint8), pu32]),
    "ks_seq_table_release": (st, [P, u32]),
    "ks_seq_table_move_row": (st, [P, u32, u32]),
    "ks_seq_table_cached": (st, [P, u32, pu64]),
    "ks_seq_table_set_cached": (st, [P, u32, u64]),
    "ks_seq_table_ctx_lens": (st, [P, pi32, u32, i32]),
    "ks_seq_table_blocks": (st, [P, u32, C.POINTER(ks_block_handle), u32, pu32]),
    "ks_seq_table_get_stats": (st, [P, C.POINTER(ks_seq_table_stats)]),
    "ks_seq_table_pending": (st, [P, pu32]),
    "ks_seq_table_sync": (st, [P, P]),
    "ks_compact": (st, [P, u64, u32, P, pu32, pu32]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error() -> str:
    return lib.ks_last_error().decode(errors="replace")

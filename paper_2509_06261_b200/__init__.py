"""B200-native KV-slab data path (FineServe, arxiv 2509.06261).

Host API mirrors the reference allocator (slabsim::SlabPool); the device path
(KV append, slab-indexed paged decode, compaction) runs as sm_100a CUDA
kernels in libkvslab.so.  See DESIGN.md.
"""
from . import _lib  # noqa: F401  (fails loudly when libkvslab.so is missing)
from .slab_pool import (BlockHandle, Error, FragmentationStats, InvalidConfigError,
                        InvalidFreeError, InvalidKeyError, InvalidProfileError, KvSlabError,
                        OpLogRecord, PoolExhaustedError, SlabPool, SlabPoolConfig, SlabState,
                        kv_block_size, token_size, write_op_log_line)

__all__ = [
    "BlockHandle", "Error", "FragmentationStats", "InvalidConfigError", "InvalidFreeError",
    "InvalidKeyError", "InvalidProfileError", "KvSlabError", "OpLogRecord",
    "PoolExhaustedError", "SlabPool", "SlabPoolConfig", "SlabState", "kv_block_size",
    "token_size", "write_op_log_line",
]

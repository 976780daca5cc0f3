"""Python mirror of the reference allocator API over the C ABI.

Same class names, method names, argument meaning and exceptions as
``slabsim::SlabPool`` (reference: proj/core/include/slabsim/slab_pool.hpp:
30-202, common.hpp:31-59), so parity tests read like the reference's own
tests (proj/tests/test_slab_pool.cpp).  Every call goes through
libkvslab.so; nothing here re-implements allocation.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

from . import _lib as L


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """slabsim::Error (common.hpp:31-34)."""


class InvalidConfigError(Error):
    pass


class InvalidKeyError(Error):
    pass


class InvalidFreeError(Error):
    pass


class PoolExhaustedError(Error):
    pass


class InvalidProfileError(Error):
    pass


class KvSlabError(Error):
    """Non-reference failures: bad arguments, CUDA errors, unsupported shapes."""


_STATUS_EXC = {
    L.KS_INVALID_CONFIG: InvalidConfigError,
    L.KS_INVALID_KEY: InvalidKeyError,
    L.KS_EXHAUSTED: PoolExhaustedError,
    L.KS_INVALID_FREE: InvalidFreeError,
    L.KS_INVALID_PROFILE: InvalidProfileError,
}


def check(status: int) -> None:
    if status != L.KS_OK:
        name = L.lib.ks_status_name(status).decode()
        raise _STATUS_EXC.get(status, KvSlabError)(f"{name}: {L.last_error()}")


# ------------------------------------------------------------------ values
class SlabState(enum.IntEnum):
    FREE = 0
    PARTIAL = 1
    FULL = 2


@dataclass
class SlabPoolConfig:
    """slabsim::SlabPoolConfig (slab_pool.hpp:41-46)."""
    capacity_bytes: int = 0
    slab_size_bytes: int = 0
    block_size_keys: List[int] = field(default_factory=list)
    require_lcm_alignment: bool = True


@dataclass(frozen=True)
class BlockHandle:
    """slabsim::BlockHandle (slab_pool.hpp:53-60)."""
    slab_id: int = 0
    local_block_id: int = 0
    global_block_id: int = 0
    key: int = 0

    def to_c(self) -> L.ks_block_handle:
        return L.ks_block_handle(self.slab_id, self.local_block_id, self.global_block_id, self.key)

    @staticmethod
    def from_c(h: L.ks_block_handle) -> "BlockHandle":
        return BlockHandle(h.slab_id, h.local_block_id, h.global_block_id, h.key)


@dataclass(frozen=True)
class FragmentationStats:
    """slabsim::FragmentationStats (slab_pool.hpp:67-78)."""
    allocated_bytes: int = 0
    free_block_bytes: int = 0
    slab_residue_bytes: int = 0
    free_slab_bytes: int = 0

    def usable_capacity(self) -> int:
        return (self.allocated_bytes + self.free_block_bytes + self.slab_residue_bytes +
                self.free_slab_bytes)

    def as_tuple(self) -> Tuple[int, int, int, int]:
        return (self.allocated_bytes, self.free_block_bytes, self.slab_residue_bytes,
                self.free_slab_bytes)


@dataclass(frozen=True)
class OpLogRecord:
    """slabsim::OpLogRecord (slab_pool.hpp:80-89)."""
    seq: int
    time: float
    op: str
    key: int
    slab_id: int
    local_block_id: int
    global_block_id: int


def write_op_log_line(rec: OpLogRecord) -> str:
    """slab_pool.cpp:45-49 line format."""
    return (f"{rec.seq} {rec.time:g} {rec.op} {rec.key} {rec.slab_id} {rec.local_block_id} "
            f"{rec.global_block_id}\n")


# ------------------------------------------------------------------ geometry
def token_size(num_kv_heads: int, head_dim: int, kv_bits: int, tp_degree: int = 1) -> int:
    """precision.cpp:76-89."""
    g = L.ks_model_geometry(num_kv_heads, head_dim, 1, tp_degree, 16, 0, kv_bits)
    out = C.c_uint64()
    check(L.lib.ks_token_size(C.byref(g), C.byref(out)))
    return out.value


def kv_block_size(num_kv_heads: int, head_dim: int, kv_bits: int, num_layers: int = 1,
                  tokens_per_block: int = 16, quant_param_bytes_per_block: int = 0,
                  tp_degree: int = 1) -> int:
    """precision.cpp:91-99 -- the slab key of a model."""
    g = L.ks_model_geometry(num_kv_heads, head_dim, num_layers, tp_degree, tokens_per_block,
                            quant_param_bytes_per_block, kv_bits)
    out = C.c_uint64()
    check(L.lib.ks_kv_block_size(C.byref(g), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ pool
class SlabPool:
    """slabsim::SlabPool (slab_pool.hpp:101-202) backed by libkvslab.so.

    ``device`` (int) additionally reserves the pool's single KV tensor on that
    CUDA device; ``None`` builds a host-only pool (the allocator alone).
    """

    def __init__(self, config: SlabPoolConfig, device: Optional[int] = None,
                 _handle: Optional[int] = None):
        self._h = C.c_void_p()
        self._log_cb = None
        self._clock_cb = None
        if _handle is not None:
            self._h = C.c_void_p(_handle)
        else:
            keys = (C.c_uint64 * max(1, len(config.block_size_keys)))(*config.block_size_keys)
            cfg = L.ks_pool_config(config.capacity_bytes, config.slab_size_bytes, keys,
                                   len(config.block_size_keys),
                                   1 if config.require_lcm_alignment else 0)
            check(L.lib.ks_pool_create(C.byref(cfg), -1 if device is None else int(device),
                                       C.byref(self._h)))
        info = self._info()
        self.device = None if info.device < 0 else info.device
        kbuf = (C.c_uint64 * info.num_keys)()
        check(L.lib.ks_pool_keys(self._h, kbuf, info.num_keys))
        self._config = SlabPoolConfig(config.capacity_bytes if config else 0,
                                      info.slab_size_bytes, list(kbuf),
                                      bool(info.require_lcm_alignment))

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(L, "lib", None)  # None during interpreter shutdown
        if h is not None and h.value and lib is not None:
            lib.ks_pool_destroy(h)
            self._h = C.c_void_p()

    def close(self) -> None:
        self.__del__()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def _info(self) -> L.ks_pool_info:
        info = L.ks_pool_info()
        check(L.lib.ks_pool_get_info(self._h, C.byref(info)))
        return info

    # -- allocation (slab_pool.cpp:193-272) --
    def alloc_block(self, key: int) -> BlockHandle:
        h = L.ks_block_handle()
        check(L.lib.ks_alloc_block(self._h, key, C.byref(h)))
        return BlockHandle.from_c(h)

    def try_alloc_block(self, key: int) -> Optional[BlockHandle]:
        h = L.ks_block_handle()
        ok = C.c_int32()
        check(L.lib.ks_try_alloc_block(self._h, key, C.byref(h), C.byref(ok)))
        return BlockHandle.from_c(h) if ok.value else None

    def alloc_blocks(self, key: int, n: int) -> List[BlockHandle]:
        """Batched try-alloc; returns the handles that could be allocated."""
        buf = (L.ks_block_handle * max(1, n))()
        done = C.c_uint32()
        check(L.lib.ks_alloc_blocks(self._h, key, n, buf, C.byref(done)))
        return [BlockHandle.from_c(buf[i]) for i in range(done.value)]

    def free_block(self, handle: BlockHandle) -> None:
        h = handle.to_c()
        check(L.lib.ks_free_block(self._h, C.byref(h)))

    def free_blocks(self, handles: Sequence[BlockHandle]) -> None:
        buf = (L.ks_block_handle * max(1, len(handles)))(*[h.to_c() for h in handles])
        check(L.lib.ks_free_blocks(self._h, buf, len(handles)))

    # -- queries --
    def blocks_per_slab(self, key: int) -> int:
        out = C.c_uint64()
        check(L.lib.ks_blocks_per_slab(self._h, key, C.byref(out)))
        return out.value

    def snapshot_stats(self) -> FragmentationStats:
        s = L.ks_frag_stats()
        check(L.lib.ks_snapshot_stats(self._h, C.byref(s)))
        return FragmentationStats(s.allocated_bytes, s.free_block_bytes, s.slab_residue_bytes,
                                  s.free_slab_bytes)

    @property
    def config(self) -> SlabPoolConfig:
        return self._config

    def slab_count(self) -> int:
        return self._info().slab_count

    def slab_size(self) -> int:
        return self._info().slab_size_bytes

    def tail_remainder_bytes(self) -> int:
        return self._info().tail_remainder_bytes

    def usable_capacity_bytes(self) -> int:
        return self._info().usable_capacity_bytes

    def slab_state(self, slab_id: int) -> SlabState:
        s, k = C.c_int32(), C.c_uint64()
        check(L.lib.ks_slab_state(self._h, slab_id, C.byref(s), C.byref(k)))
        return SlabState(s.value)

    def slab_key(self, slab_id: int) -> int:
        s, k = C.c_int32(), C.c_uint64()
        check(L.lib.ks_slab_state(self._h, slab_id, C.byref(s), C.byref(k)))
        return k.value

    def free_blocks_for_key(self, key: int) -> int:
        out = C.c_uint64()
        check(L.lib.ks_free_blocks_for_key(self._h, key, C.byref(out)))
        return out.value

    def allocated_block_count(self, key: Optional[int] = None) -> int:
        if key == 0:
            raise InvalidKeyError("block-size key 0 is not registered")
        out = C.c_uint64()
        check(L.lib.ks_allocated_block_count(self._h, 0 if key is None else key, C.byref(out)))
        return out.value

    @staticmethod
    def global_block_id(slab_id: int, local_block_id: int, blocks_per_slab: int) -> int:
        return L.lib.ks_global_block_id(slab_id, local_block_id, blocks_per_slab)

    @staticmethod
    def split_global_block_id(global_id: int, blocks_per_slab: int) -> Tuple[int, int]:
        s, l = C.c_uint32(), C.c_uint32()
        L.lib.ks_split_global_block_id(global_id, blocks_per_slab, C.byref(s), C.byref(l))
        return s.value, l.value

    def block_byte_offset(self, key: int, global_id: int) -> int:
        out = C.c_uint64()
        check(L.lib.ks_block_byte_offset(self._h, key, global_id, C.byref(out)))
        return out.value

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, SlabPool):
            return NotImplemented
        eq = C.c_int32()
        check(L.lib.ks_pool_equal(self._h, other._h, C.byref(eq)))
        return bool(eq.value)

    def clone_host(self) -> "SlabPool":
        """Deep copy of the host slab table (value semantics of the reference class)."""
        h = C.c_void_p()
        check(L.lib.ks_pool_clone_host(self._h, C.byref(h)))
        return SlabPool(self._config, _handle=h.value)

    def check_integrity(self) -> Tuple[bool, str]:
        ok = C.c_int32()
        check(L.lib.ks_check_integrity(self._h, C.byref(ok)))
        return bool(ok.value), ("" if ok.value else L.last_error())

    def set_op_log(self, sink: Optional[Callable[[OpLogRecord], None]]) -> None:
        if sink is None:
            self._log_cb = None
            check(L.lib.ks_set_op_log(self._h, C.cast(None, L.OP_LOG_FN), None))
            return

        def _cb(rec, _user):
            r = rec.contents
            sink(OpLogRecord(r.seq, r.time, r.op.decode(), r.key, r.slab_id, r.local_block_id,
                             r.global_block_id))

        self._log_cb = L.OP_LOG_FN(_cb)
        check(L.lib.ks_set_op_log(self._h, self._log_cb, None))

    def set_clock(self, clock: Optional[Callable[[], float]]) -> None:
        if clock is None:
            self._clock_cb = None
            check(L.lib.ks_set_clock(self._h, C.cast(None, L.CLOCK_FN), None))
            return
        self._clock_cb = L.CLOCK_FN(lambda _u: float(clock()))
        check(L.lib.ks_set_clock(self._h, self._clock_cb, None))

    def debug_flip_occupancy_bit(self, slab_id: int, local_block_id: int) -> None:
        check(L.lib.ks_debug_flip_occupancy_bit(self._h, slab_id, local_block_id))

    # -- compaction (new) --
    def plan_compaction(self, key: int, max_moves: int = 1 << 20) -> Tuple[List[Tuple[int, int]], int]:
        """Deterministic compaction plan for one key; applies it to the table.

        Returns ([(src_gid, dst_gid), ...], slabs_freed)."""
        buf = (L.ks_block_move * max(1, max_moves))()
        n, freed = C.c_uint32(), C.c_uint32()
        check(L.lib.ks_compact_plan(self._h, key, max_moves, buf, C.byref(n), C.byref(freed)))
        return [(buf[i].src_global_block_id, buf[i].dst_global_block_id)
                for i in range(n.value)], freed.value

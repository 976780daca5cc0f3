"""Caller-side block lifecycle of one co-located model over a shared pool.

Mirrors how the reference simulator's engines use the allocator
(proj/core/src/simulator.cpp): a per-sequence logical block table
(LiveRequest::blocks, :33-40), the prefill claim of ceil(prompt/tpb) blocks
with rollback (:500-526), decode growth need = ceil((cached+1)/tpb) with a
per-request stall (:561-578), release on completion (:621) and the
internal-fragmentation metric (:80-89).  The bookkeeping is native
(kvslab::SeqTable behind ks_seq_table_*); this class owns the int32 device
table the kernels read and forwards to the C ABI.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, List, Optional, Sequence

import torch

from . import _lib as L
from . import kv
from .kv import KvFormat
from .slab_pool import BlockHandle, SlabPool, check


class _Cached:
    """Sequence view of the table's cached-token counts (get / set by row)."""

    def __init__(self, m: "SlabModel"):
        self._m = m

    def __len__(self) -> int:
        return self._m.max_seqs

    def __getitem__(self, s: int) -> int:
        out = C.c_uint64()
        check(L.lib.ks_seq_table_cached(self._m._t, int(s), C.byref(out)))
        return out.value

    def __setitem__(self, s: int, tokens: int) -> None:
        check(L.lib.ks_seq_table_set_cached(self._m._t, int(s), int(tokens)))

    def __iter__(self):
        return (self[s] for s in range(len(self)))


class _Handles:
    """Read-only view of each row's BlockHandles in logical-block order."""

    def __init__(self, m: "SlabModel"):
        self._m = m

    def __len__(self) -> int:
        return self._m.max_seqs

    def __getitem__(self, s: int) -> List[BlockHandle]:
        cap = self._m.max_blocks
        buf = (L.ks_block_handle * cap)()
        n = C.c_uint32()
        check(L.lib.ks_seq_table_blocks(self._m._t, int(s), buf, cap, C.byref(n)))
        return [BlockHandle.from_c(buf[i]) for i in range(n.value)]

    def __iter__(self):
        return (self[s] for s in range(len(self)))


class SlabModel:
    def __init__(self, pool: SlabPool, fmt: KvFormat, max_seqs: int, max_blocks_per_seq: int):
        self.pool, self.fmt = pool, fmt
        self.key = fmt.key
        self.tpb = fmt.tokens_per_block
        self.max_seqs = max_seqs
        self.max_blocks = max_blocks_per_seq
        self.table: Optional[torch.Tensor] = None
        if pool.device is not None:
            self.table = torch.zeros((max_seqs, max_blocks_per_seq), dtype=torch.int32,
                                     device=f"cuda:{pool.device}")
        cfg = L.ks_seq_table_config(
            self.key, max_seqs, max_blocks_per_seq, self.tpb, 0,
            fmt.num_layers * fmt.token_size, fmt.num_layers * fmt.qparams,
            None if self.table is None else self.table.data_ptr(), max_blocks_per_seq)
        self._t = C.c_void_p()
        check(L.lib.ks_seq_table_create(pool.handle, C.byref(cfg), C.byref(self._t)))
        self.cached = _Cached(self)
        self.handles = _Handles(self)
        self._seq_buf = (C.c_uint32 * max_seqs)()
        self._stall_buf = (C.c_uint8 * max_seqs)()

    def __del__(self):
        t = getattr(self, "_t", None)
        lib = getattr(L, "lib", None)
        if t is not None and t.value and lib is not None:
            lib.ks_seq_table_destroy(t)
            self._t = C.c_void_p()

    # simulator.cpp:561-578 -- grow until ceil(tokens/tpb) blocks are held
    def ensure_capacity(self, seq: int, tokens: int) -> bool:
        ok = C.c_int32()
        check(L.lib.ks_seq_table_ensure(self._t, int(seq), int(tokens), C.byref(ok)))
        return bool(ok.value)

    # simulator.cpp:500-526 -- claim prompt blocks, roll back on failure
    def admit(self, seq: int, prompt_tokens: int) -> bool:
        ok = C.c_int32()
        check(L.lib.ks_seq_table_admit(self._t, int(seq), int(prompt_tokens), C.byref(ok)))
        return bool(ok.value)

    # simulator.cpp:561-578 + :609-612 -- one decode step of a batch
    def step(self, seqs: Sequence[int]) -> List[int]:
        """Grows every listed row for its next token and advances the ones
        that got their block; returns the rows that stalled."""
        n = len(seqs)
        for i, s in enumerate(seqs):
            self._seq_buf[i] = s
        act = C.c_uint32()
        check(L.lib.ks_seq_table_step(self._t, self._seq_buf, n, self._stall_buf, C.byref(act)))
        if act.value == n:
            return []
        return [seqs[i] for i in range(n) if self._stall_buf[i]]

    # simulator.cpp:621 / :583-596 -- completion or eviction
    def release(self, seq: int) -> None:
        check(L.lib.ks_seq_table_release(self._t, int(seq)))

    def move_row(self, src: int, dst: int) -> None:
        """Moves a sequence into an empty row (keeps a running batch packed)."""
        check(L.lib.ks_seq_table_move_row(self._t, int(src), int(dst)))

    def condense(self, live: Sequence[int]) -> List[int]:
        """Packs the given live rows into rows 0..len(live)-1 (row order kept
        where possible: rows already below the cut stay).  Returns, per new
        row, the old row it came from."""
        n = len(live)
        keep = sorted(s for s in live if s < n)
        movers = sorted(s for s in live if s >= n)
        holes = sorted(set(range(n)) - set(keep))
        src_of = {s: s for s in keep}
        for h, s in zip(holes, movers):
            self.move_row(s, h)
            src_of[h] = s
        return [src_of[i] for i in range(n)]

    def compact(self, max_moves: int = 1 << 20, stream=None):
        """K3 for this model's key (ks_compact): moves blocks out of the
        least-occupied slabs (freeing them for any key) and rewrites the
        handles and device tables of every model registered with this key.
        Returns (n_moves, slabs_freed)."""
        return kv.compact_key(self.pool, self.key, max_moves, stream)

    def sync(self, stream=None) -> int:
        """Uploads the table entries changed since the last sync; returns how many."""
        n = C.c_uint32()
        check(L.lib.ks_seq_table_pending(self._t, C.byref(n)))
        if n.value:
            check(L.lib.ks_seq_table_sync(self._t, kv._stream(stream) if self.table is not None else None))
        return n.value

    def stats(self) -> L.ks_seq_table_stats:
        st = L.ks_seq_table_stats()
        check(L.lib.ks_seq_table_get_stats(self._t, C.byref(st)))
        return st

    def internal_frag_bytes(self) -> int:
        """simulator.cpp:80-89: held*key - (cached*L*token_size + held*L*qparams)."""
        return self.stats().internal_frag_bytes

    def ctx_lens(self, n: Optional[int] = None, plus: int = 0) -> List[int]:
        """cached + plus per row (0 for rows holding no blocks), rows 0..n-1."""
        n = self.max_seqs if n is None else n
        buf = (C.c_int32 * n)()
        check(L.lib.ks_seq_table_ctx_lens(self._t, buf, n, int(plus)))
        return list(buf)

    def ctx_tensor(self, seqs: Optional[Iterable[int]] = None) -> torch.Tensor:
        seqs = range(self.max_seqs) if seqs is None else seqs
        return torch.tensor([self.cached[s] for s in seqs], dtype=torch.int32,
                            device=self.table.device)

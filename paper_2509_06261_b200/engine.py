"""Caller-side block lifecycle of one co-located model over a shared pool.

Mirrors how the reference simulator's engines use the allocator
(proj/core/src/simulator.cpp): a per-sequence logical block table
(LiveRequest::blocks, :33-40), the prefill claim of ceil(prompt/tpb) blocks
with rollback (:500-526), decode growth need = ceil((cached+1)/tpb) (:561-578)
and release on completion (:621).  The table lives on the GPU as int32
global block ids, kept in sync by delta uploads (ks_block_table_update).
"""
from __future__ import annotations

from typing import List, Optional

import torch

from . import kv
from .kv import KvFormat
from .slab_pool import BlockHandle, SlabPool


class SlabModel:
    def __init__(self, pool: SlabPool, fmt: KvFormat, max_seqs: int, max_blocks_per_seq: int):
        self.pool, self.fmt = pool, fmt
        self.key = fmt.key
        self.tpb = fmt.tokens_per_block
        self.max_blocks = max_blocks_per_seq
        dev = f"cuda:{pool.device}"
        self.table = torch.zeros((max_seqs, max_blocks_per_seq), dtype=torch.int32, device=dev)
        self.handles: List[List[BlockHandle]] = [[] for _ in range(max_seqs)]
        self.cached = [0] * max_seqs
        self._pending: List[tuple] = []

    # simulator.cpp:561-578 -- grow until ceil(tokens/tpb) blocks are held
    def ensure_capacity(self, seq: int, tokens: int) -> bool:
        need = (tokens + self.tpb - 1) // self.tpb
        hs = self.handles[seq]
        if need > self.max_blocks:
            raise ValueError("sequence exceeds max_blocks_per_seq")
        while len(hs) < need:
            h = self.pool.try_alloc_block(self.key)
            if h is None:
                return False  # stalled: caller evicts or waits
            self._pending.append((seq, len(hs), h.global_block_id))
            hs.append(h)
        return True

    # simulator.cpp:500-526 -- claim prompt blocks, roll back on failure
    def admit(self, seq: int, prompt_tokens: int) -> bool:
        assert not self.handles[seq]
        mark = len(self._pending)
        if not self.ensure_capacity(seq, prompt_tokens):
            self.pool.free_blocks(self.handles[seq])
            self.handles[seq] = []
            del self._pending[mark:]
            return False
        self.cached[seq] = prompt_tokens
        return True

    # simulator.cpp:621 / :583-596 -- completion or eviction
    def release(self, seq: int) -> None:
        if self.handles[seq]:
            self.pool.free_blocks(self.handles[seq])
        self.handles[seq] = []
        self.cached[seq] = 0

    def compact(self, max_moves: int = 1 << 20, stream=None):
        """K3 for this model's key: moves blocks out of the least-occupied
        slabs (freeing them for any key), rewrites the device table and the
        host handles.  Returns (moves, slabs_freed)."""
        self.sync(stream)
        moves, freed = kv.compact(self.pool, self.key, max_moves, tables=[self.table],
                                  stream=stream)
        if moves:
            bps = self.pool.blocks_per_slab(self.key)
            remap = dict(moves)
            for hs in self.handles:
                for i, h in enumerate(hs):
                    dst = remap.get(h.global_block_id)
                    if dst is not None:
                        sl, lo = SlabPool.split_global_block_id(dst, bps)
                        hs[i] = BlockHandle(sl, lo, dst, self.key)
        return moves, freed

    def sync(self, stream=None) -> int:
        """Uploads pending table entries; returns how many were written."""
        n = len(self._pending)
        if n:
            rows, cols, vals = zip(*self._pending)
            kv.block_table_update(self.pool, self.table, rows, cols, vals, stream)
            self._pending.clear()
        return n

    def ctx_tensor(self, seqs: Optional[List[int]] = None) -> torch.Tensor:
        seqs = range(len(self.cached)) if seqs is None else seqs
        return torch.tensor([self.cached[s] for s in seqs], dtype=torch.int32,
                            device=self.table.device)

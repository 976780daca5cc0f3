"""Op-log replay.

The reference allocator can log every alloc/free as one line
``seq time op key slab local gid`` (slab_pool.cpp:45-49, enabled by the
simulator's alloc_log, simulator.cpp:340-347).  Replaying such a log on this
pool re-creates the reference's exact slab table (and, with ``device``, the
device slab table), which lets any reference scenario drive the GPU pool and
serves as a regression format: a replay fails loudly at the first record the
pool would have answered differently.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, List

from .slab_pool import BlockHandle, KvSlabError, OpLogRecord, SlabPool, write_op_log_line


@dataclass(frozen=True)
class ReplayStats:
    records: int
    allocs: int
    frees: int


def parse_op_log(lines: Iterable[str]) -> List[OpLogRecord]:
    out = []
    for ln in lines:
        ln = ln.strip()
        if not ln:
            continue
        seq, time, op, key, slab, local, gid = ln.split()
        if op not in ("alloc", "free"):
            raise ValueError(f"bad op-log record: {ln!r}")
        out.append(OpLogRecord(int(seq), float(time), op, int(key), int(slab), int(local),
                               int(gid)))
    return out


def replay(pool: SlabPool, records: Iterable[OpLogRecord]) -> ReplayStats:
    """Applies the records in order; every alloc must land on the recorded
    (slab, local, gid) -- the allocation order is the reference's."""
    n = na = nf = 0
    for r in records:
        n += 1
        if r.op == "alloc":
            h = pool.alloc_block(r.key)
            if (h.slab_id, h.local_block_id, h.global_block_id) != (r.slab_id, r.local_block_id,
                                                                    r.global_block_id):
                raise KvSlabError(f"replay diverged at seq {r.seq}: pool gave {h}, log has "
                                  f"({r.slab_id}, {r.local_block_id}, {r.global_block_id})")
            na += 1
        else:
            pool.free_block(BlockHandle(r.slab_id, r.local_block_id, r.global_block_id, r.key))
            nf += 1
    return ReplayStats(n, na, nf)


def format_op_log(records: Iterable[OpLogRecord]) -> str:
    return "".join(write_op_log_line(r) for r in records)

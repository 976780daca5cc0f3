"""Engine block tables (kvslab::SeqTable behind ks_seq_table_*), host-only.

The rules are the reference simulator's allocator call sites
(proj/core/src/simulator.cpp): prefill claim with rollback (:500-526),
decode growth ceil((cached+1)/tpb) with a per-request stall (:561-578),
release (:621) and internal_frag_bytes (:80-89).  Checked here against a
Python restatement driving a second, plain pool with the same op order.
"""
import numpy as np
import pytest

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat


def _pool(fmts, nslabs, slab=None):
    keys = [f.key for f in fmts]
    slab = slab or max(keys) * 4
    return ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, keys, False))


class RefEngine:
    """simulator.cpp's LiveRequest::blocks bookkeeping over a plain pool."""

    def __init__(self, pool, fmt, max_seqs):
        self.pool, self.fmt, self.key = pool, fmt, fmt.key
        self.rows = [[] for _ in range(max_seqs)]
        self.cached = [0] * max_seqs

    def admit(self, s, prompt):  # :500-526
        need = -(-prompt // 16)
        got = []
        for _ in range(need):
            h = self.pool.try_alloc_block(self.key)
            if h is None:
                for g in got:
                    self.pool.free_block(g)
                return False
            got.append(h)
        self.rows[s], self.cached[s] = got, prompt
        return True

    def step(self, seqs):  # :561-578, :609-612
        stalled = []
        for s in seqs:
            need = -(-(self.cached[s] + 1) // 16)
            ok = True
            while len(self.rows[s]) < need:
                h = self.pool.try_alloc_block(self.key)
                if h is None:
                    ok = False
                    break
                self.rows[s].append(h)
            if ok:
                self.cached[s] += 1
            else:
                stalled.append(s)
        return stalled

    def release(self, s):  # :621
        for h in self.rows[s]:
            self.pool.free_block(h)
        self.rows[s], self.cached[s] = [], 0

    def frag(self):  # :80-89
        L, ts, qp = self.fmt.num_layers, self.fmt.token_size, self.fmt.qparams
        return sum(len(r) * self.key - (c * L * ts + len(r) * L * qp)
                   for r, c in zip(self.rows, self.cached) if r)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_seq_table_matches_reference_rules(seed):
    rng = np.random.default_rng(seed)
    fmts = [KvFormat(KvDtype.FP16, 8, 32, num_layers=2), KvFormat(KvDtype.INT4, 8, 32, num_layers=2)]
    pool_a, pool_b = _pool(fmts, 12), _pool(fmts, 12)
    S = 8
    ms = [SlabModel(pool_a, f, S, 64) for f in fmts]
    rs = [RefEngine(pool_b, f, S) for f in fmts]
    for it in range(400):
        mi = int(rng.integers(2))
        m, r = ms[mi], rs[mi]
        op = rng.random()
        if op < 0.25:
            s = int(rng.integers(S))
            if not r.rows[s]:
                prompt = int(rng.integers(1, 300))
                assert m.admit(s, prompt) == r.admit(s, prompt)
        elif op < 0.35:
            s = int(rng.integers(S))
            m.release(s)
            r.release(s)
        else:
            live = [s for s in range(S) if r.rows[s] and r.cached[s] < 64 * 16 - 1]
            assert m.step(live) == r.step(live)
        assert pool_a.snapshot_stats() == pool_b.snapshot_stats()
        for s in range(S):
            assert m.handles[s] == r.rows[s]
            assert m.cached[s] == r.cached[s]
        assert m.internal_frag_bytes() == r.frag()
        st = m.stats()
        assert st.held_blocks == sum(len(x) for x in r.rows)
        assert st.cached_tokens == sum(r.cached)
        assert m.ctx_lens(plus=1) == [c + 1 if rw else 0 for c, rw in zip(r.cached, r.rows)]
    ok, why = pool_a.check_integrity()
    assert ok, why


def test_admit_rolls_back_and_pending_deltas():
    fmt = KvFormat(KvDtype.FP16, 8, 32, num_layers=1)
    pool = _pool([fmt], 2, slab=fmt.key * 4)  # 8 blocks
    m = SlabModel(pool, fmt, 4, 16)
    before = pool.snapshot_stats()
    assert not m.admit(0, 9 * 16)  # needs 9 blocks
    assert pool.snapshot_stats() == before and m.handles[0] == []
    assert m.sync() == 0  # rolled back: nothing to upload
    assert m.admit(0, 3 * 16)
    assert m.sync() == 3
    # release + re-admit of the same row before a sync: one entry per cell
    m.release(0)
    assert m.admit(0, 16)
    assert m.admit(1, 16)
    assert m.sync() == 2  # (0,0) deduplicated to its last value, (1,0)
    # growth stalls at exhaustion and keeps what it got
    assert m.admit(2, 16 * 4)  # 6 blocks held now
    assert not m.ensure_capacity(2, 16 * 7)
    assert len(m.handles[2]) == 6
    assert m.step([2]) == [] and m.cached[2] == 65  # block 5 of 6 backs token 65
    m.cached[2] = 96  # every held block full
    assert m.step([2]) == [2] and m.cached[2] == 96  # stalled: not advanced


def test_table_errors_and_pool_teardown():
    fmt = KvFormat(KvDtype.INT8, 8, 32, num_layers=1)
    pool = _pool([fmt], 2)
    with pytest.raises(ks.InvalidKeyError):
        SlabModel(pool, KvFormat(KvDtype.FP16, 8, 32, num_layers=3), 2, 4)
    m = SlabModel(pool, fmt, 2, 4)
    with pytest.raises(ks.KvSlabError):
        m.ensure_capacity(0, 16 * 5)  # more blocks than a row holds
    with pytest.raises(ks.KvSlabError):
        m.cached[0] = 5  # no block backs it
    assert m.admit(0, 20)
    pool.close()  # the table is detached, not dangling
    with pytest.raises(ks.KvSlabError):
        m.admit(1, 4)

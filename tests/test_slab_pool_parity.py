"""Parity of the product allocator (libkvslab.so via the C ABI) with the
reference slabsim::SlabPool, pinned by golden vectors generated from the
compiled reference (oracle/make_golden.py).  Mirrors proj/tests/
test_slab_pool.cpp and acceptance criteria 1-2 (acceptance_test.cpp:87-223).
"""
import json
import os

import numpy as np
import pytest

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import _lib as L
import oracle
from _replay import churn, records_hash, run_script

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


SCRIPTS = _load("slab_scripts.json")
CHURN = _load("churn.json")
CHURN_REC = np.load(os.path.join(GOLD, "churn.npz"))


@pytest.mark.parametrize("case", SCRIPTS, ids=[s["name"] for s in SCRIPTS])
def test_script_matches_reference(case):
    """Every scripted case of test_slab_pool.cpp replays to identical output."""
    assert run_script(case["lines"]) == case["expected"], case["cite"]


def _product_ops(meta):
    pool = ks.SlabPool(ks.SlabPoolConfig(meta["capacity"], meta["slab"], meta["keys"],
                                         bool(meta["lcm"])))
    h_c = L.ks_block_handle()
    ok = L.C.c_int32() if hasattr(L, "C") else None
    import ctypes as C
    ok = C.c_int32()
    st = L.ks_frag_stats()
    lib = L.lib
    ph = pool.handle

    def alloc(key):
        s = lib.ks_try_alloc_block(ph, key, C.byref(h_c), C.byref(ok))
        assert s == 0
        return (h_c.slab_id, h_c.local_block_id, h_c.global_block_id, h_c.key) if ok.value else None

    def free(h):
        hh = L.ks_block_handle(*h)
        assert lib.ks_free_block(ph, C.byref(hh)) == 0

    def stats():
        lib.ks_snapshot_stats(ph, C.byref(st))
        return (st.allocated_bytes, st.free_block_bytes, st.slab_residue_bytes, st.free_slab_bytes)

    return pool, alloc, free, stats


FAST = [m for m in CHURN if m["ops"] <= 200000]
SLOW = [m for m in CHURN if m["ops"] > 200000]


def _check_churn(meta):
    pool, alloc, free, stats = _product_ops(meta)
    recs, draws = churn(meta, alloc, free, stats)
    gold = CHURN_REC[meta["name"]]
    n = gold.shape[0]
    mism = np.nonzero((recs[:n] != gold).any(axis=1))[0]
    assert mism.size == 0, f"first divergence at op {mism[0] if mism.size else -1}"
    assert records_hash(recs) == int(meta["hash"])
    assert draws == meta["draws"]
    assert list(stats()) == meta["final_stats"]
    ok, why = pool.check_integrity()
    assert ok, why


@pytest.mark.parametrize("meta", FAST, ids=[m["name"] for m in FAST])
def test_churn_matches_reference(meta):
    _check_churn(meta)


@pytest.mark.parametrize("meta", SLOW, ids=[m["name"] for m in SLOW])
def test_acceptance_criterion1_streams(meta):
    """Criterion 1 (1M ops over two pools) bit-exact against the reference."""
    _check_churn(meta)


def test_precision_matches_reference():
    """token_size / kv_block_size over the golden grid (precision.cpp:76-99)."""
    for row in _load("precision.json"):
        exp = row["expected"].split()
        try:
            ts = ks.token_size(row["kv_heads"], row["head_dim"], row["kv_bits"], row["tp"])
            bs = ks.kv_block_size(row["kv_heads"], row["head_dim"], row["kv_bits"], row["layers"],
                                  row["tpb"], row["qparams"], row["tp"])
            got = ["P", str(ts), str(bs)]
        except ks.InvalidProfileError:
            got = ["E", "InvalidProfileError"]
        assert got == exp, row


def test_op_log_records_allocs_and_frees_in_order():
    """test_slab_pool.cpp:302-313."""
    pool = ks.SlabPool(ks.SlabPoolConfig(4 * 65536, 65536, [65536, 32768]))
    log = []
    pool.set_op_log(log.append)
    h = pool.alloc_block(32768)
    pool.free_block(h)
    assert [r.op for r in log] == ["alloc", "free"]
    assert log[0].seq < log[1].seq and log[0].key == 32768
    assert ks.write_op_log_line(log[0]) == f"{log[0].seq} {log[0].seq} alloc 32768 0 0 0\n"
    t = [10.0]
    pool.set_clock(lambda: t[0])
    pool.alloc_block(65536)
    assert log[-1].time == 10.0
    pool.set_op_log(None)
    pool.alloc_block(65536)
    assert len(log) == 3


def test_identical_sequences_identical_handles():
    """test_slab_pool.cpp:214-238 (seed 99) -- determinism across two pools."""
    meta = next(m for m in CHURN if m["name"] == "determinism_seed99")
    a = _product_ops(meta)
    b = _product_ops(meta)
    ra, _ = churn(meta, *a[1:])
    rb, _ = churn(meta, *b[1:])
    assert (ra == rb).all()


def test_oracle_restatement_agrees_with_reference():
    """The C restatement (oracle/) replays the same churn bit-exactly."""
    for meta in FAST:
        op = oracle.OraclePool(meta["capacity"], meta["slab"], meta["keys"], bool(meta["lcm"]))

        def alloc(key):
            st, h = op.alloc(key)
            return None if st == 3 else h

        recs, _ = churn(meta, alloc, lambda h: op.free(h), op.stats)
        assert records_hash(recs) == int(meta["hash"]), meta["name"]


def test_compaction_plan_matches_oracle():
    """K3 plan: product and oracle restatement choose identical moves."""
    keys = [17408, 32768, 33280, 65536]
    slab = 72417280
    for seed in (1, 2, 3):
        draws = oracle.uniforms(seed, 200000)
        pool = ks.SlabPool(ks.SlabPoolConfig(24 * slab, slab, keys))
        op = oracle.OraclePool(24 * slab, slab, keys)
        live, d = [], 0
        for _ in range(30000):  # fill-and-churn
            key = keys[int(draws[d] * 4)]
            d += 1
            h = pool.try_alloc_block(key)
            st, oh = op.alloc(key)
            assert (h is None) == (st == 3)
            if h:
                live.append(h)
        for i in range(len(live) - 1, -1, -1):  # free ~70% at random
            if draws[d] < 0.7:
                pool.free_block(live[i])
                assert op.free((live[i].slab_id, live[i].local_block_id, live[i].global_block_id,
                                live[i].key)) == 0
            d += 1
        for key in keys:
            mv, freed = pool.plan_compaction(key, 5000)
            omv, ofreed = op.compact(key, 5000)
            assert mv == omv and freed == ofreed, (seed, key)
            assert pool.snapshot_stats().as_tuple() == op.stats()
        ok, why = pool.check_integrity()
        assert ok, why


def test_compaction_frees_stranded_slabs():
    """Demand-shift stranding recovered by compaction."""
    keys = [17408, 32768, 33280, 65536]
    slab = 72417280
    pool = ks.SlabPool(ks.SlabPoolConfig(16 * slab, slab, keys))
    draws = oracle.uniforms(11, 100000)
    live = []
    d = 0
    while True:
        key = keys[int(draws[d] * 4)]
        d += 1
        h = pool.try_alloc_block(key)
        if h is None:
            break
        live.append(h)
    for i, h in enumerate(live):
        if draws[(d + i) % len(draws)] < 0.7:
            pool.free_block(h)
    before = pool.snapshot_stats()
    freed_total = 0
    for key in keys:
        _, freed = pool.plan_compaction(key)
        freed_total += freed
    after = pool.snapshot_stats()
    assert freed_total > 0
    assert after.free_slab_bytes > before.free_slab_bytes
    assert after.allocated_bytes == before.allocated_bytes
    assert pool.check_integrity()[0]

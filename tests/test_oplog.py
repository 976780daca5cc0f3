"""Op-log replay: a log written by the reference allocator itself
(tests/golden/oplog_ref.txt, oracle/make_golden.py) replays bit-exactly on the
product pool, and the product pool's own op log reproduces it line for line."""
import os

import pytest

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200.oplog import format_op_log, parse_op_log, replay

GOLD = os.path.join(os.path.dirname(__file__), "golden", "oplog_ref.txt")
KiB = 1024


def _pool():
    return ks.SlabPool(ks.SlabPoolConfig(16 * 24 * KiB, 24 * KiB, [2 * KiB, 3 * KiB, 4 * KiB]))


def test_reference_log_replays_and_round_trips():
    text = open(GOLD).read()
    recs = parse_op_log(text.splitlines())
    assert len(recs) > 2000
    pool = _pool()
    mine = []
    pool.set_op_log(mine.append)
    st = replay(pool, recs)
    assert st.allocs + st.frees == len(recs)
    assert format_op_log(mine) == text
    assert pool.check_integrity()[0]


def test_replay_detects_divergence():
    recs = parse_op_log(open(GOLD).read().splitlines())
    pool = _pool()
    pool.alloc_block(2 * KiB)  # state differs from the log's starting point
    with pytest.raises(ks.Error):
        replay(pool, recs)

"""Replays the golden op scripts / churn streams on the product pool.

The output strings use exactly the line format oracle/ref_golden.cpp prints
for the reference allocator, so parity is a string comparison.
"""
import numpy as np

import paper_2509_06261_b200 as ks
import oracle


def _stats(p):
    s = p.snapshot_stats()
    return f" S {s.allocated_bytes} {s.free_block_bytes} {s.slab_residue_bytes} {s.free_slab_bytes}"


def _cfg(tokens):
    cap, slab, lcm, n = int(tokens[0]), int(tokens[1]), int(tokens[2]), int(tokens[3])
    keys = [int(x) for x in tokens[4:4 + n]]
    return ks.SlabPoolConfig(cap, slab, keys, bool(lcm))


def run_script(lines, make_pool=lambda cfg: ks.SlabPool(cfg)):
    out, results = [], []
    pool = saved = None
    for i, line in enumerate(lines):
        tok = line.split()
        cmd, args = tok[0], tok[1:]
        r = f"R {i}"
        results.append(None)
        try:
            if cmd == "config":
                p = make_pool(_cfg(args))
                pool = p
                r += f" CFG {p.slab_count()} {p.tail_remainder_bytes()} {p.usable_capacity_bytes()}"
                r += _stats(p)
            elif cmd in ("alloc", "try_alloc"):
                key = int(args[0])
                h = pool.alloc_block(key) if cmd == "alloc" else pool.try_alloc_block(key)
                if h is None:
                    r += " NONE"
                else:
                    r += f" H {h.slab_id} {h.local_block_id} {h.global_block_id} {h.key}"
                    results[-1] = h
                r += _stats(pool)
            elif cmd == "free":
                pool.free_block(results[int(args[0])])
                r += " OK" + _stats(pool)
            elif cmd == "free_raw":
                s, l, g, k = (int(x) for x in args)
                pool.free_block(ks.BlockHandle(s, l, g, k))
                r += " OK" + _stats(pool)
            elif cmd == "bps":
                r += f" V {pool.blocks_per_slab(int(args[0]))}"
            elif cmd == "free_blocks":
                r += f" V {pool.free_blocks_for_key(int(args[0]))}"
            elif cmd == "alloc_count":
                k = int(args[0])
                r += f" V {pool.allocated_block_count(None if k == 0 else k)}"
            elif cmd == "states":
                n = pool.slab_count()
                r += f" ST {n}" + "".join(f" {int(pool.slab_state(j))} {pool.slab_key(j)}"
                                          for j in range(n))
            elif cmd == "integrity":
                r += f" I {1 if pool.check_integrity()[0] else 0}"
            elif cmd == "flip":
                pool.debug_flip_occupancy_bit(int(args[0]), int(args[1]))
                r += " OK"
            elif cmd == "save":
                saved = pool.clone_host()
                r += " OK"
            elif cmd == "equal_saved":
                r += f" EQ {1 if pool == saved else 0}"
            elif cmd == "gid":
                s, l, b = (int(x) for x in args)
                g = ks.SlabPool.global_block_id(s, l, b)
                s2, l2 = ks.SlabPool.split_global_block_id(g, b)
                r += f" G {g} {s2} {l2}"
            else:
                r += " E UnknownCommand"
        except ks.Error as e:
            r += f" E {type(e).__name__}"
        out.append(r)
    return out


FNV_OFF, FNV_PRIME = np.uint64(0xcbf29ce484222325), np.uint64(0x100000001b3)


def records_hash(recs: np.ndarray) -> int:
    """Same fold as ref_golden.cpp Fnv: per record FNV-1a over u64 fields,
    total = sum(h_i * (2i+1)) mod 2^64."""
    recs = recs.astype(np.uint64)
    with np.errstate(over="ignore"):
        h = np.full(recs.shape[0], FNV_OFF, dtype=np.uint64)
        for j in range(recs.shape[1]):
            h = (h ^ recs[:, j]) * FNV_PRIME
        w = np.arange(recs.shape[0], dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        return int(np.sum(h * w, dtype=np.uint64))


def churn(meta, alloc, free, stats, draws=None):
    """Drives the churn loop of test_slab_pool.cpp:240-290 /
    acceptance_test.cpp:87-162 over (alloc, free, stats) callables.
    Returns the records array [ops, 9] (uint64) and the number of draws."""
    keys = meta["keys"]
    pfree = meta["pfree_milli"] / 1000.0
    ops = meta["ops"]
    if draws is None:
        draws = oracle.uniforms(meta["seed"], 2 * ops + 16)
    d = 0
    live = []
    recs = np.zeros((ops, 9), dtype=np.uint64)
    for i in range(ops):
        do_free = False
        if live:
            do_free = draws[d] < pfree
            d += 1
        if do_free:
            pick = int(draws[d] * len(live))
            d += 1
            h = live[pick]
            free(h)
            if meta["remove_mode"] == 0:
                del live[pick]
            else:
                live[pick] = live[-1]
                live.pop()
            row = (2, h[3], h[0], h[1], h[2])
        else:
            key = keys[int(draws[d] * len(keys))]
            d += 1
            h = alloc(key)
            if h is None:
                row = (1, key, 0, 0, 0)
            else:
                live.append(h)
                row = (0, key, h[0], h[1], h[2])
        recs[i, :5] = row
        recs[i, 5:] = stats()
    return recs, d

#!/usr/bin/env python3
"""Generate tests/golden/* from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Runs oracle/_ref/ref_golden -- the reference SlabPool / precision / Rng /
WholeSlabRefModel compiled from /root/reference by `make -C oracle ref` -- on
op scripts that restate the reference's own unit and acceptance tests, and
writes the answers as golden files.  The golden files are committed because
/root/reference is absent on the GPU box.

Re-run:  make -C oracle ref && python oracle/make_golden.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
BIN = os.path.join(HERE, "_ref", "ref_golden")
KiB = 1024


def run(lines):
    p = subprocess.run([BIN], input="\n".join(lines) + "\n", capture_output=True, text=True,
                       check=True)
    return p.stdout.splitlines()


def cfg(cap, slab, keys, lcm=1):
    return f"config {cap} {slab} {lcm} {len(keys)} " + " ".join(str(k) for k in keys)


TWO_KEY = cfg(4 * 64 * KiB, 64 * KiB, [64 * KiB, 32 * KiB])

# Each script restates one TEST_CASE of proj/tests/test_slab_pool.cpp (cited).
SCRIPTS = [
    ("creation_validates_geometry", "test_slab_pool.cpp:38-64",
     [TWO_KEY, "states", cfg(45, 15, [3, 5]), cfg(96 * KiB, 48 * KiB, [64 * KiB]),
      cfg(64, 16, [32])]),
    ("tail_remainder", "test_slab_pool.cpp:66-76", [cfg(100, 30, [10, 15])]),
    ("global_ids_worked_example", "test_slab_pool.cpp:78-100; acceptance_test.cpp:200-223",
     [cfg(4 * 64 * KiB, 64 * KiB, [32 * KiB]), f"bps {32*KiB}", f"alloc {32*KiB}",
      f"alloc {32*KiB}", f"alloc {32*KiB}", "gid 1 0 2", "gid 7 3 5", "gid 123456 77 1000"]),
    ("lowest_partial_first", "test_slab_pool.cpp:102-115",
     [cfg(4 * 64 * KiB, 64 * KiB, [32 * KiB]), f"alloc {32*KiB}", f"alloc {32*KiB}",
      f"alloc {32*KiB}", "free 1", f"alloc {32*KiB}", "states"]),
    ("exhaustion_and_key_mismatch", "test_slab_pool.cpp:117-130",
     [TWO_KEY] + [f"alloc {64*KiB}"] * 3 + [f"alloc {32*KiB}", f"free_blocks {32*KiB}",
                                            f"try_alloc {64*KiB}", f"alloc {64*KiB}",
                                            "alloc 1234", "try_alloc 1234", "free_blocks 1234"]),
    ("free_transitions_and_errors", "test_slab_pool.cpp:132-160",
     [cfg(2 * 64 * KiB, 64 * KiB, [32 * KiB, 64 * KiB]), f"alloc {32*KiB}", f"alloc {32*KiB}",
      "states", "free 1", "states", "free 2", "states", f"alloc {64*KiB}", "free 2", "free 8",
      "free 8", f"free_raw 99 0 0 {32*KiB}", f"free_raw 0 5 5 {32*KiB}",
      f"alloc {32*KiB}", f"free_raw 0 0 1 {32*KiB}", f"free_raw 0 0 0 {64*KiB}", "integrity"]),
    ("bps_and_residue", "test_slab_pool.cpp:162-186",
     [TWO_KEY, f"bps {32*KiB}", f"bps {64*KiB}", "bps 7", cfg(45, 15, [4]),
      cfg(45, 15, [4], lcm=0), "bps 4", "alloc 4", "states"]),
    ("single_step_stats", "test_slab_pool.cpp:188-202", [TWO_KEY, f"alloc {32*KiB}"]),
    ("alloc_free_round_trip", "test_slab_pool.cpp:204-212",
     [TWO_KEY, f"alloc {32*KiB}", "save", f"alloc {64*KiB}", "equal_saved", "free 3",
      "equal_saved"]),
    ("corruption_detected", "test_slab_pool.cpp:292-300",
     [TWO_KEY, f"alloc {32*KiB}", "integrity", "flip 0 1", "integrity"]),
    ("counts_by_key", "slab_pool.hpp:134-138",
     [TWO_KEY, f"alloc {32*KiB}", f"alloc {64*KiB}", f"alloc {32*KiB}", f"alloc {32*KiB}",
      "alloc_count 0", f"alloc_count {32*KiB}", f"alloc_count {64*KiB}", "alloc_count 5",
      f"free_blocks {32*KiB}", f"free_blocks {64*KiB}", "free 2", f"free_blocks {32*KiB}",
      "states", "integrity"]),
    ("lcm_edge_cases", "slab_pool.cpp:28-37,72-80",
     [cfg(10, 0, [1]), cfg(10, 10, []), cfg(10, 10, [0]), cfg(9, 10, [5]),
      cfg(1 << 40, 72417280, [65536, 32768, 33280, 17408]),
      cfg(1 << 40, 72417280 // 2, [65536, 32768, 33280, 17408]),
      cfg(3 * 65536, 65536, [65536, 65536, 32768]), "states"]),
]

# Churn streams: (name, cite, cap, slab, keys(sorted), lcm, seed, ops, pfree_milli, remove_mode, n_record)
CHURNS = [
    ("determinism_seed99", "test_slab_pool.cpp:214-238", 4 * 64 * KiB, 64 * KiB,
     [32 * KiB, 64 * KiB], 1, 99, 500, 400, 0, 500),
    ("churn_vs_whole_slab_ref", "test_slab_pool.cpp:240-290", 16 * 24 * KiB, 24 * KiB,
     [2 * KiB, 3 * KiB, 4 * KiB], 1, 1234, 20000, 450, 0, 20000),
    ("criterion1_aligned", "acceptance_test.cpp:166-179", 64 * 24 * KiB, 24 * KiB,
     [2 * KiB, 3 * KiB, 4 * KiB], 1, 2024, 500000, 470, 1, 5000),
    ("criterion1_relaxed", "acceptance_test.cpp:181-186", 64 * 13 * KiB, 13 * KiB,
     [2 * KiB, 3 * KiB, 4 * KiB], 0, 4048, 500000, 470, 1, 5000),
    ("bench_churn_4keys", "bench_slab_pool.cpp:25-58", 1024 * 12 * 4096, 12 * 4096,
     [4096, 2 * 4096, 3 * 4096, 6 * 4096], 1, 42, 200000, 500, 1, 2000),
    ("mixed_precision_keys", "SURVEY.md 8 C4 keys", 24 * 72417280, 72417280,
     [17408, 32768, 33280, 65536], 1, 7, 100000, 480, 1, 2000),
]

PREC = []
for h, d, L, tp, tpb, qp, bits in [
    (8, 128, 1, 1, 16, 0, 16), (8, 128, 1, 1, 16, 0, 8), (8, 128, 1, 1, 16, 0, 4),
    (8, 128, 1, 2, 16, 0, 16), (9, 128, 1, 2, 16, 0, 16), (8, 128, 1, 1, 16, 64, 8),
    (8, 128, 4, 1, 16, 0, 16), (8, 128, 1, 1, 0, 0, 16), (32, 128, 1, 1, 16, 0, 16),
    (8, 128, 32, 1, 16, 1024, 4), (8, 128, 32, 1, 16, 0, 16), (8, 128, 1, 1, 16, 512, 8),
    (1, 1, 1, 1, 16, 0, 3), (1, 2, 1, 1, 16, 0, 3), (8, 128, 1, 0, 16, 0, 16),
    (8, 64, 80, 8, 32, 0, 8), (16, 256, 2, 4, 7, 13, 4)]:
    PREC.append((h, d, L, tp, tpb, qp, bits))
rng = np.random.default_rng(5)
for _ in range(200):
    PREC.append((int(rng.integers(1, 65)), int(rng.integers(1, 257)), int(rng.integers(1, 81)),
                 int(rng.integers(1, 9)), int(rng.integers(0, 65)), int(rng.integers(0, 2049)),
                 int(rng.choice([4, 8, 16]))))


def main():
    if not os.path.exists(BIN):
        sys.exit("build the reference first: make -C oracle ref")
    os.makedirs(OUT, exist_ok=True)

    scripts = []
    for name, cite, lines in SCRIPTS:
        out = run(lines)
        assert len(out) == len(lines), (name, out)
        scripts.append({"name": name, "cite": cite, "lines": lines, "expected": out})
    with open(os.path.join(OUT, "slab_scripts.json"), "w") as f:
        json.dump(scripts, f, indent=1)

    prec_out = run([f"prec {h} {d} {L} {tp} {tpb} {qp} {b}" for h, d, L, tp, tpb, qp, b in PREC])
    with open(os.path.join(OUT, "precision.json"), "w") as f:
        json.dump([{"kv_heads": h, "head_dim": d, "layers": L, "tp": tp, "tpb": tpb,
                    "qparams": qp, "kv_bits": b, "expected": o}
                   for (h, d, L, tp, tpb, qp, b), o in zip(PREC, prec_out)], f, indent=0)

    rng_out = {}
    for seed in (0, 1, 42, 99, 1234, 2024, 4048, 2**63 + 5):
        line = run([f"rng {seed} 700"])[0].split()[1:]
        rng_out[str(seed)] = line
    with open(os.path.join(OUT, "rng.json"), "w") as f:
        json.dump(rng_out, f)

    # reference op logs (slab_pool.cpp:45-49 format) for the replay path
    oplog = run([f"oplog {16 * 24 * KiB} {24 * KiB} 1 3 2048 3072 4096 77 3000"])
    with open(os.path.join(OUT, "oplog_ref.txt"), "w") as f:
        f.write("".join(l[2:] + "\n" for l in oplog if l.startswith("L ")))

    meta, arrays = [], {}
    for name, cite, cap, slab, keys, lcm, seed, ops, pf, rm, nrec in CHURNS:
        line = (f"churn {cap} {slab} {lcm} {len(keys)} " + " ".join(map(str, keys)) +
                f" {seed} {ops} {pf} {rm} {nrec}")
        out = run([line])
        recs = np.array([[int(x) for x in l.split()[1:]] for l in out if l.startswith("C ")],
                        dtype=np.uint64)
        tail = [l for l in out if l.startswith("CH ")][0].split()
        arrays[name] = recs
        meta.append({"name": name, "cite": cite, "capacity": cap, "slab": slab, "keys": keys,
                     "lcm": lcm, "seed": seed, "ops": ops, "pfree_milli": pf,
                     "remove_mode": rm, "n_record": nrec, "hash": tail[1], "count": int(tail[2]),
                     "draws": int(tail[3]), "integrity": int(tail[4]), "live": int(tail[5]),
                     "final_stats": [int(x) for x in tail[7:11]]})
    np.savez_compressed(os.path.join(OUT, "churn.npz"), **arrays)
    with open(os.path.join(OUT, "churn.json"), "w") as f:
        json.dump(meta, f, indent=1)
    c5()
    pool_sizing()
    print("golden vectors written to", OUT)


def c5():
    """BASELINE configs[4]: the reference's own placement (place_models,
    placement.cpp:135-205) of 16 mixed-precision models onto 8 B200 groups and
    its Poisson trace (generate_workload, workload.cpp:130-190), from
    oracle/_ref/ref_c5 (oracle/ref_c5.cpp)."""
    out = subprocess.run([os.path.join(HERE, "_ref", "ref_c5")], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    models, assign, reqs = [], {}, []
    for l in out:
        t = l.split()
        if t[0] == "K":
            models.append({"name": t[1], "kv_bits": int(t[2]), "key": int(t[3])})
        elif t[0] == "A":
            assign[t[1]] = t[2]
        elif t[0] == "R":
            reqs.append([int(t[1]), t[2], float(t[3]), int(t[4]), int(t[5])])
    with open(os.path.join(OUT, "c5.json"), "w") as f:
        json.dump({"cite": "oracle/ref_c5.cpp -> placement.cpp:135-205, workload.cpp:130-190",
                   "models": models, "assign": assign, "requests": reqs}, f, indent=0)


def pool_sizing():
    """a4: the reference's per-group KV pool sizing (simulator.cpp:264-290) for
    every shipped scenario, with its inputs, from oracle/_ref/ref_calib --pools."""
    import glob
    scen = sorted(glob.glob("/root/reference/proj/scenarios/*.json"))
    out = subprocess.run([os.path.join(HERE, "_ref", "ref_calib"), "--pools", *scen], capture_output=True,
                         text=True, check=True).stdout
    with open(os.path.join(OUT, "pool_sizing.json"), "w") as f:
        json.dump({"cite": "oracle/ref_calib.cpp --pools -> simulator.cpp:264-290, precision.cpp:119-127",
                   "scenarios": json.loads(out)}, f, indent=0)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "c5":
        c5()
    elif len(sys.argv) > 1 and sys.argv[1] == "pool_sizing":
        pool_sizing()
    else:
        main()

"""BASELINE configs[3] -- four co-located models (FP16 / FP8-E4M3 / INT8 / INT4
KV, Llama-3-8B shape: 32 layers, 32q/8kv, d128) on one relaxed slab pool,
with the batch of every model following a seeded square wave and slab
compaction (K3) whenever stranded free-block bytes exceed 25 %.

Per phase: release / admit sequences to the phase's batch (prompt lengths
uniform in [512, 2048]; claims by the reference growth rules), compaction if
triggered (timed: K3 bytes = 2 x moved key bytes), then STEPS decode steps
(growth rule on the host, then one CUDA graph, timed on the device per step: per layer and model one fused
K1+K2 launch, the four models on their own streams).  KV contents are not
prefilled (timing only; parity of this config is tests/test_gpu_configs.py).
Prints one JSON line; run on the GPU box:  python scripts/bench_c4.py
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

L, HKV, HQ, D = 32, 8, 32, 128
MAXB = int(os.environ.get("MAXB", 64))
PHASES = int(os.environ.get("PHASES", 8))
STEPS = int(os.environ.get("STEPS", 8))
WAVE = [MAXB, 8]  # square wave of the batch per model
TRIGGER = float(os.environ.get("TRIGGER", 0.25))  # stranded free-block fraction

fmts = [KvFormat(dt, HKV, HQ, D, L) for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4)]
keys = [f.key for f in fmts]
slab = 8 << 20  # the keys' lcm is tens of GB: a relaxed (residue) pool
max_blocks = (2048 + PHASES * STEPS + 15) // 16 + 1
need = sum(MAXB * max_blocks * k for k in keys)
pool = ks.SlabPool(ks.SlabPoolConfig((need * 5 // 4 // slab + 8) * slab, slab, keys, False), device=0)
kv.kv_tensor(pool).zero_()
models = [SlabModel(pool, f, MAXB, max_blocks) for f in fmts]
rng = np.random.default_rng(2024)
dev = torch.device("cuda:0")
scales = torch.ones(2 * HKV, dtype=torch.float32, device=dev)
q = [[torch.randn(MAXB, HQ, D, dtype=torch.float16, device=dev) for _ in range(L)] for _ in fmts]
out = [[torch.empty(MAXB, HQ, D, dtype=torch.float16, device=dev) for _ in range(L)] for _ in fmts]
knew = torch.randn(MAXB, HKV, D, dtype=torch.float16, device=dev)
ctx = [torch.zeros(MAXB, dtype=torch.int32, device=dev) for _ in fmts]
step_inc = [torch.zeros(MAXB, dtype=torch.int32, device=dev) for _ in fmts]
ws = [kv.DecodeWorkspace(pool, f, MAXB) for f in fmts]
streams = [torch.cuda.Stream() for _ in fmts]
live = [set() for _ in fmts]


def device_step():
    main = torch.cuda.current_stream()
    for st in streams:
        st.wait_stream(main)
    for layer in range(L):
        for mi, m in enumerate(models):
            kv.paged_decode(pool, m.fmt, layer, q[mi][layer], m.table, ctx[mi], out=out[mi][layer],
                            kv_scales=scales, workspace=ws[mi], k_new=knew[:, :, :], v_new=knew,
                            stream=streams[mi])
    for mi in range(len(models)):
        with torch.cuda.stream(streams[mi]):
            ctx[mi].add_(step_inc[mi])
    for st in streams:
        main.wait_stream(st)


# MPS-style spatial split (ks_set_decode_sm_share): SMs in proportion to the
# KV bytes per token, INT4 weighted 2x (its K2 is consumer-bound)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
w = [4096.0, 2048.0 + 64 / 16, 2048.0 + 64, 2 * (1024.0 + 64)]
SHARE = [max(8, int(nsm * x / sum(w))) for x in w]

def set_shares(shares):
    for m, sh in zip(models, shares):
        kv.set_decode_sm_share(pool, m.key, sh)


if os.environ.get("NO_SHARE") is None:
    set_shares(SHARE)


def tune_shares():
    """Pick the SM split once, like bench.py's co-location autotune: a few
    candidate splits (byte-proportional, INT4 weighted 1x/2x/3x, all SMs or
    92 %) timed on an 8-layer eager pass at the full batch."""
    for mi, m in enumerate(models):
        for s_ in range(MAXB):
            assert m.admit(s_, 1024)
        m.sync()
        ctx[mi].fill_(1024)
    cands = []
    for w4 in (1.0, 2.0, 3.0):
        for tot in (nsm, int(nsm * 0.92)):
            ww = [4096.0, 2052.0, 2112.0, w4 * 1088.0]
            cands.append(tuple(max(8, int(tot * x / sum(ww))) for x in ww))
    best, best_ms = None, None
    for c in cands:
        set_shares(c)
        for _ in range(2):
            a, b = ev(), ev()
            a.record()
            for layer in range(8):
                for mi, m in enumerate(models):
                    kv.paged_decode(pool, m.fmt, layer, q[mi][layer], m.table, ctx[mi], out=out[mi][layer],
                                    kv_scales=scales, workspace=ws[mi], stream=streams[mi])
            for st_ in streams:
                torch.cuda.current_stream().wait_stream(st_)
            b.record()
            torch.cuda.synchronize()
        t = a.elapsed_time(b)
        if best_ms is None or t < best_ms:
            best, best_ms = c, t
    for mi, m in enumerate(models):
        for s_ in range(MAXB):
            m.release(s_)
        ctx[mi].zero_()
    return list(best)


ev = lambda: torch.cuda.Event(enable_timing=True)
if os.environ.get("NO_SHARE") is None and os.environ.get("NO_TUNE") is None:
    SHARE = tune_shares()
    set_shares(SHARE)

# capture once: inactive rows have ctx 0 and cost nothing
for mi, m in enumerate(models):  # a valid table for the warm-up launch
    assert m.admit(0, 16)
    m.sync()
    ctx[mi][0] = 17
    m.ensure_capacity(0, 17)
    m.sync()
cap = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(cap):
    device_step()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=cap):
        device_step()
torch.cuda.synchronize()
for m in models:
    m.release(0)

dec_bytes = dec_ms = 0.0
tokens = 0
cmp_bytes = cmp_ms = 0.0
compactions = moves_total = slabs_freed = 0
trace = []  # stranded fraction per phase
phase_ms = []  # device ms per decode step, per phase
ev = lambda: torch.cuda.Event(enable_timing=True)
for ph in range(PHASES):
    target = WAVE[ph % 2]
    for mi, m in enumerate(models):
        while len(live[mi]) > target:
            s = sorted(live[mi])[int(rng.integers(len(live[mi])))]
            live[mi].discard(s)
            m.release(s)
        free = [s for s in range(MAXB) if s not in live[mi]]
        while len(live[mi]) < target and free:
            s = free.pop(int(rng.integers(len(free))))
            if not m.admit(s, int(rng.integers(512, 2049))):
                break
            live[mi].add(s)
        m.sync()
    st = pool.snapshot_stats()
    stranded = st.free_block_bytes / max(1, st.allocated_bytes + st.free_block_bytes)
    trace.append(round(stranded, 3))
    if stranded > TRIGGER or (ph == PHASES - 1 and compactions == 0):  # at least one K3 pass measured
        a, b = ev(), ev()
        a.record()
        for m in models:
            mv, fr = m.compact()
            moves_total += len(mv)
            slabs_freed += fr
            cmp_bytes += 2.0 * len(mv) * m.key
        b.record()
        torch.cuda.synchronize()
        cmp_ms += a.elapsed_time(b)
        compactions += 1
    for mi, m in enumerate(models):  # device ctx and per-step increments of the phase
        ctx[mi].copy_(torch.tensor([m.cached[s] + 1 if s in live[mi] else 0 for s in range(MAXB)],
                                   dtype=torch.int32))
        step_inc[mi].copy_(torch.tensor([1 if s in live[mi] else 0 for s in range(MAXB)], dtype=torch.int32))
    torch.cuda.synchronize()
    pairs = []
    for _ in range(STEPS):
        for mi, m in enumerate(models):  # growth rule for this step's token (simulator.cpp:561-578)
            for s in live[mi]:
                if not m.ensure_capacity(s, m.cached[s] + 1):
                    raise RuntimeError("pool exhausted")
            m.sync()
        cls = [[m.cached[s] + 1 for s in sorted(live[mi])] for mi, m in enumerate(models)]
        dec_bytes += sum(L * (m.fmt.decode_bytes(c) + m.fmt.append_bytes(len(c))) for m, c in zip(models, cls))
        tokens += sum(len(c) for c in cls)
        a, b = ev(), ev()  # device time of the step (the host growth work above is not in it)
        a.record()
        g.replay()
        b.record()
        pairs.append((a, b))
        for mi, m in enumerate(models):
            for s in live[mi]:
                m.cached[s] += 1
    torch.cuda.synchronize()
    ph_ms = sum(a.elapsed_time(b) for a, b in pairs)
    dec_ms += ph_ms
    phase_ms.append(round(ph_ms / STEPS, 3))
assert pool.check_integrity()[0]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6534.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6534.0
gbs = dec_bytes / (dec_ms / 1e3) / 1e9
print(json.dumps({
    "metric": "slab paged-decode attention HBM GB/s", "value": round(gbs, 1), "unit": "GB/s",
    "frac_of_peak": round(gbs / peak, 4), "decode_tok_s": round(tokens / (dec_ms / 1e3), 1),
    "config": {"workload": "c4: four co-located Llama-3-8B-shape models (32L, 32q/8kv, d128), FP16 / FP8-E4M3 / "
                           "INT8 / INT4 KV, one relaxed 8 MiB-slab pool, batch square wave "
                           f"{WAVE} per model, {PHASES} phases x {STEPS} decode steps, compaction at > {TRIGGER:.0%} stranded "
                           "(and once in the last phase if it never triggered)",
               "data": "synthetic, KV not prefilled (timing only)",
               "sm_share": None if os.environ.get("NO_SHARE") else SHARE},
    "compaction": {"note": "K3 moves + table remap, host plan included in the time", "runs": compactions, "moves": moves_total, "slabs_freed": slabs_freed,
                   "GBps": round(cmp_bytes / (cmp_ms / 1e3) / 1e9, 1) if cmp_ms else None},
    "residue_bytes": pool.snapshot_stats().slab_residue_bytes,
    "stranded_per_phase": trace,
    "step_ms_per_phase": phase_ms,
}))

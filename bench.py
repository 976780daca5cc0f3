#!/usr/bin/env python3
"""bench.py -- KV-slab data path on B200.

Default workload (N=1 headline, BASELINE.json configs[3], the largest
single-GPU configuration): four co-located Llama-3-8B-shaped models (32
layers, 32 q / 8 kv heads, d=128) with FP16 / FP8-E4M3 / INT8 / INT4 KV on
ONE relaxed slab pool (64 MiB slabs) per GPU.  Every model's batch follows a
seeded square wave 64 / 8 sequences (phases of --phase-steps decode steps);
prompts are uniform in [512, 2048] tokens.  A phase change releases the
sequences that finish (the survivors are packed into rows 0..B-1), or admits
new ones (prefill claim + K1 prompt append for all 32 layers), and runs K3
compaction on every key when the stranded free-block bytes exceed 25 % of the
bytes in formatted slabs.  A decode step = host growth rule
(kvslab::SeqTable, simulator.cpp:561-578) + table delta upload, then one CUDA
graph: per layer and model one fused K1+K2 launch, the models on their own
streams with SM shares autotuned per batch size (the consumer-bound INT4
model fenced into a few dozen SMs at B = 64).  The warm-up runs one low /
high cycle; the timed steps then alternate 8, 64, 8, 64 (--phase-steps each).

value  = algorithmic HBM bytes (K2 decode + K1 appends + K3 moves, SURVEY.md
         8d) / device time of exactly --steps steps (phase changes included),
         whole job over all ranks (max-over-ranks time).
e2e    = the same schedule (twice) through the public API with every step's
         inputs (Q, new K/V, admitted prompts' K/V) copied in from pinned host
         memory and O copied back (prompt K/V pipelined one admission ahead);
         graph replay, plus an eager variant.
roofline = the FP16 K2 launch (dominant kernel) timed live by CUDA events.
c3     = BASELINE configs[2] (FP16 + INT4 co-located, B8, ctx 8k), same
         contract, nested in the line (N=1).
cpu_baseline = the fp64 OpenMP oracle (oracle/) on a bounded sample.
--gpus N: one process per GPU (self-spawned through torch.distributed.run
when WORLD_SIZE is unset); every rank owns an independent pool (placement
sharding, no collective on the data path).  --workload c5 places BASELINE
configs[4]'s 16 models by the reference's own placement (tests/golden/c5.json).
--impl reference: the reference's CPU path (reference SlabPool from
oracle/_ref + the oracle port for append/attention), rank 0 only.
"""
import argparse
import ctypes as C
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P = argparse.ArgumentParser()
P.add_argument("--gpus", type=int, default=1)
P.add_argument("--steps", type=int, default=20)
P.add_argument("--warmup", type=int, default=5)
P.add_argument("--impl", default="ours", choices=["ours", "reference"])
P.add_argument("--layers", type=int, default=32)
P.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5"],
               help="c4 (default): FP16/FP8/INT8/INT4 co-located, batch wave 64/8, compaction; "
                    "c3: FP16 + INT4, B8 ctx 8k; c2: FP16 + FP8, B16 ctx 2k; c1: FP16 MHA layer "
                    "B8 ctx 1k; c5: the reference placement of 16 models over the GPUs")
P.add_argument("--phase-steps", type=int, default=5, help="c4: decode steps per batch phase")
P.add_argument("--no-cpu-baseline", action="store_true")
P.add_argument("--no-sweep", action="store_true", help="skip the per-format K2 / K4 sweep")
P.add_argument("--no-c3", action="store_true", help="skip the nested c3 measurement")
P.add_argument("--profile", action="store_true", help="a few eager steps, no timing (for ncu)")
P.add_argument("--dry-run-spawn", action="store_true", help="print the multi-GPU launch and exit")
ARGS = P.parse_args()

RANK = int(os.environ.get("RANK", "0"))
WORLD = int(os.environ.get("WORLD_SIZE", "1"))
LOCAL = int(os.environ.get("LOCAL_RANK", "0"))

HQ, HKV, D = 32, 8, 128
DT_NAMES = {0: "fp16", 1: "fp8_e4m3", 2: "int8", 3: "int4"}
C4_WAVE = (64, 8)
C4_SLAB = 64 << 20
C4_TRIGGER = 0.25

# BASELINE.json configs: dts = KV dtype codes of the co-located models (0 FP16,
# 1 FP8-E4M3, 2 INT8, 3 INT4), batch per model, context
WORKLOADS = {
    "c1": dict(dts=(0,), batch=8, ctx=1024, hq=32, hkv=32, layers=1,
               text="c1: single FP16 Llama-style layer (32 heads MHA, d128), batch 8, ctx 1024"),
    "c2": dict(dts=(0, 1), batch=16, ctx=2048,
               text="c2: two co-located Llama-3-8B-shape models (32L, 32q/8kv, d128) on one slab pool, "
                    "FP16 KV + FP8-E4M3 KV (64 B/layer params)"),
    "c3": dict(dts=(0, 3), batch=8, ctx=8192,
               text="c3: two co-located Llama-3-8B-shape models (32L, 32q/8kv, d128) on one slab pool, "
                    "FP16 KV + INT4 KV (QoQ-style fp16 scale/zero per token and head), ctx 8k"),
    "c4": dict(dts=(0, 1, 2, 3), batch=C4_WAVE[0], ctx=2048,
               text="c4: four co-located Llama-3-8B-shape models (32L, 32q/8kv, d128), FP16 / FP8-E4M3 / "
                    "INT8 / INT4 KV on one relaxed 64 MiB-slab pool, batch square wave 64/8 per model, "
                    "prompts U[512,2048], K1 prompt append on admission, K3 compaction when stranded "
                    "free-block bytes > 25 %"),
    "c5": dict(dts=(), batch=32, ctx=0,
               text="c5: the reference's placement of 16 mixed-precision models (4 per KV precision, "
                    "Llama-3-8B shape) over 8 groups (tests/golden/c5.json: place_models + "
                    "generate_workload), rank r = group r, each with an independent pool; requests "
                    "of the reference Poisson trace cycled through each model's running batch"),
}
WL = WORKLOADS[ARGS.workload]


def cpu_model() -> str:
    """The host CPU (CPU model and core count in every report)."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn() -> None:
    """--gpus N without a torchrun environment: re-launch as N ranks (one
    process per GPU).  Refuses, instead of silently measuring fewer GPUs,
    when the box has fewer than N devices."""
    if ARGS.impl != "ours" or ARGS.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ARGS.gpus}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    if ARGS.dry_run_spawn:
        print(json.dumps({"spawn": cmd}))
        sys.exit(0)
    import torch
    n = torch.cuda.device_count()
    if n < ARGS.gpus:
        sys.stderr.write(f"bench.py: --gpus {ARGS.gpus} needs {ARGS.gpus} CUDA devices, found {n}\n")
        sys.exit(2)
    os.execv(sys.executable, cmd)


def config_dict(wl, batch, ctx, extra=None):
    d = {"workload": wl["text"], "layers": wl.get("layers", ARGS.layers),
         "batch_per_model": batch, "ctx": ctx, "tokens_per_block": 16,
         "kv_dtypes": [DT_NAMES[x] for x in wl["dts"]],
         "parallelism": f"placement x{WORLD} (independent pool per GPU, no collective)",
         "l2": "inputs larger than L2: each step streams GBs of KV per GPU (126 MB L2)"}
    if extra:
        d.update(extra)
    return d


# ======================================================================
# Phase schedules shared by both arms
# ======================================================================
def c4_phase_targets(warmup, steps, phase_steps):
    """Batch per model for every step: the warm-up runs one low / high cycle
    (so the first shrink, compaction, slab scrub and admission -- lazy module
    loads, first-touch costs: up to 35 ms once on a fresh box -- happen before
    the timed region) and ends high; the timed steps then alternate low / high
    every phase_steps steps."""
    lo = warmup // 2 if warmup >= 3 else 0
    out = [C4_WAVE[1]] * lo + [C4_WAVE[0]] * (warmup - lo)
    for k in range(steps):
        out.append(C4_WAVE[(k // max(1, phase_steps) + 1) % 2])
    return out


def c5_group(rank):
    """Models the reference placement put on group `rank % 8`, and their
    requests (prompt, output) in trace order (tests/golden/c5.json)."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c5.json")))
    g = f"gpu{rank % 8}"
    names = sorted(n for n, a in gold["assign"].items() if a == g)
    dt = {"fp16": 0, "fp8": 1, "int8": 2, "int4": 3}
    reqs = {n: [(int(r[3]), int(r[4])) for r in gold["requests"] if r[1] == n] for n in names}
    return names, [dt[n.split("_")[1]] for n in names], reqs


# ======================================================================
# CPU legs (oracle port / reference allocator) -- bounded samples
# ======================================================================
def oracle_qparams(dt, hkv=HKV):
    """Natural per-layer quant-param bytes of a block (precision.cpp:91-99 +
    DESIGN.md section 3): FP8 fp32 scale per (K|V, head), INT8 fp16 scale and
    INT4 fp16 (scale, zero) per (K|V, head, token)."""
    return {0: 0, 1: 2 * hkv * 4, 2: 2 * hkv * 16 * 2, 3: 2 * hkv * 16 * 4}[dt]


def cpu_sample(wl, seconds_target=10.0, nthreads=None):
    """fp64 OpenMP oracle decode over one layer of every model of the
    workload (B sequences at ctx), repeated until ~seconds_target.  Returns
    (GB/s, cores, sample text)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    nthreads = nthreads or oracle.NPROC
    rng = np.random.default_rng(0)
    hq, hkv = wl.get("hq", HQ), wl.get("hkv", HKV)
    B = min(wl["batch"], 16)
    ctx = wl["ctx"] if wl["ctx"] <= 2048 else wl["ctx"] // 2
    ctx = ctx or 512
    dts = wl["dts"] or (0, 1, 2, 3)
    res = []
    for dt in dts:
        f = oracle.fmt(dt, hkv, hq, D, 1, 16, oracle_qparams(dt, hkv))
        key = oracle.lib.orc_fmt_key(C.byref(f))
        nb = (ctx + 15) // 16
        img = np.zeros(B * nb * key, dtype=np.uint8)
        table = np.arange(B * nb, dtype=np.int32).reshape(B, nb)
        k = rng.standard_normal((B * ctx, hkv, D)).astype(np.float16).view(np.uint16)
        ts = np.repeat(np.arange(B, dtype=np.int32), ctx)
        tp = np.tile(np.arange(ctx, dtype=np.int32), B)
        sc = np.ones(2 * hkv, np.float32) if dt == 1 else None
        oracle.append(img, B * nb * key, B * nb, f, 0, k, k, ts, tp, table, sc)
        q = rng.standard_normal((B, hq, D)).astype(np.float16).view(np.uint16)
        cl = np.full(B, ctx, np.int32)
        res.append((img, table, f, q, cl, sc, oracle.decode_bytes(f, cl)))
    t0 = time.perf_counter()
    nbytes, reps = 0, 0
    while True:
        for img, table, f, q, cl, sc, by in res:
            oracle.paged_decode(img, img.size, table.size, f, 0, q, table, cl, 1 / math.sqrt(D),
                                sc, nthreads=nthreads)
            nbytes += by
        reps += 1
        if time.perf_counter() - t0 >= seconds_target:
            break
    dt_s = time.perf_counter() - t0
    names = "/".join(DT_NAMES[x] for x in dts)
    return (nbytes / dt_s / 1e9, nthreads,
            f"oracle fp64 decode, 1 layer of each model ({names}) x {reps} reps "
            f"({B} seqs x ctx {ctx}, {hq}q/{hkv}kv), {nthreads} OpenMP threads, {dt_s:.1f} s")


class CpuModel:
    """One model of the reference arm: a host block table over the reference
    allocator (simulator.cpp:33-40, 500-526, 561-578, 621), one layer of KV."""

    def __init__(self, oracle, dt, alloc, free, slab, hq, hkv, max_seqs, max_blocks):
        self.dt = dt
        self.f = oracle.fmt(dt, hkv, hq, D, 1, 16, oracle_qparams(dt, hkv))
        self.key = int(oracle.lib.orc_fmt_key(C.byref(self.f)))
        self.bps = slab // self.key
        self.alloc, self.free = alloc, free
        self.table = np.zeros((max_seqs, max_blocks), np.int32)
        self.blocks = [[] for _ in range(max_seqs)]
        self.cached = [0] * max_seqs
        self.sc = np.ones(2 * hkv, np.float32) if dt == 1 else None

    def grow(self, s, tokens):
        while len(self.blocks[s]) < (tokens + 15) // 16:
            h = self.alloc(self.key)
            if h is None:
                return False
            self.table[s, len(self.blocks[s])] = h[2]
            self.blocks[s].append(h)
        return True

    def admit(self, s, prompt):
        if not self.grow(s, prompt):
            self.release(s)
            return False
        self.cached[s] = prompt
        return True

    def release(self, s):
        for h in self.blocks[s]:
            self.free(h)
        self.blocks[s], self.cached[s] = [], 0


def run_reference():
    """--impl reference: the reference CPU path, rank 0 only, on the same
    workload and phase schedule as the GPU arm, one of the 32 layers per step
    (bounded sample): the reference SlabPool (oracle/_ref) for every block
    claim and release, the oracle port for append and attention.  The
    reference has no compaction, so none runs here."""
    if RANK != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    ref = oracle.ref_lib()
    nthreads = oracle.NPROC
    rng = np.random.default_rng(1)
    wl = WL
    hq, hkv = wl.get("hq", HQ), wl.get("hkv", HKV)
    if ARGS.workload == "c5":
        names, dts, reqs = c5_group(0)
    else:
        dts = wl["dts"]
    keys = [int(oracle.lib.orc_fmt_key(C.byref(oracle.fmt(dt, hkv, hq, D, 1, 16, oracle_qparams(dt, hkv)))))
            for dt in dts]
    total = ARGS.warmup + ARGS.steps
    if ARGS.workload == "c4":
        maxb, max_ctx = C4_WAVE[0], 2048 + total + 16
        slab, lcm = C4_SLAB // ARGS.layers, 0  # same blocks per slab as the 32-layer GPU pool
        targets = c4_phase_targets(ARGS.warmup, ARGS.steps, ARGS.phase_steps)
    elif ARGS.workload == "c5":
        maxb = wl["batch"]
        max_ctx = max(p + o for rs in reqs.values() for p, o in rs) + 16
        slab, lcm = math.lcm(*keys), 1
        targets = [maxb] * total
    else:
        maxb, max_ctx = wl["batch"], wl["ctx"] + total + 16
        slab, lcm = math.lcm(*keys), 1
        targets = [maxb] * total
    nb_max = (max_ctx + 15) // 16 + 1
    need = sum(maxb * nb_max * k for k in keys)
    nslabs = need * 5 // 4 // slab + 2 * len(keys) + 2
    kl = (C.c_uint64 * len(keys))(*keys)
    if ref is not None:
        rp = ref.ref_pool_create(nslabs * slab, slab, kl, len(keys), lcm)
        kind = "port"  # the attention / append half is the oracle port either way

        def alloc(key):
            out = (C.c_uint64 * 4)()
            return tuple(out) if ref.ref_try_alloc(rp, key, out) == 0 else None

        def free(h):
            assert ref.ref_free(rp, (C.c_uint64 * 4)(*h)) == 0
    else:
        op = oracle.OraclePool(nslabs * slab, slab, keys, bool(lcm))
        kind = "port"

        def alloc(key):
            st, h = op.alloc(key)
            return h if st == 0 else None

        def free(h):
            assert op.free(h) == 0
    img = np.zeros(nslabs * slab, dtype=np.uint8)
    models = [CpuModel(oracle, dt, alloc, free, slab, hq, hkv, maxb, nb_max) for dt in dts]
    src = rng.standard_normal((maxb * 2048 + 16, hkv, D)).astype(np.float16).view(np.uint16)
    q = rng.standard_normal((maxb, hq, D)).astype(np.float16).view(np.uint16)
    knew = rng.standard_normal((maxb, hkv, D)).astype(np.float16).view(np.uint16)
    queues = {i: 0 for i in range(len(models))}
    gen = [[0] * maxb for _ in models]

    def prompt_append(m, rows):
        if not rows:
            return 0
        ts = np.concatenate([np.full(m.cached[s], s, np.int32) for s in rows])
        tp = np.concatenate([np.arange(m.cached[s], dtype=np.int32) for s in rows])
        oracle.append(img, slab, m.bps, m.f, 0, src[:ts.size], src[:ts.size], ts, tp, m.table, m.sc)
        return ts.size

    def admit_rows(mi, m, rows):
        n_tok = 0
        for s in rows:
            if ARGS.workload == "c5":
                p, o = reqs[names[mi]][queues[mi] % len(reqs[names[mi]])]
                queues[mi] += 1
                gen[mi][s] = o
            else:
                p = int(rng.integers(512, 2049)) if ARGS.workload == "c4" else wl["ctx"]
            assert m.admit(s, p), "reference pool exhausted"
        n_tok += prompt_append(m, rows)
        return n_tok

    live = [list(range(targets[0])) for _ in models]
    for mi, m in enumerate(models):
        admit_rows(mi, m, live[mi])

    def step(target):
        nbytes = 0
        for mi, m in enumerate(models):
            if ARGS.workload == "c5":  # completed requests leave, the next ones of the trace join
                done = [s for s in live[mi] if gen[mi][s] <= 0]
                for s in done:
                    m.release(s)
                nbytes += m_append_bytes(m, admit_rows(mi, m, done))
            elif target < len(live[mi]):
                keep = sorted(rng.choice(live[mi], size=target, replace=False).tolist())
                for s in live[mi]:
                    if s not in keep:
                        m.release(s)
                live[mi] = keep
            elif target > len(live[mi]):
                new = [s for s in range(maxb) if s not in live[mi]][:target - len(live[mi])]
                nbytes += m_append_bytes(m, admit_rows(mi, m, new))
                live[mi] = sorted(live[mi] + new)
            rows = live[mi]
            for s in rows:  # growth rule, simulator.cpp:561-578
                assert m.grow(s, m.cached[s] + 1), "reference pool exhausted"
            pos = np.array([m.cached[s] for s in rows], np.int32)
            oracle.append(img, slab, m.bps, m.f, 0, knew[:len(rows)], knew[:len(rows)],
                          np.array(rows, np.int32), pos, m.table, m.sc)
            cl = np.zeros(maxb, np.int32)
            cl[rows] = pos + 1
            oracle.paged_decode(img, slab, m.bps, m.f, 0, q, m.table, cl, 1 / math.sqrt(D), m.sc,
                                nthreads=nthreads)
            nbytes += oracle.decode_bytes(m.f, cl[rows]) + m_append_bytes(m, len(rows))
            for s in rows:
                m.cached[s] += 1
                gen[mi][s] -= 1
        return nbytes

    def m_append_bytes(m, n_tok):
        per_tok = {0: 0, 1: 0, 2: 2 * hkv * 2, 3: 2 * hkv * 4}[m.dt]
        ts = hkv * D * 2 * {0: 16, 1: 8, 2: 8, 3: 4}[m.dt] // 8
        return n_tok * (2 * hkv * D * 2 + ts + per_tok + 12)

    for k in range(ARGS.warmup):
        step(targets[k])
    t0 = time.perf_counter()
    total_b = 0
    for k in range(ARGS.steps):
        total_b += step(targets[ARGS.warmup + k])
    dt_s = time.perf_counter() - t0
    gbs = total_b / dt_s / 1e9
    sample = (f"1 of {ARGS.layers} layers per step, every model; allocator = "
              f"{'reference SlabPool (oracle/_ref)' if ref is not None else 'oracle port'}, "
              f"append/attention = oracle port (fp64, {nthreads} threads); no compaction (the reference has none)")
    line = {"metric": "slab paged-decode attention HBM GB/s", "value": round(gbs, 3),
            "unit": "GB/s", "impl": "reference", "n_gpus": WORLD, "steps": ARGS.steps,
            "warmup": ARGS.warmup, "ms_per_step": round(dt_s / ARGS.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "/".join(DT_NAMES[x] for x in dts), "data": "synthetic",
            "config": config_dict(wl, maxb, max_ctx),
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": nthreads,
                             "kind": kind, "sample": sample, "cpu_model": cpu_model(),
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ======================================================================
# GPU leg
# ======================================================================
class Clocks:
    """nvidia-smi sampler during the timed region."""

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}



def format_sweep(peak):
    """K2 decode of each KV precision alone (Llama-3-8B shape, 8-layer CUDA
    graph of fused append+decode launches, per-launch average, algorithmic
    bytes) and K4 chunked prefill (whole 4k prompt, causal FLOPs vs the
    measured dense fp16/bf16 tensor peak).  Reported beside the headline; not
    part of the timed step."""
    import torch
    import paper_2509_06261_b200 as ks
    from paper_2509_06261_b200 import kv
    from paper_2509_06261_b200.engine import SlabModel
    from paper_2509_06261_b200.kv import KvDtype, KvFormat
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    tpeak = pk.get("bf16_tflops", 2250.0)
    Ls = 8
    res = {"decode": {}, "prefill": {}}

    def world(dt, B, ctx0):
        fmt = KvFormat(dt, HKV, HQ, D, Ls)
        slab = fmt.key * 16
        nb = (ctx0 + 15) // 16 + 1
        pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
        m = SlabModel(pool, fmt, B, nb)
        for s_ in range(B):
            assert m.admit(s_, ctx0)
        m.sync()
        return fmt, pool, m

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    for B, ctx0 in ((16, 2048), (64, 4096)):
        row = {}
        for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4):
            fmt, pool, m = world(dt, B, ctx0)
            ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
            qs = [torch.randn(B, HQ, D, dtype=torch.float16, device="cuda") for _ in range(Ls)]
            kn = torch.randn(B, HKV, D, dtype=torch.float16, device="cuda")
            sc = torch.ones(2 * HKV, device="cuda")
            ws = kv.DecodeWorkspace(pool, fmt, B)
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for layer in range(Ls):
                    kv.paged_decode(pool, fmt, layer, qs[layer], m.table, ctx, kv_scales=sc,
                                    workspace=ws, k_new=kn, v_new=kn)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=st):
                    for layer in range(Ls):
                        kv.paged_decode(pool, fmt, layer, qs[layer], m.table, ctx, kv_scales=sc,
                                        workspace=ws, k_new=kn, v_new=kn)
            ms = timed(g.replay, 10) / Ls
            by = fmt.decode_bytes([ctx0] * B)
            gbs = by / (ms / 1e3) / 1e9
            row[dt.name.lower()] = {"us": round(ms * 1e3, 2), "gbs": round(gbs, 1),
                                    "frac": round(gbs / peak, 4)}
            del g, pool
        res["decode"][f"B{B}_ctx{ctx0}"] = row
    nq = 4096
    for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4):
        fmt, pool, m = world(dt, 1, nq)
        ctx = torch.full((1,), nq, dtype=torch.int32, device="cuda")
        cu = torch.tensor([0, nq], dtype=torch.int32, device="cuda")
        q = torch.randn(nq, HQ, D, dtype=torch.float16, device="cuda")
        out = torch.empty_like(q)
        sc = torch.ones(2 * HKV, device="cuda")
        ms = timed(lambda: kv.paged_prefill(pool, fmt, 0, q, m.table, cu, ctx, nq, out=out,
                                            kv_scales=sc), 10)
        flops = 4.0 * D * HQ * nq * (nq + 1) / 2
        tf = flops / (ms / 1e3) / 1e12
        res["prefill"][dt.name.lower()] = {"workload": "1 seq, whole 4096-token prompt, causal",
                                           "us": round(ms * 1e3, 1), "tflops": round(tf, 1),
                                           "frac": round(tf / tpeak, 4), "bound": "tensor"}
        del pool
        # chunked prefill's steady state: a 64-token chunk per sequence at the end
        # of an 8k context (4 seqs; split-KV)
        Bc, cc, nc = 4, 8192, 64
        fmt, pool, m = world(dt, Bc, cc)
        ctx = torch.full((Bc,), cc, dtype=torch.int32, device="cuda")
        cu = torch.arange(0, (Bc + 1) * nc, nc, dtype=torch.int32, device="cuda")
        q = torch.randn(Bc * nc, HQ, D, dtype=torch.float16, device="cuda")
        out = torch.empty_like(q)
        ms = timed(lambda: kv.paged_prefill(pool, fmt, 0, q, m.table, cu, ctx, nc, out=out,
                                            kv_scales=sc), 10)
        flops = 4.0 * D * HQ * Bc * sum(cc - nc + i + 1 for i in range(nc))
        tf = flops / (ms / 1e3) / 1e12
        res["prefill"][dt.name.lower() + "_chunk64_ctx8k"] = {
            "workload": f"{Bc} seqs, 64-token chunk at ctx 8192, causal", "us": round(ms * 1e3, 1),
            "tflops": round(tf, 1), "frac": round(tf / tpeak, 4), "bound": "tensor"}
        del pool
    res["decode"]["note"] = ("K2 alone per KV precision: 8-layer graph of fused append+decode, "
                             "per-launch average, algorithmic bytes / measured HBM copy peak")
    return res


# ======================================================================
class Group:
    """The co-located models of one GPU: one slab pool, one engine table per
    model (engine.SlabModel over kvslab::SeqTable), the running batch of
    every model packed in rows 0..B-1, and per batch size two sets of flat
    step buffers (Q, new K/V per layer in; O per layer out) with one CUDA
    graph each.  Every model runs on its own stream (FineServe shares a GPU
    spatially between co-located engines)."""

    def __init__(self, dev, dts, maxb, max_ctx, layers, hq=HQ, hkv=HKV, slab=None, seed=0,
                 churn=False, max_prompt_tokens=0):
        import torch
        import paper_2509_06261_b200 as ks
        from paper_2509_06261_b200 import kv
        from paper_2509_06261_b200.engine import SlabModel
        from paper_2509_06261_b200.kv import KvDtype, KvFormat
        self.torch, self.kv = torch, kv
        self.dev, self.L, self.hq, self.hkv, self.maxb = dev, layers, hq, hkv, maxb
        self.fmts = [KvFormat(KvDtype(dt), hkv, hq, D, layers) for dt in dts]
        self.names = [DT_NAMES[dt] for dt in dts]
        keys = [f.key for f in self.fmts]
        aligned = slab is None
        self.slab = math.lcm(*keys) if aligned else slab
        self.max_blocks = (max_ctx + 15) // 16 + 1
        need = sum(maxb * self.max_blocks * k for k in keys) * (2 if churn else 1)
        nslabs = need * 5 // 4 // self.slab + 2 * len(keys) + 2
        self.pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * self.slab, self.slab, keys, aligned),
                                device=dev.index)
        self.models = [SlabModel(self.pool, f, maxb, self.max_blocks) for f in self.fmts]
        if churn:  # scatter the claims: holes all over the pool, other keys interleaved
            rng = np.random.default_rng(seed + 99)
            junk = [h for h in (self.pool.try_alloc_block(keys[i % len(keys)])
                                for i in range(maxb * len(keys) * 24)) if h]
            for i in rng.permutation(len(junk))[: len(junk) * 2 // 3]:
                self.pool.free_block(junk[i])
        self.streams = [torch.cuda.Stream(dev) for _ in self.fmts]
        self.ctx = [torch.zeros(maxb, dtype=torch.int32, device=dev) for _ in self.fmts]
        self.ctx_host = torch.zeros(len(self.fmts), maxb, dtype=torch.int32).pin_memory()
        self.ctx_ev = torch.cuda.Event()
        self.ctx_ev.record()
        self.scales = torch.full((2 * hkv,), 0.5, dtype=torch.float32, device=dev)
        self.ws = [kv.DecodeWorkspace(self.pool, f, maxb, stream=st) for f, st in zip(self.fmts, self.streams)]
        self.rng = np.random.default_rng(seed)
        self.bufs, self.graphs = {}, {}
        self.shares = {}
        self.B = 0
        self.n_launch_graph = {}
        # K1 prompt source (admissions): fp16 K and V rows, larger than L2
        self.max_prompt_tokens = max_prompt_tokens
        if max_prompt_tokens:
            # one prompt K/V source per model: co-located engines' prefills are
            # distinct data (a shared source let the four models' concurrent
            # K1 reads hit each other's L2 lines)
            self.src_m = [torch.randn(2, max_prompt_tokens, hkv, D, dtype=torch.float16, device=dev)
                          for _ in self.fmts]
            self.src = self.src_m[0]
            n = len(self.fmts)
            self.tok_host = torch.zeros(n, 2, max_prompt_tokens, dtype=torch.int32).pin_memory()
            self.tok_host_np = self.tok_host.numpy()  # same (pinned) memory
            self.arange_np = np.arange(max_prompt_tokens, dtype=np.int32)
            self.tok_dev = torch.zeros(n, 2, max_prompt_tokens, dtype=torch.int32, device=dev)
            self.tok_ev = [torch.cuda.Event() for _ in range(n)]
            for e in self.tok_ev:
                e.record()
        self.compactions, self.moves, self.slabs_freed = 0, 0, 0
        self.stranded_trace, self.frag_trace = [], []
        self.reb_marks = []  # (K1 bytes, K3 bytes, events) per phase change
        self.pending_prompts = None  # e2e: prompts of the next admission, drawn ahead
        self.step_ms_est = {}  # device ms per step by batch (+ "grow"), from the timed leg

    # ---- step buffers ----
    def buffers(self, B):
        if B in self.bufs:
            return self.bufs[B]
        torch, L, hq, hkv = self.torch, self.L, self.hq, self.hkv
        n = len(self.fmts)
        per_in, per_out = L * B * (hq + 2 * hkv) * D, L * B * hq * D
        sets = []
        for _ in range(2):
            inbuf = torch.randn(n * per_in, dtype=torch.float16, device=self.dev)
            outbuf = torch.empty(n * per_out, dtype=torch.float16, device=self.dev)
            q, kn, vn, out = [], [], [], []
            for mi in range(n):
                base = inbuf[mi * per_in:(mi + 1) * per_in]
                q.append([base[l * B * hq * D:(l + 1) * B * hq * D].view(B, hq, D) for l in range(L)])
                o0 = L * B * hq * D
                kn.append([base[o0 + l * B * hkv * D:o0 + (l + 1) * B * hkv * D].view(B, hkv, D)
                           for l in range(L)])
                o1 = o0 + L * B * hkv * D
                vn.append([base[o1 + l * B * hkv * D:o1 + (l + 1) * B * hkv * D].view(B, hkv, D)
                           for l in range(L)])
                ob = outbuf[mi * per_out:(mi + 1) * per_out]
                out.append([ob[l * B * hq * D:(l + 1) * B * hq * D].view(B, hq, D) for l in range(L)])
            sets.append(dict(inbuf=inbuf, outbuf=outbuf, q=q, kn=kn, vn=vn, out=out))
        self.bufs[B] = sets
        return sets

    # ---- one decode step on the device ----
    def device_step(self, B, X=0):
        """Per layer and model one fused K1+K2 launch (ks_paged_decode_append)
        on the model's stream, then ctx += 1 for the batch."""
        torch, kv = self.torch, self.kv
        bs = self.buffers(B)[X]
        main = torch.cuda.current_stream(self.dev)
        for st in self.streams:
            st.wait_stream(main)
        for layer in range(self.L):
            for mi, m in enumerate(self.models):
                kv.paged_decode(self.pool, m.fmt, layer, bs["q"][mi][layer], m.table, self.ctx[mi][:B],
                                out=bs["out"][mi][layer], kv_scales=self.scales, workspace=self.ws[mi],
                                k_new=bs["kn"][mi][layer], v_new=bs["vn"][mi][layer],
                                stream=self.streams[mi])
        for mi, st in enumerate(self.streams):
            with torch.cuda.stream(st):
                self.ctx[mi][:B].add_(1)
            main.wait_stream(st)

    def graph(self, B, X=0):
        k = (B, X)
        if k not in self.graphs:
            torch, kv = self.torch, self.kv
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.dev)
            cap.wait_stream(torch.cuda.current_stream(self.dev))
            n0 = kv.launch_count()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    self.device_step(B, X)
            torch.cuda.current_stream(self.dev).wait_stream(cap)
            self.n_launch_graph[k] = kv.launch_count() - n0
            self.graphs[k] = g
        return self.graphs[k]

    # ---- host side of a step ----
    def host_step(self):
        """Growth rule for this step's token (simulator.cpp:561-578) and the
        table delta upload; returns the step's algorithmic bytes (K1+K2)."""
        main = self.torch.cuda.current_stream(self.dev)
        rows = list(range(self.B))
        nbytes = 0
        for m in self.models:
            if m.step(rows):
                raise RuntimeError("pool exhausted: a sequence stalled")
            m.sync(main)
            nbytes += self.L * (m.fmt.decode_bytes(m.ctx_lens(self.B)) + m.fmt.append_bytes(self.B))
        return nbytes

    def set_ctx(self):
        """Device ctx of the rows 0..B-1 = cached + 1 (the token the next step writes)."""
        torch = self.torch
        self.ctx_ev.synchronize()  # the previous upload has read the pinned buffer
        main = torch.cuda.current_stream(self.dev)
        for mi, m in enumerate(self.models):
            self.ctx_host[mi, :self.B] = torch.tensor(m.ctx_lens(self.B, plus=1), dtype=torch.int32)
            self.ctx[mi][:self.B].copy_(self.ctx_host[mi, :self.B], non_blocking=True)
        self.ctx_ev.record(main)

    def admit_rows(self, mi, rows, prompts, src_fn=None, stream=None):
        """Prefill claim (simulator.cpp:500-526) + K1 append of the prompts'
        K/V for every layer (src_fn(T, mi): the e2e leg's copy of the T prompt
        tokens' K/V from host memory).  Returns the K1 algorithmic bytes."""
        T = self.prepare_admission(mi, rows, prompts)
        return self.launch_admission(mi, T, src_fn, stream)

    def prepare_admission(self, mi, rows, prompts):
        """Host half of an admission: the claims, the table delta upload and
        the token -> (row, position) lists (pinned staging buffer, reused once
        its previous upload finished), all on the main stream.  Returns T."""
        torch = self.torch
        m = self.models[mi]
        main = torch.cuda.current_stream(self.dev)
        for s, p in zip(rows, prompts):
            if not m.admit(s, int(p)):
                raise RuntimeError("pool exhausted at admission")
        m.sync(main)
        T = int(sum(prompts))
        if T == 0:
            return 0
        assert T <= self.max_prompt_tokens
        self.tok_ev[mi].synchronize()
        # numpy writes into the pinned buffer (one memcpy on this thread: a
        # torch slice copy went through the intra-op thread pool and was
        # measured stalling 4-7 ms at a time)
        hv = self.tok_host_np[mi]
        hv[0, :T] = np.repeat(np.asarray(rows, np.int32), np.asarray(prompts))
        o = 0
        for p in prompts:
            hv[1, o:o + p] = self.arange_np[:p]
            o += p
        for j in range(2):  # contiguous pinned rows: asynchronous DMA
            self.tok_dev[mi, j, :T].copy_(self.tok_host[mi, j, :T], non_blocking=True)
        self.tok_ev[mi].record(main)
        return T

    def launch_admission(self, mi, T, src_fn=None, stream=None):
        """Device half: the K1 launches of every layer on `stream` (the
        model's own: co-located engines prefill side by side, as they decode),
        ordered after the main stream's uploads."""
        if T == 0:
            return 0
        torch, kv = self.torch, self.kv
        m = self.models[mi]
        main = torch.cuda.current_stream(self.dev)
        ts, tp = self.tok_dev[mi, 0, :T], self.tok_dev[mi, 1, :T]
        src = self.src_m[mi] if src_fn is None else src_fn(T, mi)
        st = main if stream is None else stream
        if st is not main:
            st.wait_stream(main)
        for layer in range(self.L):
            kv.kv_append(self.pool, m.fmt, layer, src[0, :T], src[1, :T], ts, tp, m.table,
                         self.scales, stream=st)
        return self.L * m.fmt.append_bytes(T)

    def stranded(self):
        st = self.pool.snapshot_stats()
        return st.free_block_bytes / max(1, st.allocated_bytes + st.free_block_bytes)

    def rebalance(self, target, src_fn=None):
        """Phase change of the c4 wave: shrink (random survivors packed into
        rows 0..target-1) or grow (admissions with prompts U[512, 2048]); then
        K3 compaction of every key when stranded bytes exceed the trigger.
        Returns (K1 bytes, K3 bytes)."""
        k1 = k3 = 0
        if target == self.B:
            return 0, 0
        main = self.torch.cuda.current_stream(self.dev)
        ev = [self.torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(main)
        for mi, m in enumerate(self.models):
            if target < self.B:
                keep = sorted(self.rng.choice(self.B, size=target, replace=False).tolist())
                ks_ = set(keep)
                for s in range(self.B):
                    if s not in ks_:
                        m.release(s)
                m.condense(keep)
            else:
                # model by model, so the device runs model i's K1 while the
                # host prepares model i+1 (preparing all four first left the
                # GPU idle for the whole host half: measured 0.5-5 ms per grow)
                rows = list(range(self.B, target))
                if self.pending_prompts is not None:  # e2e: drawn (and copied) ahead
                    prompts = self.pending_prompts[mi]
                    assert len(prompts) == len(rows)
                else:
                    prompts = self.rng.integers(512, 2049, size=len(rows)).tolist()
                T = self.prepare_admission(mi, rows, prompts)
                k1 += self.launch_admission(mi, T, src_fn, stream=self.streams[mi])
        # the phase change's small host->device uploads (tables, token lists)
        # are all issued: bulk copies on other streams may go after this
        self.uploads_done = self.torch.cuda.Event()
        self.uploads_done.record(main)
        for st in self.streams:  # every model's admission K1 done before compaction / the step
            main.wait_stream(st)
        self.B = target
        for m in self.models:
            m.sync(main)
        ev[1].record(main)
        strd = self.stranded()
        self.stranded_trace.append(round(strd, 3))
        if strd > C4_TRIGGER:
            for m in self.models:
                n, fr = m.compact(stream=main)
                self.moves += n
                self.slabs_freed += fr
                k3 += 2 * n * m.key
            self.compactions += 1
        ev[2].record(main)
        self.reb_marks.append((k1, k3, ev))
        self.frag_trace.append(sum(m.internal_frag_bytes() for m in self.models))
        self.set_ctx()
        return k1, k3

    def kernel_times(self, reps=5):
        """Every model's fused K1+K2 launch alone (whole GPU), as a graph of
        its L layer launches at the current batch: (bytes, ms per launch)."""
        torch, kv = self.torch, self.kv
        B = self.B
        bs = self.buffers(B)[0]
        main = torch.cuda.current_stream(self.dev)
        saved = [self.shares.get(nm, 0) for nm in self.names]
        out = {}
        for mi, m in enumerate(self.models):
            kv.set_decode_sm_share(self.pool, m.key, 0)
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.dev)
            cap.wait_stream(main)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    for layer in range(self.L):
                        kv.paged_decode(self.pool, m.fmt, layer, bs["q"][mi][layer], m.table,
                                        self.ctx[mi][:B], out=bs["out"][mi][layer], kv_scales=self.scales,
                                        workspace=self.ws[mi], k_new=bs["kn"][mi][layer],
                                        v_new=bs["vn"][mi][layer])
            main.wait_stream(cap)
            g.replay()
            torch.cuda.synchronize(self.dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main)
            for _ in range(reps):
                g.replay()
            b.record(main)
            torch.cuda.synchronize(self.dev)
            ms = a.elapsed_time(b) / (reps * self.L)
            cl = [int(x) for x in self.ctx[mi][:B].cpu().tolist()]
            by = m.fmt.decode_bytes(cl) + m.fmt.append_bytes(B)
            out[self.names[mi]] = (by, ms)
            del g
        for m, sh in zip(self.models, saved):
            kv.set_decode_sm_share(self.pool, m.key, sh)
        return out

    def k1_times(self, per_row=512, reps=5):
        """Every model's K1 alone (ks_kv_append, one layer, per_row tokens of
        each of rows 0..B-1 rewritten in place, the whole GPU): (bytes, ms)."""
        torch, kv = self.torch, self.kv
        B = self.B
        T = min(B * per_row, self.max_prompt_tokens)
        per_row = T // B
        ts = torch.arange(B, dtype=torch.int32, device=self.dev).repeat_interleave(per_row)
        tp = torch.arange(per_row, dtype=torch.int32, device=self.dev).repeat(B)
        main = torch.cuda.current_stream(self.dev)
        out = {}
        for mi, m in enumerate(self.models):
            fn = lambda: kv.kv_append(self.pool, m.fmt, 0, self.src[0, :B * per_row], self.src[1, :B * per_row],
                                      ts, tp, m.table, self.scales, stream=main)
            fn()
            torch.cuda.synchronize(self.dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main)
            for _ in range(reps):
                fn()
            b.record(main)
            torch.cuda.synchronize(self.dev)
            out[self.names[mi]] = (m.fmt.append_bytes(B * per_row), a.elapsed_time(b) / reps)
        return out

    def tune_shares(self, B):
        """MPS-style spatial split (ks_set_decode_sm_share): a few candidate
        splits of the SMs between the co-located models (KV bytes per token,
        the consumer-bound INT4 weighted 1-3x; all SMs, 92 % or 84 %; or no
        partition), each captured as an 8-layer graph at batch B and timed by
        replay, as the step graphs will run it; the fastest is kept."""
        torch, kv = self.torch, self.kv
        n = len(self.models)
        if n == 1:
            return None
        nsm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        wbytes = {0: 4096.0, 1: 2052.0, 2: 2112.0, 3: 1088.0}
        cands = set()
        for w4 in (1.0, 2.0, 3.0):
            ww = [wbytes[int(f.kv_dtype)] * (w4 if int(f.kv_dtype) == 3 else 1.0) for f in self.fmts]
            for tot in (nsm, int(nsm * 0.92), int(nsm * 0.84)):
                for skew in (0.9, 1.0, 1.1) if n == 2 else (1.0,):
                    w0 = [ww[0] * skew] + ww[1:]
                    cands.add(tuple(max(8, min(tot - 8, int(tot * x / sum(w0)))) for x in w0))
        cands.add(tuple([nsm] * n))  # no partition: every model's grid spans the GPU
        # the consumer-bound INT4 model fenced into k SMs, the HBM-bound
        # models sharing the rest without a partition among themselves
        if any(int(f.kv_dtype) == 3 for f in self.fmts) and n > 1:
            for k4 in (24, 30, 37, 44, 52):
                for rest in (nsm - k4, nsm - k4 + 12, nsm):
                    cands.add(tuple(k4 if int(f.kv_dtype) == 3 else min(nsm, rest) for f in self.fmts))
        if n > 2:  # proportional splits that overlap (caps summing past the SM count)
            ww = [wbytes[int(f.kv_dtype)] * (2.0 if int(f.kv_dtype) == 3 else 1.0) for f in self.fmts]
            for over in (1.1, 1.2, 1.35, 1.5):
                tot = nsm * over
                cands.add(tuple(max(8, min(nsm, int(tot * x / sum(ww)))) for x in ww))
        bs = self.buffers(B)[0]
        main = torch.cuda.current_stream(self.dev)
        times = {}

        def few():
            cur = torch.cuda.current_stream(self.dev)  # the capture stream
            for st in self.streams:
                st.wait_stream(cur)
            for layer in range(min(8, self.L)):
                for mi, m in enumerate(self.models):
                    kv.paged_decode(self.pool, m.fmt, layer, bs["q"][mi][layer], m.table,
                                    self.ctx[mi][:B], out=bs["out"][mi][layer], kv_scales=self.scales,
                                    workspace=self.ws[mi], stream=self.streams[mi])
            for st in self.streams:
                cur.wait_stream(st)
        for c in sorted(cands):  # each split as the graphs will run it: captured, replayed
            for m, sh in zip(self.models, c):
                kv.set_decode_sm_share(self.pool, m.key, sh)
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.dev)
            cap.wait_stream(main)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    few()
            main.wait_stream(cap)
            g.replay()
            torch.cuda.synchronize(self.dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = []
            for _ in range(5):  # best of 5 timed replays (single replays are noisy)
                a.record(main)
                g.replay()
                b.record(main)
                torch.cuda.synchronize(self.dev)
                reps.append(a.elapsed_time(b))
            times[c] = min(reps)
            del g
        pick = min(times, key=times.get)
        for m, sh in zip(self.models, pick):
            kv.set_decode_sm_share(self.pool, m.key, sh)
        self.shares = dict(zip(self.names, pick))
        return {"split": dict(zip(self.names, pick)),
                "autotune_ms": {"+".join(map(str, k)): round(v, 3) for k, v in times.items()}}


def time_steps(grp, targets, clocks_index=None, e2e=None, eager=False):
    """Runs len(targets) steps (phase changes at batch changes) and times them
    on the device.  e2e: host buffers for the public-API leg (inputs copied in
    and outputs copied back every step, two copy streams, double-buffered).
    Returns (ms, bytes, decode tokens, launches, h2d bytes, d2h bytes, clocks)."""
    torch, kv = grp.torch, grp.kv
    main = torch.cuda.current_stream(grp.dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nbytes = tokens = h2d = d2h = 0
    n0 = kv.launch_count()
    graph_launches = 0
    marks = []
    clk = Clocks(clocks_index) if clocks_index is not None else None
    if clk:
        clk.__enter__()
    torch.cuda.synchronize(grp.dev)
    if e2e:
        up, down = e2e["up"], e2e["down"]
    e0.record(main)
    # e2e: the admitted prompts' K/V come from host memory too.  They are
    # pipelined like the step inputs: two device staging slots per model
    # (alternate admissions), the next admission's prompts drawn right after
    # the previous one and their K/V copied in chunks issued on the copy
    # stream right after each step's own input copy -- sized to the PCIe time
    # the step's compute leaves (about 50 GB/s x the step's device time,
    # less the next step's inputs) -- so the copies overlap the steps instead
    # of stalling the admission.  The step waits only for its own inputs.
    pf = None
    n_models = len(grp.models)
    tok_bytes = grp.hkv * D * 2  # one token's K (or V) rows, fp16
    pcie = 50e9  # bytes/s budget per second of device time (H2D measured 55 GB/s)
    est_ms = {b: grp.step_ms_est.get(b, 4.3 * b / 64) for b in set(targets)}
    est_ms["grow"] = grp.step_ms_est.get("grow", 10.0)

    def next_grow(k):
        return next((j for j in range(k, len(targets)) if targets[j] > (targets[j - 1] if j else grp.B)), None)

    def plan_prefetch(k):
        """Prompts for the next admission at or after step k, and their copy queue."""
        g = next_grow(k)
        if g is None:
            return None
        before = targets[g - 1] if g else grp.B
        prompts = {mi: grp.rng.integers(512, 2049, size=targets[g] - before).tolist() for mi in range(n_models)}
        slot = e2e["slot"]
        queue = [[mi, i, 0, int(sum(prompts[mi]))] for mi in range(n_models) for i in range(2)]
        return {"g": g, "prompts": prompts, "queue": queue, "slot": slot, "waited": set(),
                "ready": [torch.cuda.Event() for _ in range(n_models)]}

    def pump(limit_bytes):
        """Issue up to `limit_bytes` of the pending prompt copies on `up`."""
        nonlocal h2d
        limit = int(limit_bytes // tok_bytes)
        while pf["queue"] and limit > 0:
            q = pf["queue"][0]
            mi, i, lo, hi = q
            if mi not in pf["waited"]:  # the admission before last is done with this slot
                up.wait_event(e2e["src_free"][pf["slot"]][mi])
                pf["waited"].add(mi)
            n = min(hi - lo, limit)
            e2e["src_dev"][pf["slot"]][mi][i][lo:lo + n].copy_(e2e["src_host"][i][lo:lo + n], non_blocking=True)
            h2d += n * tok_bytes
            q[2] += n
            limit -= n
            if q[2] == hi:
                pf["queue"].pop(0)
                if i == 1:
                    pf["ready"][mi].record(up)

    for k, B in enumerate(targets):
        X = k & 1
        src_fn = None
        if e2e:
            hin, hout, free_ev = e2e["host"](B)
            bs = grp.buffers(B)[X]
            with torch.cuda.stream(up):
                if pf is None and grp.max_prompt_tokens and B > grp.B:
                    pf = plan_prefetch(k)  # an admission nothing was copied ahead for
                if pf is not None and k == pf["g"]:
                    pump(1 << 62)  # whatever did not fit in the earlier steps
                up.wait_event(free_ev[X])
                bs["inbuf"].copy_(hin[X], non_blocking=True)
                h2d += bs["inbuf"].numel() * 2
                in_ready = torch.cuda.Event()
                in_ready.record(up)
            main.wait_event(in_ready)

            if pf is not None and k == pf["g"]:
                grp.pending_prompts = pf["prompts"]
                src_slot, src_ready = pf["slot"], pf["ready"]

                def src_fn(T, mi):  # this admission's prompts, copied ahead
                    grp.streams[mi].wait_event(src_ready[mi])
                    return e2e["src_dev"][src_slot][mi]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(main)
        grew = phase_changed = False
        if B != grp.B:
            phase_changed = True
            grew = B > grp.B
            k1, k3 = grp.rebalance(B, src_fn)
            nbytes += k1 + k3
            if src_fn is not None:  # this slot is free again after these K1
                for mi, st in enumerate(grp.streams):
                    e2e["src_free"][src_slot][mi].record(st)
                grp.pending_prompts = None
                e2e["slot"] ^= 1
                pf = None
        ev[1].record(main)
        marks.append((B, ev))
        nbytes += grp.host_step()
        tokens += len(grp.models) * B
        if eager:
            grp.device_step(B, X if e2e else 0)
        else:
            grp.graph(B, X if e2e else 0).replay()
            graph_launches += grp.n_launch_graph[(B, X if e2e else 0)]
        ev[2].record(main)
        if e2e and grp.max_prompt_tokens:
            # the next admission's prompts ride in the PCIe time this step's
            # compute leaves (after its own inputs, before the next step's)
            if pf is None:
                pf = plan_prefetch(k + 1)
            if pf is not None and k + 1 < pf["g"]:
                nxt = targets[k + 1]
                # (half the admission's time: copies beside the four models'
                # K1 were measured slowing it; 0 / 0.5 / 1 gave 3.94 / 4.07 / 4.0 TB/s)
                budget = pcie * (est_ms[B] + (0.5 * est_ms["grow"] if grew else 0.0)) / 1e3 \
                    - grp.buffers(nxt)[0]["inbuf"].numel() * 2
                with torch.cuda.stream(up):
                    if phase_changed:
                        # a bulk copy queued ahead of the phase change's small
                        # uploads on the copy engine stalled the admission 13 ms
                        up.wait_event(grp.uploads_done)
                    pump(max(0.0, budget))
        if e2e:
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(down):
                down.wait_event(done)
                hout[X].copy_(bs["outbuf"], non_blocking=True)
                d2h += bs["outbuf"].numel() * 2
                free_ev[X].record(down)
    if e2e:
        main.wait_stream(down)
    e1.record(main)
    torch.cuda.synchronize(grp.dev)
    if clk:
        clk.__exit__()
    ms = e0.elapsed_time(e1)
    launches = kv.launch_count() - n0 + graph_launches
    # device-time breakdown: phase changes (admission K1, compaction) vs steps per batch size
    bd = {"phase_change_ms": round(sum(e[0].elapsed_time(e[1]) for _, e in marks), 3)}
    reb = [m for m in grp.reb_marks if m[2][0].query()]
    grp.reb_marks = []
    if reb:
        adm = sum(e[0].elapsed_time(e[1]) for _, _, e in reb)
        cmp_ = sum(e[1].elapsed_time(e[2]) for _, _, e in reb)
        bd["admission_ms"] = round(adm, 3)
        bd["phase_change_ms_each"] = [round(e[0].elapsed_time(e[1]), 3) for _, _, e in reb]
        bd["admission_k1_gbs"] = round(sum(k for k, _, _ in reb) / max(adm, 1e-9) / 1e6, 1)
        bd["compaction_ms"] = round(cmp_, 3)
        k3b = sum(k for _, k, _ in reb)
        bd["compaction_gbs"] = round(k3b / max(cmp_, 1e-9) / 1e6, 1) if k3b else None
    for b in sorted({b for b, _ in marks}):
        t = [e[1].elapsed_time(e[2]) for bb, e in marks if bb == b]
        bd[f"step_ms_B{b}"] = round(float(np.mean(t)), 4)
    time_steps.breakdown = bd
    return ms, nbytes, tokens, launches, h2d, d2h, (clk.summary() if clk else None)


def make_e2e(grp):
    """Pinned host buffers per batch size (two sets) for the e2e leg."""
    torch = grp.torch
    cache = {}

    def host(B):
        if B not in cache:
            sets = grp.buffers(B)
            hin = [torch.empty(sets[0]["inbuf"].numel(), dtype=torch.float16).pin_memory() for _ in range(2)]
            for h, s in zip(hin, sets):
                h.copy_(s["inbuf"].cpu())
            hout = [torch.empty(sets[0]["outbuf"].numel(), dtype=torch.float16).pin_memory() for _ in range(2)]
            ev = [torch.cuda.Event(), torch.cuda.Event()]
            for e in ev:
                e.record()
            cache[B] = (hin, hout, ev)
        return cache[B]

    e2e = {"host": host, "up": torch.cuda.Stream(grp.dev), "down": torch.cuda.Stream(grp.dev)}
    if grp.max_prompt_tokens:
        e2e["src_host"] = [grp.src[i].cpu().pin_memory() for i in range(2)]
        # two staging slots per model: admissions alternate, so the next one's
        # prompts can be copied while the last one's K1 still reads its slot
        e2e["src_dev"] = [[torch.zeros_like(grp.src) for _ in grp.models] for _ in range(2)]
        e2e["src_free"] = [[torch.cuda.Event() for _ in grp.models] for _ in range(2)]
        for sl in e2e["src_free"]:
            for e in sl:
                e.record()
        e2e["slot"] = 0
    return e2e


def reduce_over_ranks(ms, nbytes, tokens):
    """max time, summed bytes and tokens over ranks (no collective on the
    data path: this is the bench's bookkeeping only)."""
    if WORLD == 1:
        return ms, nbytes, tokens
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
    s = torch.tensor([float(nbytes), float(tokens)], dtype=torch.float64, device=t.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t.item()), float(s[0].item()), float(s[1].item())


def build_group(name, dev, seed):
    """The GPU arm's Group for a workload and its step schedule."""
    wl = WORKLOADS[name]
    total = ARGS.warmup + ARGS.steps
    # the e2e leg runs two of the timed schedule back to back: its prompt
    # copies are pipelined one admission ahead, and the leg's first admission
    # (nothing before it to overlap with) would otherwise weigh as much as a
    # steady-state one
    e2e_steps = max(8, 2 * ARGS.steps)
    if name == "c4":
        max_ctx = 2048 + 3 * (total + e2e_steps) + 16
        grp = Group(dev, wl["dts"], C4_WAVE[0], max_ctx, ARGS.layers, slab=C4_SLAB, seed=seed,
                    max_prompt_tokens=C4_WAVE[0] * 2048)
        grp.rebalance(C4_WAVE[0])  # the first batch (K1 prefill of every layer), untimed
        return grp, c4_phase_targets(ARGS.warmup, ARGS.steps, ARGS.phase_steps), \
            c4_phase_targets(0, e2e_steps, ARGS.phase_steps)
    B, ctx0 = wl["batch"], wl["ctx"]
    layers = wl.get("layers", ARGS.layers)
    grp = Group(dev, wl["dts"], B, ctx0 + 3 * (total + e2e_steps) + 16, layers, hq=wl.get("hq", HQ),
                hkv=wl.get("hkv", HKV), seed=seed, churn=True, max_prompt_tokens=B * ctx0)
    for mi in range(len(grp.models)):  # the whole batch, K1 prefill of every layer, untimed
        grp.admit_rows(mi, list(range(B)), [ctx0] * B)
    grp.B = B
    grp.set_ctx()
    return grp, [B] * total, [B] * e2e_steps


def measure(name, dev, clocks_index, with_e2e=True, tune=True):
    """One workload on this rank: timed graph steps, the e2e legs, the
    per-model kernel roofline.  Returns a dict of raw numbers."""
    import torch
    grp, targets, e2e_targets = build_group(name, dev, seed=1234 + RANK)
    # the SM split is baked into each captured graph (grid sizes): tune it
    # per batch size of the schedule, then capture that size's graphs
    shares = {}
    for B in sorted(set(targets + e2e_targets), reverse=True):  # capture outside the timed region
        if tune:
            shares[f"B{B}"] = grp.tune_shares(B)
        grp.graph(B, 0)
        if with_e2e:
            grp.graph(B, 1)
    shares = shares or None
    warm, timed = targets[:ARGS.warmup], targets[ARGS.warmup:]
    time_steps(grp, warm)
    # the serving loop's long-lived objects out of the cyclic collector: a
    # full collection inside a host-side admission was measured stalling the
    # device 4-6 ms (gc.freeze, as serving engines do)
    import gc
    gc.collect()
    gc.freeze()
    if WORLD > 1:
        import torch.distributed as dist
        dist.barrier()
    c0, m0, s0 = grp.compactions, grp.moves, grp.slabs_freed
    st0 = len(grp.stranded_trace)
    ms, nbytes, tokens, launches, _, _, clk = time_steps(grp, timed, clocks_index=clocks_index)
    bd = time_steps.breakdown
    grp.step_ms_est = {b: bd[f"step_ms_B{b}"] for b in set(timed) if f"step_ms_B{b}" in bd}
    if bd.get("phase_change_ms_each"):
        grp.step_ms_est["grow"] = max(bd["phase_change_ms_each"])
    res = dict(ms=ms, bytes=nbytes, tokens=tokens, launches=launches, clocks=clk, shares=shares,
               breakdown=time_steps.breakdown,
               compactions=grp.compactions - c0, moves=grp.moves - m0, slabs_freed=grp.slabs_freed - s0,
               stranded=grp.stranded_trace[st0:], frag=grp.frag_trace[st0:], B=timed)
    if with_e2e:
        e2e = make_e2e(grp)
        for B in set(e2e_targets):  # pinned host buffers before the timed region
            e2e["host"](B)
        r = time_steps(grp, e2e_targets, e2e=e2e)
        res["e2e"] = dict(ms=r[0], bytes=r[1], h2d=r[4] / len(e2e_targets), d2h=r[5] / len(e2e_targets),
                          breakdown=time_steps.breakdown, steps=len(e2e_targets))
        r = time_steps(grp, e2e_targets, e2e=e2e, eager=True)
        res["e2e_eager"] = dict(ms=r[0], bytes=r[1], h2d=r[4] / len(e2e_targets), d2h=r[5] / len(e2e_targets))
    if max(targets) != grp.B:  # the kernels at the workload's largest batch
        grp.rebalance(max(targets))
    res["kernels"] = grp.kernel_times()
    res["k1"] = grp.k1_times() if grp.max_prompt_tokens else {}
    res["kernel_batch"] = grp.B
    res["kernel_ctx"] = int(np.mean(grp.models[0].ctx_lens(grp.B)))
    res["names"] = grp.names
    res["hkv"] = grp.hkv
    res["internal_frag_bytes"] = sum(m.internal_frag_bytes() for m in grp.models)
    res["pool"] = dict(slab_bytes=grp.slab, slabs=grp.pool.slab_count(),
                       residue_bytes=grp.pool.snapshot_stats().slab_residue_bytes,
                       scrubbed_bytes_total=grp.kv.scrubbed_bytes(grp.pool))
    del grp
    torch.cuda.synchronize(dev)
    return res


def summarise(name, r, peak, peak_kind, world):
    """The contract's JSON fields for one workload (rank 0, reduced numbers)."""
    ms, nbytes, tokens = reduce_over_ranks(r["ms"], r["bytes"], r["tokens"])
    steps = len(r["B"])
    value = nbytes / (ms / 1e3) / 1e9
    kernels = {k: {"bytes": int(v[0]), "us": round(v[1] * 1e3, 2),
                   "gbs": round(v[0] / (v[1] / 1e3) / 1e9, 1),
                   "frac": round(v[0] / (v[1] / 1e3) / 1e9 / peak, 4)} for k, v in r["kernels"].items()}
    dom = "fp16" if "fp16" in kernels else next(iter(kernels))
    by, pl = r["kernels"][dom]
    achieved = by / (pl / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(f"{name}_decode_{dom}", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    out = {
        "value": round(value, 2), "ms_per_step": round(ms / steps, 4),
        "decode_tok_s": round(tokens / (ms / 1e3), 1),
        "decode_tok_s_per_gpu": round(tokens / (ms / 1e3) / world, 1),
        "frac_of_peak": round(value / world / peak, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": f"paged_decode_kernel<{dom.upper()}> fused append+decode, one layer of "
                               f"{r['kernel_batch']} seqs x ctx~{r['kernel_ctx']}, {r.get('hkv', HKV)} kv heads",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "frac_of_8TBps": round(achieved / 8000.0, 4)},
        "kernels": kernels,
        "k1_append": {k: {"bytes": int(v[0]), "us": round(v[1] * 1e3, 2),
                          "gbs": round(v[0] / (v[1] / 1e3) / 1e9, 1),
                          "frac": round(v[0] / (v[1] / 1e3) / 1e9 / peak, 4)} for k, v in r.get("k1", {}).items()},
        "breakdown": r.get("breakdown"),
        "sm_share": r["shares"],
        "gpu_launches": int(r["launches"]),
    }
    if "e2e" in r:
        e = r["e2e"]
        ems, eb, _ = reduce_over_ranks(e["ms"], e["bytes"], 0)
        ee = r["e2e_eager"]
        xms, xb, _ = reduce_over_ranks(ee["ms"], ee["bytes"], 0)
        out["e2e"] = {"value": round(eb / (ems / 1e3) / 1e9, 2), "unit": "GB/s",
                      "h2d_bytes_per_step": int(e["h2d"]), "d2h_bytes_per_step": int(e["d2h"]),
                      "mode": "CUDA-graph replay of each step; inputs from pinned host memory, outputs back",
                      "steps": e.get("steps"), "ms": round(ems, 3), "breakdown": e.get("breakdown"),
                      "eager": {"value": round(xb / (xms / 1e3) / 1e9, 2), "unit": "GB/s",
                                "mode": "per-layer ks_paged_decode_append calls from Python (ctypes), no graph"}}
    if name == "c4":
        out["c4"] = {"phases_B": sorted(set(r["B"]), reverse=True), "phase_steps": ARGS.phase_steps,
                     "compactions": r["compactions"], "moves": r["moves"], "slabs_freed": r["slabs_freed"],
                     "stranded_at_phase_start": r["stranded"],
                     "internal_frag_bytes_per_phase": r["frag"],
                     "trigger": C4_TRIGGER, "pool": r["pool"]}
    out["internal_frag_bytes"] = r["internal_frag_bytes"]
    out["clocks"] = r["clocks"]
    return out


def run_c5(dev, clocks_index):
    """BASELINE configs[4] on this rank: the models the reference placed on
    group `rank` (tests/golden/c5.json), one pool, each model's running batch
    refilled from its requests of the reference trace (cycled): completed
    requests release their blocks, new ones claim their prompt blocks and get
    their prompt K/V appended (K1, all layers); decode steps as in c4."""
    import torch
    names, dts, reqs = c5_group(RANK)
    maxb = WORKLOADS["c5"]["batch"]
    max_ctx = max(p + o for rs in reqs.values() for p, o in rs) + 16
    grp = Group(dev, dts, maxb, max_ctx, ARGS.layers, seed=77 + RANK,
                max_prompt_tokens=maxb * max(p for rs in reqs.values() for p, _ in rs))
    qi = [0] * len(names)
    left = [[0] * maxb for _ in names]

    def refill(mi, rows):
        ps = []
        for s in rows:
            p, o = reqs[names[mi]][qi[mi] % len(reqs[names[mi]])]
            qi[mi] += 1
            left[mi][s] = o
            ps.append(p)
        return grp.admit_rows(mi, rows, ps) if rows else 0

    for mi in range(len(names)):
        refill(mi, list(range(maxb)))
    grp.B = maxb
    grp.set_ctx()
    grp.graph(maxb)
    main = torch.cuda.current_stream(dev)

    def steps(n, clk=None):
        nbytes = tokens = 0
        for _ in range(n):
            changed = False
            for mi, m in enumerate(grp.models):
                done = [s for s in range(maxb) if left[mi][s] <= 0]
                for s in done:
                    m.release(s)
                nbytes += refill(mi, done)
                changed |= bool(done)
            if changed:
                grp.set_ctx()
            nbytes += grp.host_step()
            tokens += len(grp.models) * maxb
            grp.graph(maxb).replay()
            for mi in range(len(grp.models)):
                for s in range(maxb):
                    left[mi][s] -= 1
        return nbytes, tokens

    steps(ARGS.warmup)
    torch.cuda.synchronize(dev)
    if WORLD > 1:
        import torch.distributed as dist
        dist.barrier()
    clk = Clocks(clocks_index)
    clk.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = grp.kv.launch_count()
    e0.record(main)
    nbytes, tokens = steps(ARGS.steps)
    e1.record(main)
    torch.cuda.synchronize(dev)
    clk.__exit__()
    ms = e0.elapsed_time(e1)
    launches = grp.kv.launch_count() - n0 + ARGS.steps * grp.n_launch_graph[(maxb, 0)]
    kern = grp.kernel_times()
    return dict(ms=ms, bytes=nbytes, tokens=tokens, launches=launches, clocks=clk.summary(),
                shares=None, kernels=kern, kernel_batch=maxb,
                kernel_ctx=int(np.mean(grp.models[0].ctx_lens(maxb))), names=grp.names,
                internal_frag_bytes=sum(m.internal_frag_bytes() for m in grp.models),
                B=[maxb] * ARGS.steps, models=names)


def run_ours():
    import torch
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    if ndev == 0:
        sys.stderr.write("bench.py: no CUDA device (the product path has no CPU fallback)\n")
        sys.exit(2)
    if WORLD > ndev:
        sys.stderr.write(f"bench.py: {WORLD} ranks need {WORLD} CUDA devices, found {ndev}\n")
        sys.exit(2)
    torch.cuda.set_device(LOCAL)
    dev = torch.device(f"cuda:{LOCAL}")
    if WORLD > 1:
        # the data path has no collective: the process group only carries the
        # barrier and the max-over-ranks timing reduction
        dist.init_process_group("nccl", device_id=dev)
    if ARGS.profile:  # a few eager steps at the workload's shape, for ncu
        grp, targets, _ = build_group(ARGS.workload, dev, seed=1234)
        for B in targets[:3]:
            if B != grp.B:
                grp.rebalance(B)
            grp.host_step()
            grp.device_step(B)
        torch.cuda.synchronize()
        print(json.dumps({"profile": f"{ARGS.workload}: {min(3, len(targets))} eager steps done"}))
        return
    peak, peak_kind = peaks()
    if ARGS.workload == "c5":
        r = run_c5(dev, LOCAL)
    else:
        r = measure(ARGS.workload, dev, LOCAL)
    head = summarise(ARGS.workload, r, peak, peak_kind, WORLD)
    extra = {}
    if ARGS.workload == "c5":
        per = [None] * WORLD
        mine = {"rank": RANK, "group": f"gpu{RANK % 8}", "models": r["models"],
                "gbs": round(r["bytes"] / (r["ms"] / 1e3) / 1e9, 1),
                "hbm_frac": round(r["bytes"] / (r["ms"] / 1e3) / 1e9 / peak, 4)}
        if WORLD > 1:
            dist.all_gather_object(per, mine)
        else:
            per = [mine]
        extra["per_gpu"] = per
    if RANK == 0 and WORLD == 1 and ARGS.workload == "c4" and not ARGS.no_c3:
        r3 = measure("c3", dev, LOCAL)
        s3 = summarise("c3", r3, peak, peak_kind, 1)
        s3["config"] = config_dict(WORKLOADS["c3"], 8, 8192)
        extra["c3"] = s3
    sweep = format_sweep(peak) if (RANK == 0 and WORLD == 1 and not ARGS.no_sweep) else None
    if RANK != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    names = r["names"]
    line = {"metric": "slab paged-decode attention HBM GB/s", "value": head.pop("value"), "unit": "GB/s",
            "n_gpus": WORLD, "steps": ARGS.steps, "warmup": ARGS.warmup,
            "ms_per_step": head.pop("ms_per_step"), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "/".join(names) + " KV, fp32 accumulate",
            "data": "synthetic (random fp16 Q/K/V, prompts and KV not from a model)",
            "config": config_dict(WL, WL["batch"], WL["ctx"]),
            **head, **extra}
    if sweep:
        line["formats"], line["prefill"] = sweep["decode"], sweep["prefill"]
    if not ARGS.no_cpu_baseline and WORLD == 1:  # rank 0 at N=1 only
        v, cores, sample = cpu_sample(WL)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GB/s", "cores": cores,
                                "kind": "port", "sample": sample, "cpu_model": cpu_model(),
                                "host_cpus": os.cpu_count()}
    print(json.dumps(line), flush=True)
    if WORLD > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    maybe_spawn()
    if ARGS.impl == "reference":
        run_reference()
    else:
        run_ours()

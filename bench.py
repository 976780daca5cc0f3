#!/usr/bin/env python3
"""bench.py -- KV-slab data path on B200.

Workload (BASELINE.json configs[1]): two co-located Llama-3-8B-shaped models
(32 layers, 32 q / 8 kv heads, d=128) sharing ONE slab pool per GPU, one with
FP16 KV (key 2 MiB) and one with FP8-E4M3 KV + 64 B/layer quant params (key
32*32832 B) -> mixed block sizes, lcm slab 1.0 GiB.  16 sequences per model
at ctx 2048 (growing by one token per step).  Synthetic fp16 Q/K/V.

A step = one decode step of both models through all 32 layers: host block
growth (SlabPool, simulator.cpp:561-578) + block-table delta upload, then per
layer and model K1 (append + quantise the new token) and K2 (paged decode),
replayed as one CUDA graph.  Each step streams ~6.4 GB of KV, far above L2
(126 MB); consecutive kernels read disjoint layer sub-blocks.

value  = algorithmic HBM bytes of K1+K2 per step / step time,
         whole job over all ranks (weak scaling, one pool per GPU, no NCCL on
         the data path).
e2e    = same, through the public API with Q/K/V copied in from pinned host
         memory and O copied back every step.
roofline = K2 FP16 launch (dominant kernel), timed live by CUDA events.
cpu_baseline = the fp64 OpenMP oracle (oracle/) on a bounded sample.
--impl reference: the reference's CPU path (reference SlabPool from
oracle/_ref + the oracle port for append/attention), rank 0 only.
"""
import argparse
import ctypes as C
import json
import math
import os
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
P.add_argument("--workload", default="c2", choices=["c2", "c3"],
               help="c2 (default, the BASELINE metric): FP16 + FP8 co-located, B16 ctx 2k; "
                    "c3: FP16 + INT4 co-located, B8 ctx 8k")
P.add_argument("--batch", type=int, default=None)
P.add_argument("--ctx", type=int, default=None)
P.add_argument("--no-cpu-baseline", action="store_true")
P.add_argument("--no-sweep", action="store_true", help="skip the per-format K2 / K4 sweep")
P.add_argument("--profile", action="store_true", help="one eager step, no timing (for ncu)")
ARGS = P.parse_args()
# BASELINE.json configs[1] / configs[2]: the two co-located models' KV dtypes
# (oracle/kernel codes: 0 FP16, 1 FP8-E4M3, 3 INT4), batch per model, context
WORKLOADS = {
    "c2": dict(dts=(0, 1), batch=16, ctx=2048,
               text="c2: two co-located Llama-3-8B-shape models (32L, 32q/8kv, d128) on one slab pool, "
                    "FP16 KV + FP8-E4M3 KV (64 B/layer params)"),
    "c3": dict(dts=(0, 3), batch=8, ctx=8192,
               text="c3: two co-located Llama-3-8B-shape models (32L, 32q/8kv, d128) on one slab pool, "
                    "FP16 KV + INT4 KV (QoQ-style fp16 scale/zero per token and head), ctx 8k"),
}
WL = WORKLOADS[ARGS.workload]
if ARGS.batch is None:
    ARGS.batch = WL["batch"]
if ARGS.ctx is None:
    ARGS.ctx = WL["ctx"]
DT_NAMES = {0: "fp16", 1: "fp8_e4m3", 2: "int8", 3: "int4"}
NAMES = [DT_NAMES[d] for d in WL["dts"]]

RANK = int(os.environ.get("RANK", "0"))
WORLD = int(os.environ.get("WORLD_SIZE", "1"))
LOCAL = int(os.environ.get("LOCAL_RANK", "0"))

HQ, HKV, D = 32, 8, 128


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


def config_dict(extra=None):
    d = {"workload": WL["text"],
         "layers": ARGS.layers, "batch_per_model": ARGS.batch, "ctx": ARGS.ctx,
         "tokens_per_block": 16, "kv_dtypes": NAMES,
         "parallelism": f"placement x{WORLD} (independent pool per GPU, no collective)",
         "l2": "inputs larger than L2: each step streams several GB of KV per GPU (126 MB L2)"}
    if extra:
        d.update(extra)
    return d


# ======================================================================
# CPU legs (oracle port / reference allocator) -- bounded samples
# ======================================================================
def oracle_qparams(dt):
    """Natural per-layer quant-param bytes of a block (precision.cpp:91-99 +
    DESIGN.md section 3): FP8 fp32 scale per (K|V, head), INT8 fp16 scale and
    INT4 fp16 (scale, zero) per (K|V, head, token)."""
    return {0: 0, 1: 2 * HKV * 4, 2: 2 * HKV * 16 * 2, 3: 2 * HKV * 16 * 4}[dt]


def cpu_sample(seconds_target=10.0, nthreads=None):
    """fp64 OpenMP oracle decode over one layer of both models (all 16 seqs),
    repeated until ~seconds_target.  Returns (GB/s, cores, sample text)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    nthreads = nthreads or oracle.NPROC
    rng = np.random.default_rng(0)
    B, ctx = ARGS.batch, ARGS.ctx
    res = []
    for dt in WL["dts"]:
        f = oracle.fmt(dt, HKV, HQ, D, 1, 16, oracle_qparams(dt))
        key = oracle.lib.orc_fmt_key(C.byref(f))
        nb = (ctx + 15) // 16
        img = np.zeros(B * nb * key, dtype=np.uint8)
        table = np.arange(B * nb, dtype=np.int32).reshape(B, nb)
        k = rng.standard_normal((B * ctx, HKV, D)).astype(np.float16).view(np.uint16)
        v = rng.standard_normal((B * ctx, HKV, D)).astype(np.float16).view(np.uint16)
        ts = np.repeat(np.arange(B, dtype=np.int32), ctx)
        tp = np.tile(np.arange(ctx, dtype=np.int32), B)
        sc = np.ones(2 * HKV, np.float32) if dt == 1 else None
        oracle.append(img, B * nb * key, B * nb, f, 0, k, v, ts, tp, table, sc)
        q = rng.standard_normal((B, HQ, D)).astype(np.float16).view(np.uint16)
        cl = np.full(B, ctx, np.int32)
        res.append((img, key, table, f, q, cl, sc, oracle.decode_bytes(f, cl)))
    t0 = time.perf_counter()
    nbytes, reps = 0, 0
    while True:
        for img, key, table, f, q, cl, sc, by in res:
            oracle.paged_decode(img, img.size, table.size, f, 0, q, table, cl, 1 / math.sqrt(D),
                                sc, nthreads=nthreads)
            nbytes += by
        reps += 1
        if time.perf_counter() - t0 >= seconds_target:
            break
    dt = time.perf_counter() - t0
    return (nbytes / dt / 1e9, nthreads,
            f"oracle fp64 decode, 1 layer of both models x {reps} reps "
            f"({B} seqs x ctx {ctx}, 32q/8kv), {nthreads} OpenMP threads, {dt:.1f} s")


def run_reference():
    """--impl reference: the reference CPU path, rank 0 only."""
    if RANK != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    ref = oracle.ref_lib()
    B, ctx = ARGS.batch, ARGS.ctx
    nthreads = oracle.NPROC
    rng = np.random.default_rng(1)
    models = []
    fl = [oracle.fmt(dt, HKV, HQ, D, 1, 16, oracle_qparams(dt)) for dt in WL["dts"]]
    kl = [int(oracle.lib.orc_fmt_key(C.byref(f))) for f in fl]
    slab = math.lcm(*kl)
    nb_max = (ctx + ARGS.steps + ARGS.warmup + 16) // 16 + 1
    nslabs = sum((B * nb_max * k) // slab for k in kl) + 4
    keys = (C.c_uint64 * 2)(*kl)
    if ref is not None:
        rp = ref.ref_pool_create(nslabs * slab, slab, keys, 2, 1)
        kind = "reference"

        def alloc(key):
            out = (C.c_uint64 * 4)()
            assert ref.ref_try_alloc(rp, key, out) == 0
            return int(out[2])
    else:
        op = oracle.OraclePool(nslabs * slab, slab, kl)
        kind = "port"

        def alloc(key):
            st, h = op.alloc(key)
            assert st == 0
            return h[2]
    img = np.zeros(nslabs * slab, dtype=np.uint8)
    for dt, f, key in zip(WL["dts"], fl, kl):
        models.append(dict(f=f, key=key, table=np.zeros((B, nb_max), np.int32),
                           nblk=[0] * B, cached=[0] * B,
                           sc=np.ones(2 * HKV, np.float32) if dt == 1 else None))

    def grow(m, s, tokens):  # simulator.cpp:561-578
        while m["nblk"][s] < (tokens + 15) // 16:
            m["table"][s, m["nblk"][s]] = alloc(m["key"])
            m["nblk"][s] += 1

    for s in range(B):  # prefill claim, simulator.cpp:500-526
        for m in models:
            grow(m, s, ctx)
            m["cached"][s] = ctx
    kpre = rng.standard_normal((B * ctx, HKV, D)).astype(np.float16).view(np.uint16)
    ts = np.repeat(np.arange(B, dtype=np.int32), ctx)
    tp = np.tile(np.arange(ctx, dtype=np.int32), B)
    for m in models:
        bps = slab // m["key"]
        oracle.append(img, slab, bps, m["f"], 0, kpre, kpre, ts, tp, m["table"], m["sc"])
    q = rng.standard_normal((B, HQ, D)).astype(np.float16).view(np.uint16)
    knew = rng.standard_normal((B, HKV, D)).astype(np.float16).view(np.uint16)

    def step():
        nbytes = 0
        for m in models:
            for s in range(B):
                grow(m, s, m["cached"][s] + 1)
            pos = np.array(m["cached"], np.int32)
            bps = slab // m["key"]
            oracle.append(img, slab, bps, m["f"], 0, knew, knew, np.arange(B, dtype=np.int32),
                          pos, m["table"], m["sc"])
            cl = pos + 1
            oracle.paged_decode(img, slab, bps, m["f"], 0, q, m["table"], cl, 1 / math.sqrt(D),
                                m["sc"], nthreads=nthreads)
            nbytes += oracle.decode_bytes(m["f"], cl)
            for s in range(B):
                m["cached"][s] += 1
        return nbytes

    for _ in range(ARGS.warmup):
        step()
    t0 = time.perf_counter()
    total = 0
    for _ in range(ARGS.steps):
        total += step()
    dt = time.perf_counter() - t0
    gbs = total / dt / 1e9
    sample = (f"1 of {ARGS.layers} layers per step, both models, {B} seqs each, ctx {ctx}+; "
              f"allocator = {'reference SlabPool (oracle/_ref)' if kind == 'reference' else 'oracle port'}, "
              f"append/attention = oracle port (fp64, {nthreads} threads)")
    line = {"metric": "slab paged-decode attention HBM GB/s", "value": round(gbs, 3),
            "unit": "GB/s", "impl": "reference", "n_gpus": WORLD, "steps": ARGS.steps,
            "warmup": ARGS.warmup, "ms_per_step": round(dt / ARGS.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "/".join(NAMES),
            "data": "synthetic", "config": config_dict(),
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": nthreads,
                             "kind": "port", "sample": sample, "cpu_model": cpu_model(),
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


def run_ours():
    import torch
    import torch.distributed as dist
    import paper_2509_06261_b200 as ks
    from paper_2509_06261_b200 import kv
    from paper_2509_06261_b200.engine import SlabModel
    from paper_2509_06261_b200.kv import KvDtype, KvFormat

    ndev = torch.cuda.device_count()
    local = LOCAL % ndev  # ranks > devices only in code-path smoke tests
    torch.cuda.set_device(local)
    if WORLD > 1:
        # the data path has no collective: the process group only carries the
        # barrier and the max-over-ranks timing reduction
        if ndev >= WORLD:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    dev = torch.device(f"cuda:{local}")
    L, B, ctx0 = ARGS.layers, ARGS.batch, ARGS.ctx
    fmts = [KvFormat(KvDtype(dt), HKV, HQ, D, L) for dt in WL["dts"]]
    keys = [f.key for f in fmts]
    slab = math.lcm(*keys)
    total_steps = ARGS.warmup + ARGS.steps + 2
    nb_max = (ctx0 + total_steps + 15) // 16 + 1
    need = sum(B * nb_max * k for k in keys)
    nslabs = need // slab + 2 * len(keys) + 2
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, keys), device=local)
    rng = np.random.default_rng(1234 + RANK)
    # churn so both models' blocks are scattered and interleaved
    junk = [h for h in (pool.try_alloc_block(keys[i % 2]) for i in range(B * 16)) if h]
    models = [SlabModel(pool, f, B, nb_max) for f in fmts]
    for s in range(B):
        for m in models:
            assert m.admit(s, ctx0)
            if s % 3 == 0 and junk:
                pool.free_block(junk.pop(int(rng.integers(len(junk)))))
    for m in models:
        m.sync()
    kv_scales = torch.ones(2 * HKV, dtype=torch.float32, device=dev) * 0.5
    # prefill KV for every layer with K1 (synthetic fp16 K/V)
    T = B * ctx0
    kpre = torch.randn(T, HKV, D, dtype=torch.float16, device=dev)
    vpre = torch.randn(T, HKV, D, dtype=torch.float16, device=dev)
    ts = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(ctx0)
    tp = torch.arange(ctx0, dtype=torch.int32, device=dev).repeat(B)
    for m in models:
        for layer in range(L):
            kv.kv_append(pool, m.fmt, layer, torch.roll(kpre, layer, 0), vpre, ts, tp, m.table,
                         kv_scales)
    torch.cuda.synchronize()
    # per-step device inputs (resident): Q per layer/model, new K/V.  Two
    # buffer sets (flat, so the e2e leg moves each step with one H2D and one
    # D2H copy) let the e2e leg overlap copies of step k+1 with compute of k.
    per_in = L * B * HQ * D + 2 * B * HKV * D
    per_out = L * B * HQ * D

    def make_set():
        inbuf = torch.randn(2 * per_in, dtype=torch.float16, device=dev)
        outbuf = torch.empty(2 * per_out, dtype=torch.float16, device=dev)
        qv, kv_, vv, ov = [], [], [], []
        for mi in range(2):
            base = inbuf[mi * per_in:(mi + 1) * per_in]
            qv.append([base[l * B * HQ * D:(l + 1) * B * HQ * D].view(B, HQ, D) for l in range(L)])
            off = L * B * HQ * D
            kv_.append(base[off:off + B * HKV * D].view(B, HKV, D))
            vv.append(base[off + B * HKV * D:off + 2 * B * HKV * D].view(B, HKV, D))
            ob = outbuf[mi * per_out:(mi + 1) * per_out]
            ov.append([ob[l * B * HQ * D:(l + 1) * B * HQ * D].view(B, HQ, D) for l in range(L)])
        return dict(inbuf=inbuf, outbuf=outbuf, q=qv, knew=kv_, vnew=vv, out=ov)

    sets = [make_set(), make_set()]
    q, knew, vnew, out = sets[0]["q"], sets[0]["knew"], sets[0]["vnew"], sets[0]["out"]
    seqs = torch.arange(B, dtype=torch.int32, device=dev)
    ctxd = torch.full((B,), ctx0 + 1, dtype=torch.int32, device=dev)  # includes the new token
    ws = [kv.DecodeWorkspace(pool, f, B) for f in fmts]

    side = torch.cuda.Stream()

    def device_step(bs=None):
        # the two co-located models run on their own streams (FineServe shares
        # the GPU spatially between co-located engines); per layer one fused
        # K1+K2 launch per model
        bs = sets[0] if bs is None else bs
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        for layer in range(L):
            for mi, m in enumerate(models):
                kv.paged_decode(pool, m.fmt, layer, bs["q"][mi][layer], m.table, ctxd,
                                out=bs["out"][mi][layer], kv_scales=kv_scales, workspace=ws[mi],
                                k_new=bs["knew"][mi], v_new=bs["vnew"][mi],
                                stream=main if mi == 0 else side)
        main.wait_stream(side)
        ctxd.add_(1)

    def host_step():
        # growth rule for the token written this step (simulator.cpp:561-578)
        for m in models:
            for s in range(B):
                if not m.ensure_capacity(s, m.cached[s] + 1):
                    raise RuntimeError("pool exhausted")
                m.cached[s] += 1
            m.sync()

    def step_bytes():
        total = 0
        for m in models:
            cl = [c for c in m.cached]  # after host_step: ctx of this step
            total += L * (m.fmt.decode_bytes(cl) + m.fmt.append_bytes(B))
        return total

    # MPS-style spatial sharing: the two co-located models get disjoint SM
    # budgets for their persistent K2 grids; the split is autotuned once.
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count

    def time_split(split):
        kv.set_decode_sm_share(pool, models[0].key, split[0])
        kv.set_decode_sm_share(pool, models[1].key, split[1])
        gg = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()

        def few():
            main = torch.cuda.current_stream()
            side.wait_stream(main)
            for layer in range(min(L, 8)):
                for mi, m in enumerate(models):
                    kv.paged_decode(pool, m.fmt, layer, q[mi][layer], m.table, ctxd,
                                    out=out[mi][layer], kv_scales=kv_scales, workspace=ws[mi],
                                    stream=main if mi == 0 else side)
            main.wait_stream(side)
        with torch.cuda.stream(cap):
            few()
            torch.cuda.synchronize()
            with torch.cuda.graph(gg, stream=cap):
                few()
        gg.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            gg.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    # candidates: the FP16 model's fraction of the budget, and a budget of all
    # SMs or slightly fewer (free SMs let each model's next launch start while
    # the current one drains; see decode.cu launch_fmt)
    cands = sorted({(s16, tot - s16) for tot in (n_sm, round(n_sm * 0.92), round(n_sm * 0.84))
                    for s16 in [max(1, min(tot - 1, round(tot * f))) for f in (0.42, 0.47, 0.52, 0.57, 0.62)]})
    if ARGS.profile:  # no autotune launches under the profiler
        times = {(n_sm // 2, n_sm - n_sm // 2): 0.0}
    else:
        times = {c: time_split(c) for c in cands}
    share16, share8 = min(times, key=times.get)
    kv.set_decode_sm_share(pool, models[0].key, 0 if ARGS.profile else share16)
    kv.set_decode_sm_share(pool, models[1].key, 0 if ARGS.profile else share8)

    if ARGS.profile:
        host_step()
        device_step()
        torch.cuda.synchronize()
        print(json.dumps({"profile": "one eager step done"}))
        return

    # capture one step as a CUDA graph (host work stays outside)
    host_step()
    device_step()  # warm (func attributes, workspaces)
    torch.cuda.synchronize()
    n0 = kv.launch_count()
    g = torch.cuda.CUDAGraph()
    s_cap = torch.cuda.Stream()
    s_cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_cap):
        with torch.cuda.graph(g, stream=s_cap):
            device_step()
    torch.cuda.current_stream().wait_stream(s_cap)
    per_graph = kv.launch_count() - n0
    g_b = torch.cuda.CUDAGraph()  # same step over buffer set 1 (e2e leg)
    with torch.cuda.stream(s_cap):
        with torch.cuda.graph(g_b, stream=s_cap):
            device_step(sets[1])
    torch.cuda.current_stream().wait_stream(s_cap)
    graphs = [g, g_b]
    # the capture advanced nothing on device (graph not yet replayed); the eager
    # warm step advanced pos/ctx by one: keep host mirror consistent
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    for _ in range(ARGS.warmup):
        host_step()
        g.replay()
    torch.cuda.synchronize()
    if WORLD > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nbytes = 0
    n_tab0 = kv.launch_count()
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(ARGS.steps):
            host_step()
            nbytes += step_bytes()
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    table_launches = kv.launch_count() - n_tab0
    gpu_launches = per_graph * ARGS.steps + table_launches

    # e2e through the public API with host buffers (pinned): every step's
    # Q/new K/V come from host memory and every output goes back; copies run
    # on a copy stream, double-buffered against compute (step k+1's inputs
    # and step k-1's outputs move while step k computes).  Timed on device.
    hin = [torch.empty(2 * per_in, dtype=torch.float16).pin_memory() for _ in range(2)]
    hout = [torch.empty(2 * per_out, dtype=torch.float16).pin_memory() for _ in range(2)]
    for h in hin:
        h.copy_(sets[0]["inbuf"].cpu())
    h2d, d2h = 2 * per_in * 2, 2 * per_out * 2
    cstream = torch.cuda.Stream()
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    ev_out = [torch.cuda.Event(), torch.cuda.Event()]
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_bytes = 0
    e2e_steps = max(4, ARGS.steps)
    torch.cuda.synchronize()
    e2.record(stream)
    cstream.wait_stream(stream)
    with torch.cuda.stream(cstream):  # inputs of step 0
        sets[0]["inbuf"].copy_(hin[0], non_blocking=True)
        ev_in[0].record(cstream)
    for k in range(e2e_steps):
        X = k & 1
        host_step()
        e2e_bytes += step_bytes()
        if k + 1 < e2e_steps:  # prefetch step k+1 into the other set once step k-1 is done
            Y = X ^ 1
            with torch.cuda.stream(cstream):
                if k >= 1:
                    cstream.wait_event(ev_out[Y])
                    sets[Y]["outbuf"].view(-1)  # outputs of step k-1 leave first
                    hout[Y].copy_(sets[Y]["outbuf"], non_blocking=True)
                sets[Y]["inbuf"].copy_(hin[Y], non_blocking=True)
                ev_in[Y].record(cstream)
        stream.wait_event(ev_in[X])
        graphs[X].replay()
        ev_out[X].record(stream)
    with torch.cuda.stream(cstream):  # last outputs
        X = (e2e_steps - 1) & 1
        cstream.wait_event(ev_out[X])
        hout[X].copy_(sets[X]["outbuf"], non_blocking=True)
    stream.wait_stream(cstream)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3)

    # roofline: K2 per model over the 32 layers as one graph (cold layers)
    for m in models:  # blocks for the device-side ctx (one token ahead of the host)
        for s_ in range(B):
            m.ensure_capacity(s_, m.cached[s_] + 1)
        m.sync()
    rl = {}
    for m in models:  # isolated kernels get the whole GPU
        kv.set_decode_sm_share(pool, m.key, 0)
    for mi, m in enumerate(models):
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_cap):
            with torch.cuda.graph(g2, stream=s_cap):
                for layer in range(L):
                    kv.paged_decode(pool, m.fmt, layer, q[mi][layer], m.table, ctxd,
                                    out=out[mi][layer], kv_scales=kv_scales, workspace=ws[mi])
        torch.cuda.current_stream().wait_stream(s_cap)
        g2.replay()
        torch.cuda.synchronize()
        reps = 5
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            g2.replay()
        b.record(stream)
        torch.cuda.synchronize()
        per_launch_ms = a.elapsed_time(b) / (reps * L)
        cl = [int(x) for x in ctxd.cpu().tolist()]
        by = m.fmt.decode_bytes(cl)
        rl[NAMES[mi]] = (by, per_launch_ms)

    # every KV precision's K2 alone (outside the timed region, rank 0 / N=1
    # only): the bench shape and a large batch, 8-layer graphs
    sweep = format_sweep(peaks()[0]) if (RANK == 0 and WORLD == 1 and not ARGS.no_sweep) else None
    del pool

    # ---- reduce over ranks (max time) ----
    from paper_2509_06261_b200.placement import reduce_max
    ms, e2e_ms = reduce_max(ms), reduce_max(e2e_ms)
    if RANK != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    value = WORLD * nbytes / (ms / 1e3) / 1e9
    e2e_val = WORLD * e2e_bytes / (e2e_ms / 1e3) / 1e9
    tok_s = WORLD * 2 * B * ARGS.steps / (ms / 1e3)
    by, pl = rl["fp16"]
    achieved = by / (pl / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f)
        if ARGS.workload == "c2":  # the committed capture is of the c2 FP16 launch
            traffic = prof.get("decode_fp16", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    kernels = {k: {"bytes": v[0], "us": round(v[1] * 1e3, 2),
                   "gbs": round(v[0] / (v[1] / 1e3) / 1e9, 1),
                   "frac": round(v[0] / (v[1] / 1e3) / 1e9 / peak, 4)} for k, v in rl.items()}
    line = {
        "metric": "slab paged-decode attention HBM GB/s",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": WORLD, "steps": ARGS.steps,
        "warmup": ARGS.warmup, "ms_per_step": round(ms / ARGS.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "/".join(NAMES) + " KV, fp32 accumulate", "data": "synthetic",
        "config": config_dict(),
        "decode_tok_s": round(tok_s, 1), "decode_tok_s_per_gpu": round(tok_s / WORLD, 1),
        "sm_share": {f"{NAMES[0]}_model": share16, f"{NAMES[1]}_model": share8,
                     "autotune_ms": {f"{k[0]}+{k[1]}": round(v, 3) for k, v in times.items()}},
        "frac_of_peak": round(value / WORLD / peak, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": f"paged_decode_kernel<FP16> (one layer, {B} seqs x ctx~{ARGS.ctx + ARGS.warmup + ARGS.steps}, 8 kv heads)",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "frac_of_8TBps": round(achieved / 8000.0, 4)},
        "kernels": kernels,
        "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(gpu_launches),
        **({"formats": sweep["decode"], "prefill": sweep["prefill"]} if sweep else {}),
        "clocks": clk.summary(),
    }
    if not ARGS.no_cpu_baseline and WORLD == 1:  # rank 0 at N=1 only
        v, cores, sample = cpu_sample()
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GB/s", "cores": cores,
                                "kind": "port", "sample": sample, "cpu_model": cpu_model(),
                                "host_cpus": os.cpu_count()}
    print(json.dumps(line), flush=True)
    if WORLD > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    if ARGS.impl == "reference":
        run_reference()
    else:
        run_ours()

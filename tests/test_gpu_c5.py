"""BASELINE.json configs[4] as a GPU parity case: 8xB200 global placement of
16 mixed-precision models with a Poisson request trace and per-GPU slab pools.

The placement and the trace are the REFERENCE's own (tests/golden/c5.json,
from oracle/ref_c5.cpp: place_models placement.cpp:135-205 and
generate_workload workload.cpp:130-190).  Each of the 8 groups gets an
independent pool holding only its models' keys (no exchange between groups,
SURVEY.md 8e); the groups run one after another on this single GPU.  Per
group the trace drives the reference engine lifecycle through the C ABI:
admission claims ceil(prompt/tpb) blocks with rollback (simulator.cpp:500-526),
K1 appends the prompt and K4 attends it, decode steps grow the tables
(:561-578) and run fused K1+K2, completion releases (:621).  Sampled prefill
and decode outputs are checked against the fp64 oracle on the live pool image
(blocks reused after frees, keys interleaved); the pool must end empty and
consistent.  Layers are reduced to 2 (the keys are checked at 32 layers).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "c5.json")))
DT = {"fp16": KvDtype.FP16, "fp8": KvDtype.FP8_E4M3, "int8": KvDtype.INT8, "int4": KvDtype.INT4}
TOL = {KvDtype.FP16: 1e-3, KvDtype.FP8_E4M3: 1e-3, KvDtype.INT8: 1e-2, KvDtype.INT4: 1e-2}
LAYERS, MAX_SEQS, DT_STEP = 2, 48, 0.02


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(o, r):
    o = o.reshape(-1, 128).astype(np.float64)
    r = r.reshape(-1, 128)
    return (np.abs(o - r).max(1) / np.maximum(np.abs(r).max(1), 1e-30)).max()


def fmt_of(name, layers):
    return KvFormat(DT[name.split("_")[1]], 8, 32, 128, layers)


def test_c5_reference_geometry_and_placement():
    """Keys at 32 layers equal the reference's kv_block_size; every model is
    placed exactly once over the 8 groups."""
    for m in GOLD["models"]:
        assert fmt_of(m["name"], 32).key == m["key"], m
    assert sorted(GOLD["assign"]) == sorted(m["name"] for m in GOLD["models"])
    assert set(GOLD["assign"].values()) <= {f"gpu{g}" for g in range(8)}


class Engine:
    def __init__(self, pool, name, seed):
        self.name, self.fmt = name, fmt_of(name, LAYERS)
        self.sm = SlabModel(pool, self.fmt, MAX_SEQS, 512 // 16 + 2)
        self.rng = np.random.default_rng(seed)
        self.scales = (np.linspace(0.5, 1.5, 16).astype(np.float32)
                       if self.fmt.kv_dtype == KvDtype.FP8_E4M3 else None)
        self.waiting, self.running = [], {}  # slot -> [request, generated]
        self.free_slots = list(range(MAX_SEQS))
        self.checked_prefill = self.checked_decode = 0

    def sc(self):
        return None if self.scales is None else cu(self.scales)


def oracle_check(pool, e, layer, q, table, ctx, out, cu_q=None):
    img = kv.kv_tensor(pool).cpu().numpy()
    f = oracle.fmt(int(e.fmt.kv_dtype), 8, 32, 128, LAYERS, 16, e.fmt.qparams)
    args = (img, pool.slab_size(), pool.blocks_per_slab(e.fmt.key), f, layer, q.view(np.uint16),
            table)
    if cu_q is None:
        ref, _ = oracle.paged_decode(*args, ctx, 1 / math.sqrt(128), e.scales, nthreads=oracle.NPROC)
    else:
        ref, _ = oracle.paged_prefill(*args, cu_q, ctx, 1 / math.sqrt(128), e.scales,
                                      nthreads=oracle.NPROC)
    err = rel_err(out, ref)
    assert err <= TOL[e.fmt.kv_dtype], (e.name, "prefill" if cu_q is not None else "decode", err)


def run_group(group):
    names = sorted(m for m, g in GOLD["assign"].items() if g == group)
    reqs = [r for r in GOLD["requests"] if r[1] in names]
    fmts = {n: fmt_of(n, LAYERS) for n in names}
    keys = sorted({f.key for f in fmts.values()})
    slab = math.lcm(*keys)
    # a pool for ~40 % of the trace's worst-case demand: admission must defer
    demand = sum(fmts[r[1]].key * -(-(r[3] + r[4]) // 16) for r in reqs)
    nslabs = max(2 * len(keys) + 2, int(0.4 * demand) // slab + len(keys))
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, keys), device=0)
    kv.kv_tensor(pool).zero_()
    eng = {n: Engine(pool, n, 7 + i) for i, n in enumerate(names)}
    pending = list(reqs)  # arrival order
    step, done, deferred = 0, 0, 0
    while done < len(reqs):
        now = step * DT_STEP
        while pending and pending[0][2] <= now:
            r = pending.pop(0)
            eng[r[1]].waiting.append(r)
        for e in eng.values():
            # admission, FIFO (simulator.cpp:500-526): claim, append, attend
            admitted = []
            while e.waiting and e.free_slots:
                r = e.waiting[0]
                slot = e.free_slots[-1]
                if not e.sm.admit(slot, r[3]):
                    deferred += 1
                    break
                e.free_slots.pop()
                e.waiting.pop(0)
                e.running[slot] = [r, 0]
                admitted.append(slot)
            if admitted:
                e.sm.sync()
                lens = [e.running[s][0][3] for s in admitted]
                T = sum(lens)
                H = 8
                ts = np.repeat(np.asarray(admitted, np.int32), lens)
                tp = np.concatenate([np.arange(n, dtype=np.int32) for n in lens])
                for layer in range(LAYERS):
                    k = e.rng.standard_normal((T, H, 128)).astype(np.float16)
                    v = e.rng.standard_normal((T, H, 128)).astype(np.float16)
                    kv.kv_append(pool, e.fmt, layer, cu(k), cu(v), cu(ts), cu(tp), e.sm.table, e.sc())
                # K4 over the admitted prompts (rows of the table gathered)
                idx = torch.tensor(admitted, dtype=torch.long, device="cuda")
                table = e.sm.table.index_select(0, idx).contiguous()
                ctx = torch.tensor(lens, dtype=torch.int32, device="cuda")
                cuq = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
                q = e.rng.standard_normal((T, 32, 128)).astype(np.float16)
                layer = step % LAYERS
                out = kv.paged_prefill(pool, e.fmt, layer, cu(q), table, cu(cuq), ctx, max(lens),
                                       kv_scales=e.sc())
                torch.cuda.synchronize()
                if e.checked_prefill < 2:
                    oracle_check(pool, e, layer, q, table.cpu().numpy(), np.asarray(lens, np.int32),
                                 out.cpu().numpy(), cu_q=cuq)
                    e.checked_prefill += 1
            # one decode step for every running sequence (simulator.cpp:561-578)
            slots = sorted(e.running)
            live = []
            for s in slots:
                if e.sm.ensure_capacity(s, e.sm.cached[s] + 1):
                    live.append(s)
                else:  # stalled growth: evict (simulator.cpp:583-596) and requeue
                    e.sm.release(s)
                    e.waiting.insert(0, e.running.pop(s)[0])
                    e.free_slots.append(s)
            if not live:
                continue
            for s in live:
                e.sm.cached[s] += 1
            e.sm.sync()
            B = len(live)
            idx = torch.tensor(live, dtype=torch.long, device="cuda")
            table = e.sm.table.index_select(0, idx).contiguous()
            ctx = torch.tensor([e.sm.cached[s] for s in live], dtype=torch.int32, device="cuda")
            check = e.checked_decode < 3 and step % 7 == 0
            for layer in range(LAYERS):
                q = e.rng.standard_normal((B, 32, 128)).astype(np.float16)
                kn = e.rng.standard_normal((B, 8, 128)).astype(np.float16)
                vn = e.rng.standard_normal((B, 8, 128)).astype(np.float16)
                out = kv.paged_decode(pool, e.fmt, layer, cu(q), table, ctx, kv_scales=e.sc(),
                                      k_new=cu(kn), v_new=cu(vn))
                if check and layer == LAYERS - 1:
                    torch.cuda.synchronize()
                    oracle_check(pool, e, layer, q, table.cpu().numpy(), ctx.cpu().numpy(),
                                 out.cpu().numpy())
                    e.checked_decode += 1
            # completion (simulator.cpp:621): the generated token count reached
            for s in live:
                e.running[s][1] += 1
                if e.running[s][1] >= e.running[s][0][4]:
                    e.sm.release(s)
                    del e.running[s]
                    e.free_slots.append(s)
                    done += 1
        step += 1
        assert step < 20000, "trace did not drain"
    torch.cuda.synchronize()
    ok, why = pool.check_integrity()
    assert ok, why
    assert pool.allocated_block_count() == 0
    st = pool.snapshot_stats()
    assert st.allocated_bytes == 0
    return dict(models=len(names), requests=len(reqs), steps=step, deferred=deferred,
                checks=sum(e.checked_prefill + e.checked_decode for e in eng.values()))


@pytest.mark.gpu
@pytest.mark.parametrize("group", [f"gpu{g}" for g in range(8)])
def test_c5_group_trace(group):
    if group not in set(GOLD["assign"].values()):
        pytest.skip("no model placed on this group")
    res = run_group(group)
    assert res["requests"] > 0 and res["checks"] > 0, res

#!/usr/bin/env python3
"""Calibrate the reference simulator's decode cost from measured K1+K2 time
(SURVEY.md section 8f, rank 1).

The reference models one decode step of an engine as
    dur = gamma_s + delta_s_per_seq * active + epsilon_s_per_cached_token * sum(cached)
(simulator.cpp:602-604, precision.hpp:156-162), with epsilon = 1e-9 s/token in
its scenarios -- not bandwidth-grounded.  This script
times the real attention part of a decode step (one fused append+decode launch
per layer, all layers, one CUDA graph) on this B200 over a grid of
(batch, context) per KV precision for a Llama-3-8B-shaped model (32 layers,
32q/8kv, d128), fits the three coefficients by least squares and writes
profiles/decode_cost_fit.json, whose "decode_cost" objects drop into a
reference scenario file (scenario.cpp:137-143 field names).

GEMMs are outside the path, so the fitted cost is the attention/KV share of a
step only.  Run on the GPU box:  python scripts/calibrate_decode_cost.py
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

L, HKV, HQ = 32, 8, 32
GRID = [(b, c) for b in (1, 4, 8, 16, 32) for c in (256, 1024, 4096)]


def time_step(fmt, B, ctx):
    slab = fmt.key * 16
    nb = (ctx + 16) // 16 + 1
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx + 1)
    m.sync()
    ctxd = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")
    q = [torch.randn(B, HQ, 128, dtype=torch.float16, device="cuda") for _ in range(L)]
    kn = torch.randn(B, HKV, 128, dtype=torch.float16, device="cuda")
    sc = torch.ones(2 * HKV, device="cuda")
    ws = kv.DecodeWorkspace(pool, fmt, B)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()

    def step():
        for layer in range(L):
            kv.paged_decode(pool, fmt, layer, q[layer], m.table, ctxd, kv_scales=sc,
                            workspace=ws, k_new=kn, v_new=kn)
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    del pool
    return a.elapsed_time(b) / 10 / 1e3  # seconds per step


def main():
    out = {"model": "Llama-3-8B shape (32 layers, 32q/8kv, d128), attention+append only",
           "gpu": torch.cuda.get_device_name(0), "grid": GRID, "fits": {}}
    for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4):
        fmt = KvFormat(dt, HKV, HQ, 128, L)
        X, y = [], []
        for B, c in GRID:
            t = time_step(fmt, B, c)
            X.append([1.0, B, B * (c + 1)])
            y.append(t)
        X, y = np.array(X), np.array(y)
        # relative-error weighted, non-negative least squares (the reference
        # requires non-negative coefficients, precision.cpp:315-318)
        from scipy.optimize import nnls
        coef, _ = nnls(X / y[:, None], np.ones_like(y))
        pred = X @ coef
        out["fits"][dt.name] = {
            "decode_cost": {"gamma_s": float(coef[0]), "delta_s_per_seq": float(coef[1]),
                            "epsilon_s_per_cached_token": float(coef[2])},
            "max_rel_residual": float(np.max(np.abs(pred - y) / y)),
            "measured_s": y.tolist(),
            "implied_GBps": float(fmt.token_size * L / coef[2] / 1e9) if coef[2] > 0 else None,
        }
        print(dt.name, out["fits"][dt.name]["decode_cost"], "resid",
              out["fits"][dt.name]["max_rel_residual"], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out["note"] = ("drop fits[<dtype>].decode_cost into a reference scenario model entry "
                   "(scenario.cpp:137-143); costs are per decode step of the whole model")
    with open(os.path.join(ROOT, "gpurun_out", "decode_cost_fit.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

"""Probe K2 variants on one layer of the bench workload (design exploration)."""
import os, sys, math, time, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

L = 8
B, ctx0 = int(os.environ.get("B", 16)), int(os.environ.get("CTX", 2048))
dts = [KvDtype[x] for x in os.environ.get("DTS", "FP16,FP8_E4M3,INT8,INT4").split(",")]
res = {}
for dt in dts:
    fmt = KvFormat(dt, 8, 32, 128, L)
    slab = fmt.key * 64
    nb = (ctx0 + 15) // 16
    nslabs = B * nb // 64 + 4
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    qs = [torch.randn(B, 32, 128, dtype=torch.float16, device="cuda") for _ in range(L)]
    sc = torch.ones(16, device="cuda")
    ws = kv.DecodeWorkspace(pool, fmt, B)
    by = fmt.decode_bytes([ctx0] * B)
    for dbg in [int(x) for x in os.environ.get("DBGS", "0,1,2,3").split(",")]:
        os.environ["KVSLAB_DECODE_DEBUG"] = str(dbg)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for l in range(L):
                kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for l in range(L):
                    kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws)
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            g.replay()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / (10 * L) * 1e3
        print(f"{dt.name:9s} debug={dbg}  {us:7.2f} us  {by/us/1e3:7.1f} GB/s", flush=True)
    del pool

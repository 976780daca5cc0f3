"""C1 (BASELINE configs[0]): one FP16 Llama-style MHA layer (32 heads, d128),
B=8, ctx 1024 -- K2 per-launch time in an 8-launch CUDA graph (design probe)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

for spec in os.environ.get("CASES", "FP16:32:32:8:1024,FP16:8:32:8:1024,INT4:32:32:8:1024").split(","):
    dtn, hk, hq, bs, cs = spec.split(":")
    dt, Hk, Hq, B, ctx0 = KvDtype[dtn], int(hk), int(hq), int(bs), int(cs)
    L = 8
    fmt = KvFormat(dt, Hk, Hq, 128, L)
    slab = fmt.key * 16
    nb = (ctx0 + 15) // 16 + 1
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    q = torch.randn(L, B, Hq, 128, dtype=torch.float16, device="cuda")
    out = torch.empty_like(q)
    ws = kv.DecodeWorkspace(pool, fmt, B)
    sc = torch.ones(2 * Hk, device="cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        for l in range(L):
            kv.paged_decode(pool, fmt, l, q[l], m.table, ctx, out=out[l], workspace=ws, kv_scales=sc)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for l in range(L):
                kv.paged_decode(pool, fmt, l, q[l], m.table, ctx, out=out[l], workspace=ws, kv_scales=sc)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / (10 * L) * 1e3
    by = fmt.decode_bytes([ctx0] * B)
    print(f"{dtn:6s} {Hk}kv/{Hq}q B={B} ctx={ctx0}: {us:7.2f} us  {by / us / 1e3:7.1f} GB/s", flush=True)
    del pool

"""K4 chunked-prefill attention throughput (design probe / DESIGN.md numbers).

Llama-3-8B shape (8 kv heads, 32 q heads, d128), one layer.  Cases: whole
prompts (chunk = context) and chunks at the end of a long context.  FLOPs
counted causally: 4 * d * Hq * sum over queries of (position + 1); the
tensor roofline is MEASURED_PEAKS bf16_tflops (dense fp16/bf16 tensor peak)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
peak = peaks.get("bf16_tflops", 2250.0)
H, Hq = 8, 32
for spec in os.environ.get("CASES", "FP16:1:4096:4096,FP16:4:8192:512,FP8_E4M3:1:4096:4096,"
                           "INT8:1:4096:4096,INT4:1:4096:4096,INT4:4:8192:512").split(","):
    dtn, bs, cs, ns = spec.split(":")
    dt, B, ctx0, nq = KvDtype[dtn], int(bs), int(cs), int(ns)
    fmt = KvFormat(dt, H, Hq, 128, 1)
    slab = fmt.key * 16
    nb = (ctx0 + 15) // 16 + 1
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    cu = torch.arange(0, (B + 1) * nq, nq, dtype=torch.int32, device="cuda")
    q = torch.randn(B * nq, Hq, 128, dtype=torch.float16, device="cuda")
    sc = torch.ones(2 * H, device="cuda")
    out = torch.empty_like(q)
    for _ in range(3):
        kv.paged_prefill(pool, fmt, 0, q, m.table, cu, ctx, nq, out=out, kv_scales=sc)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        kv.paged_prefill(pool, fmt, 0, q, m.table, cu, ctx, nq, out=out, kv_scales=sc)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    pos = np.arange(ctx0 - nq, ctx0, dtype=np.float64)
    flops = 4.0 * 128 * Hq * B * (pos + 1).sum()
    tf = flops / us / 1e6
    print(f"{dtn:9s} B={B} ctx={ctx0:5d} chunk={nq:5d}: {us:9.1f} us  {tf:7.1f} TFLOP/s "
          f"({tf / peak:.3f} of {peak:.0f})", flush=True)
    del pool

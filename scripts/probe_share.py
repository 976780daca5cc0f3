"""Co-located FP16 + FP8 models on two streams with SM shares (design probe)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import math, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
L, B, ctx0 = 8, 16, 2048
fmts = [KvFormat(KvDtype.FP16, 8, 32, 128, L), KvFormat(KvDtype.FP8_E4M3, 8, 32, 128, L)]
slab = math.lcm(*[f.key for f in fmts])
nb = (ctx0 + 15) // 16
need = sum(B * nb * f.key for f in fmts)
pool = ks.SlabPool(ks.SlabPoolConfig((need // slab + 6) * slab, slab, [f.key for f in fmts]), device=0)
ms = [SlabModel(pool, f, B, nb) for f in fmts]
for s in range(B):
    for m in ms:
        assert m.admit(s, ctx0)
for m in ms:
    m.sync()
ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
qs = [[torch.randn(B, 32, 128, dtype=torch.float16, device="cuda") for _ in range(L)] for _ in ms]
sc = torch.ones(16, device="cuda")
ws = [kv.DecodeWorkspace(pool, f, B) for f in fmts]
by = sum(f.decode_bytes([ctx0] * B) for f in fmts) * L
side = torch.cuda.Stream()
for share16 in [int(x) for x in os.environ.get("SHARES", "0,74").split(",")]:
    if share16:
        kv.set_decode_sm_share(pool, fmts[0].key, share16)
        kv.set_decode_sm_share(pool, fmts[1].key, 148 - share16)
    else:
        kv.set_decode_sm_share(pool, fmts[0].key, 0)
        kv.set_decode_sm_share(pool, fmts[1].key, 0)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    def step():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        for l in range(L):
            for mi, m in enumerate(ms):
                kv.paged_decode(pool, m.fmt, l, qs[mi][l], m.table, ctx, kv_scales=sc, workspace=ws[mi],
                                stream=main if mi == 0 else side)
        main.wait_stream(side)
    with torch.cuda.stream(cap):
        step(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=cap):
            step()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 10 / L * 1e3
    print(f"share16={share16:3d}  per-layer {us:6.2f} us  {by / L / us / 1e3:7.1f} GB/s", flush=True)

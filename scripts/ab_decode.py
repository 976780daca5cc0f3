"""A/B timing of K2 launch configurations in ONE process (design probe).

Each configuration (a dict of KVSLAB_* environment overrides, read by the C
ABI when a pool is created) gets its own pool and CUDA graph of L layers; rounds alternate the
configurations so box-to-box and drift effects cancel.  Usage:
  AB='{"a":{}, "b":{"KVSLAB_MERGE_THREADS":"128"}}' CASES=FP16:16:2048,INT4:32:1024 \
      python scripts/ab_decode.py
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

L = int(os.environ.get("LAYERS", 8))
configs = json.loads(os.environ.get("AB", '{"base": {}}'))
cases = [c.split(":") for c in os.environ.get("CASES", "FP16:16:2048").split(",")]
rounds = int(os.environ.get("ROUNDS", 5))
noapp = os.environ.get("NOAPP") == "1"  # probe builds' compute-only mode cannot append
for dtn, bs, cs in cases:
    dt, B, ctx0 = KvDtype[dtn], int(bs), int(cs)
    fmt = KvFormat(dt, 8, 32, 128, L)
    slab = fmt.key * 16
    nb = (ctx0 + 15) // 16 + 1
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    qs = [torch.randn(B, 32, 128, dtype=torch.float16, device="cuda") for _ in range(L)]
    kn = torch.randn(B, 8, 128, dtype=torch.float16, device="cuda")
    sc = torch.ones(16, device="cuda")
    by = fmt.decode_bytes([ctx0] * B)
    graphs, keep = {}, []
    base_env = dict(os.environ)
    for name, env in configs.items():
        # the tuning overrides are read when a pool is created: one pool per configuration
        os.environ.clear(); os.environ.update(base_env); os.environ.update(env)
        pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
        m = SlabModel(pool, fmt, B, nb)
        for s in range(B):
            assert m.admit(s, ctx0)
        m.sync()
        ws = kv.DecodeWorkspace(pool, fmt, B)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        def step():
            for l in range(L):
                kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws,
                                k_new=None if noapp else kn, v_new=None if noapp else kn)
        with torch.cuda.stream(st):
            step(); torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=st):
                step()
        graphs[name] = g
        keep.append((pool, m, ws))
    os.environ.clear(); os.environ.update(base_env)
    res = {n: [] for n in graphs}
    for r in range(rounds):
        for n, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.replay()
            b.record(); torch.cuda.synchronize()
            res[n].append(a.elapsed_time(b) / 10 / L * 1e3)
    line = " | ".join(f"{n}: {np.median(v):6.2f} us ({by / np.median(v) / 1e3:6.0f} GB/s)"
                      for n, v in res.items())
    print(f"{dtn:9s} B={B:3d} ctx={ctx0:5d}  {line}", flush=True)
    del graphs, keep

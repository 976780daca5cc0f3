"""One K1 launch per KV format (Llama-3-8B layer, 65536 tokens) -- for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
H, HQ, D, B, T = 8, 32, 128, 16, 4096
for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4):
    if os.environ.get("ONLY") and dt.name not in os.environ["ONLY"].split(","):
        continue
    fmt = KvFormat(dt, H, HQ, D, 1)
    slab = fmt.key * 64
    pool = ks.SlabPool(ks.SlabPoolConfig((B * T // 16 // 64 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, T // 16)
    for s in range(B):
        assert m.admit(s, T)
    m.sync()
    n = B * T
    k = torch.randn(n, H, D, dtype=torch.float16, device="cuda")
    v = torch.randn(n, H, D, dtype=torch.float16, device="cuda")
    ts = torch.arange(B, dtype=torch.int32, device="cuda").repeat_interleave(T)
    tp = torch.arange(T, dtype=torch.int32, device="cuda").repeat(B)
    sc = torch.ones(2 * H, device="cuda")
    kv.kv_append(pool, fmt, 0, k, v, ts, tp, m.table, sc)
    torch.cuda.synchronize()
    del pool, m

"""Does a concurrent host->device copy slow K1?  One K1 launch sequence (32
layers of one model's prompt tokens) alone, then with a 1 GB pinned H2D copy
running on another stream (design probe)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
H, HQ, D, B, T = 8, 32, 128, 16, 4096
host = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
devb = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
cp = torch.cuda.Stream()
for dt in (KvDtype.FP16, KvDtype.INT4):
    fmt = KvFormat(dt, H, HQ, D, 8)
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
    def run():
        for layer in range(8):
            kv.kv_append(pool, fmt, layer, k, v, ts, tp, m.table, sc)
    run(); torch.cuda.synchronize()
    for with_copy in (False, True, False, True):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if with_copy:
            with torch.cuda.stream(cp):
                devb.copy_(host, non_blocking=True)
        a.record(); run(); b.record(); torch.cuda.synchronize()
        print(f"{dt.name} 8 layers x {n} tokens: {a.elapsed_time(b):.3f} ms {'with 1 GB H2D' if with_copy else 'alone'}")
    del pool, m

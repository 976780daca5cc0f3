"""K1 (quantising append) and K3 (slab compaction) throughput (design probe /
DESIGN.md numbers).  Llama-3-8B layer geometry (8 kv heads, d128, tpb 16).

K1: one prefill chunk of T tokens for one layer; algorithmic bytes = fp16 K+V
in + quantised K+V out + params + one table lookup per token.
K3: a fragmented pool (every other block of each slab freed), one compaction
of the key; bytes = 2 x key x moves (read + write), the host plan outside the
timed region."""
import ctypes as C, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200 import _lib as L
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat

pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
peak = pk.get("hbm_gbs", 6536.0)
H, HQ, D = 8, 32, 128


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4):
    fmt = KvFormat(dt, H, HQ, D, 1)
    B, T = 16, 4096  # 16 sequences x 4096 tokens
    slab = fmt.key * 64
    nb = T // 16
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 64 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, T)
    m.sync()
    n = B * T
    k = torch.randn(n, H, D, dtype=torch.float16, device="cuda")
    v = torch.randn(n, H, D, dtype=torch.float16, device="cuda")
    ts = torch.arange(B, dtype=torch.int32, device="cuda").repeat_interleave(T)
    tp = torch.arange(T, dtype=torch.int32, device="cuda").repeat(B)
    sc = torch.ones(2 * H, device="cuda")
    ms = timed(lambda: kv.kv_append(pool, fmt, 0, k, v, ts, tp, m.table, sc))
    by = n * (2 * H * D * 2 + fmt.token_size + 4) + (n // 16) * fmt.qparams
    print(f"K1 {dt.name:9s} {n} tokens: {ms * 1e3:8.1f} us  {by / ms / 1e6:7.1f} GB/s "
          f"({by / ms / 1e6 / peak:.2f} of copy peak)", flush=True)
    del pool

for dt in (KvDtype.FP16, KvDtype.INT4):
    fmt = KvFormat(dt, H, HQ, D, 32)  # whole 32-layer blocks move
    slab = fmt.key * 16
    nslabs = 256
    pool = ks.SlabPool(ks.SlabPoolConfig(nslabs * slab, slab, [fmt.key]), device=0)
    hs = [pool.alloc_block(fmt.key) for _ in range(nslabs * 16)]
    rng = np.random.default_rng(0)
    for i in rng.permutation(len(hs))[: len(hs) // 2]:
        pool.free_block(hs[i])
    moves, freed = pool.plan_compaction(fmt.key, 1 << 20)
    buf = (L.ks_block_move * len(moves))(*[L.ks_block_move(s, d) for s, d in moves])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.lib.ks_compact_apply(pool.handle, fmt.key, buf, len(moves), None)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    by = 2 * fmt.key * len(moves)
    print(f"K3 {dt.name:9s} {len(moves)} moves of {fmt.key} B, {freed} slabs freed: {ms * 1e3:8.1f} us  "
          f"{by / ms / 1e6:7.1f} GB/s ({by / ms / 1e6 / peak:.2f} of copy peak)", flush=True)
    del pool

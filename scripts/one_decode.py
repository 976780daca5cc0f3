"""One K2 launch configuration for ncu captures (design probe): CASES=FMT:B:CTX, 4 layers."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
dtn, bs, cs = os.environ.get("CASE", "INT4:64:4096").split(":")
dt, B, ctx0 = KvDtype[dtn], int(bs), int(cs)
L = 4
fmt = KvFormat(dt, 8, 32, 128, L)
slab = fmt.key * 16
nb = (ctx0 + 15) // 16 + 1
pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
m = SlabModel(pool, fmt, B, nb)
for s in range(B):
    assert m.admit(s, ctx0)
m.sync()
ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
q = torch.randn(B, 32, 128, dtype=torch.float16, device="cuda")
kn = torch.randn(B, 8, 128, dtype=torch.float16, device="cuda")
sc = torch.ones(16, device="cuda")
for layer in range(L):
    kv.paged_decode(pool, fmt, layer, q, m.table, ctx, kv_scales=sc, k_new=kn, v_new=kn)
torch.cuda.synchronize()
print("done")

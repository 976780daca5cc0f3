"""Host cost of one kv.paged_decode / kv.kv_append call from Python (design
probe): wall time of 2000 back-to-back calls on a tiny batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
fmt = KvFormat(KvDtype.FP8_E4M3, 8, 32, 128, 4)
slab = fmt.key * 16
pool = ks.SlabPool(ks.SlabPoolConfig(64 * slab, slab, [fmt.key]), device=0)
m = SlabModel(pool, fmt, 8, 64)
for s in range(8):
    assert m.admit(s, 100)
m.sync()
ctx = torch.full((8,), 101, dtype=torch.int32, device="cuda")
q = torch.randn(8, 32, 128, dtype=torch.float16, device="cuda")
kn = torch.randn(8, 8, 128, dtype=torch.float16, device="cuda")
out = torch.empty_like(q)
sc = torch.ones(16, device="cuda")
ws = kv.DecodeWorkspace(pool, fmt, 8)
st = torch.cuda.current_stream()
for _ in range(50):
    kv.paged_decode(pool, fmt, 1, q, m.table, ctx, out=out, kv_scales=sc, workspace=ws, k_new=kn, v_new=kn, stream=st)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for i in range(n):
    kv.paged_decode(pool, fmt, i % 4, q, m.table, ctx, out=out, kv_scales=sc, workspace=ws, k_new=kn, v_new=kn, stream=st)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"paged_decode: host {1e6 * (t1 - t0) / n:.2f} us/call, incl. drain {1e6 * (t2 - t0) / n:.2f} us/call")
ts = torch.zeros(64, dtype=torch.int32, device="cuda")
tp = torch.arange(64, dtype=torch.int32, device="cuda")
kk = torch.randn(64, 8, 128, dtype=torch.float16, device="cuda")
t0 = time.perf_counter()
for i in range(n):
    kv.kv_append(pool, fmt, i % 4, kk, kk, ts, tp, m.table, sc, stream=st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"kv_append: host {1e6 * (t1 - t0) / n:.2f} us/call")
# Python-only share: the same loop with the C entry point stubbed out
import paper_2509_06261_b200._lib as L
real = L.lib.ks_paged_decode_append
class _Stub:
    def __getattr__(self, n):
        return getattr(L.lib_real, n)
L.lib_real = L.lib
try:
    kv.L.lib = type("S", (), {"ks_paged_decode_append": staticmethod(lambda *a: 0),
                              "__getattr__": lambda self, n: getattr(L.lib_real, n)})()
    t0 = time.perf_counter()
    for i in range(n):
        kv.paged_decode(pool, fmt, i % 4, q, m.table, ctx, out=out, kv_scales=sc, workspace=ws, k_new=kn, v_new=kn, stream=st)
    t1 = time.perf_counter()
    print(f"paged_decode Python only: {1e6 * (t1 - t0) / n:.2f} us/call")
finally:
    kv.L.lib = L.lib_real

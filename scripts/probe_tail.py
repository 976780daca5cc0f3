"""Per-CTA finish times of one K2 layer (design probe, probe build): which
CTAs are the tail stragglers, their range and unit-boundary count."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
L = 4
NT = 8192
for spec in os.environ.get("CASES", "INT4:16:2048").split(","):
    dtn, bs, cs = spec.split(":")
    dt, B, ctx0 = KvDtype[dtn], int(bs), int(cs)
    fmt = KvFormat(dt, 8, 32, 128, L)
    slab = fmt.key * 16
    nb = (ctx0 + 15) // 16 + 1
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    qs = [torch.randn(B, 32, 128, dtype=torch.float16, device="cuda") for _ in range(L)]
    kn = torch.randn(B, 8, 128, dtype=torch.float16, device="cuda")
    sc = torch.ones(16, device="cuda")
    ws = kv.DecodeWorkspace(pool, fmt, B)
    tr = torch.zeros(L, NT, dtype=torch.int64, device="cuda")
    app = os.environ.get("APPEND", "1") == "1"
    def step():
        for l in range(L):
            ks._lib.lib.ks_probe_set_decode_trace(pool.handle, tr[l].data_ptr())
            kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws,
                            k_new=kn if app else None, v_new=kn if app else None)
        ks._lib.lib.ks_probe_set_decode_trace(pool.handle, None)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        step(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            step()
    for it in range(3):
        tr.zero_(); tr[:, 2048] = 2**62
        g.replay(); torch.cuda.synchronize()
    t = tr.cpu().numpy()
    cta = t[:, :2048].reshape(L, -1, 8)
    live = cta[1, :, 0] > 0
    C = int(live.sum())
    total = B * ((ctx0 + 15) // 16)
    for l in (1, 2):
        c = cta[l]
        done = c[:C, 5].astype(np.float64)
        med = np.median(done)
        order = np.argsort(done)[::-1]
        rows = []
        for i in order[:12]:
            lo, hi = i * total // C, (i + 1) * total // C
            nbd = len([u for u in range(0, total + 1, (ctx0 + 15) // 16) if lo < u < hi])
            rows.append(f"{i}:+{(done[i]-med)/1e3:.2f}us[{lo},{hi}) b{nbd} st{(c[i,0]-c[:C,0].min())/1e3:.1f}")
        print(f"{dtn} L{l} slowest: " + "  ".join(rows))
        seg = t[l, 5200:5200 + 8 * C].reshape(C, 2, 4).astype(np.float64)
        for i in list(order[:4]) + list(order[-2:]):
            sg = seg[i]
            txt = []
            for k in range(2):
                if sg[k, 0] > 0:
                    a, b_, c_, d_ = (sg[k] - med) / 1e3
                    txt.append(f"seg{k}: qwait {a:+.2f}->{b_:+.2f} loop->{c_:+.2f} epi->{d_:+.2f}")
            print(f"   cta {i}: " + " | ".join(txt))
        fast = order[-5:]
        print(f"   fastest: " + "  ".join(f"{i}:{(done[i]-med)/1e3:.2f}" for i in fast))

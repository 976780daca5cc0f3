"""Per-stage timeline of K2 (design probe): for layer 1 of an L-layer graph,
per CTA the producer issue time and consumer-ready time of its first 32 stages
(us from the layer's first CTA start).  Prints percentiles over CTAs per stage
index, plus the layer's Q-available time (merge of the previous layer done).
Needs the stamps compiled in:
  make -C paper_2509_06261_b200/csrc clean && make -C paper_2509_06261_b200/csrc NVFLAGS_EXTRA=-DKVSLAB_STAGE_PROBES"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
L = int(os.environ.get("LAYERS", 4))
TR_STAGE = 12288
TR_READY = TR_STAGE + 148 * 4 * 32
NT = TR_READY + 148 * 4 * 32
for spec in os.environ.get("CASES", "FP8_E4M3:16:2048").split(","):
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
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    def step():
        for l in range(L):
            ks._lib.lib.ks_probe_set_decode_trace(pool.handle, tr[l].data_ptr())
            kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws,
                            k_new=kn, v_new=kn)
        ks._lib.lib.ks_probe_set_decode_trace(pool.handle, None)
    with torch.cuda.stream(st):
        step(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            step()
    for it in range(3):
        tr.zero_()
        tr[:, 2048] = 2**62
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
    t = tr.cpu().numpy()
    l = 1
    cta = t[l, :2048].reshape(-1, 8)
    live = cta[:, 0] > 0
    base = cta[live, 0].min()
    us = lambda x: (x.astype(np.float64) - base) / 1e3
    prev_merge_done = us(np.array([t[l - 1, 2049]]))[0]
    iss = t[l, TR_STAGE:TR_STAGE + 148 * 4 * 32].reshape(-1, 32)[:live.sum()]
    rdy = t[l, TR_READY:TR_READY + 148 * 4 * 32].reshape(-1, 32)[:live.sum()]
    nst = int(np.median(cta[live, 3]))
    print(f"{dtn} B={B} ctx={ctx0}: {live.sum()} CTAs, {nst} stages/CTA; prev merge done {prev_merge_done:.2f}; "
          f"CTA start p50 {np.median(us(cta[live,0])):.2f}; cons done p50/max {np.median(us(cta[live,5])):.2f}/{us(cta[live,5]).max():.2f}")
    pc = lambda x: "/".join("%6.2f" % np.percentile(x, q) for q in (10, 50, 90))
    # CTAs whose block range holds a unit start past its first block (two segments)
    C = int(live.sum())
    nblk = (ctx0 + 15) // 16
    T = B * nblk  # one head group of 8
    bnd = np.array([any(c * T // C < u * nblk < (c + 1) * T // C for u in range(1, B)) for c in range(C)])
    for name, sel in (("interior", ~bnd), ("boundary", bnd)):
        print(f" {name} CTAs ({sel.sum()}): start p50 {np.median(us(cta[:C][sel,0])):.2f} data p50 "
              f"{np.median(us(cta[:C][sel,4])):.2f} cons done p10/50/90 {pc(us(cta[:C][sel,5]))}")
        for k in range(min(nst, 32)):
            ok = sel & (iss[:, k] > 0) & (rdy[:, k] > 0)
            if not ok.any():
                continue
            print(f"  stage {k:2d}: issue {pc(us(iss[ok, k]))}  ready {pc(us(rdy[ok, k]))}  lat {pc((rdy[ok,k]-iss[ok,k])/1e3)}")
    del pool

"""Timeline of L consecutive K2 layers (decode + merge, PDL, one CUDA graph) from
globaltimer stamps -- design probe; needs a probe build of the library:
  make -C paper_2509_06261_b200/csrc BUILD=$PWD/build_ab/probe/obj OUT=$PWD/build_ab/probe/libkvslab.so \
       NVFLAGS_EXTRA=-DKVSLAB_PROBES CXXFLAGS_EXTRA=-DKVSLAB_PROBES
  KVSLAB_LIB_PATH=$PWD/build_ab/probe/libkvslab.so python scripts/probe_timeline.py  Per layer (us from the first decode CTA start):
decode CTA start (min/max), consumer first data (median), consumer done (max),
merge past its wait (min), merge done (max)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
L = int(os.environ.get("LAYERS", 6))
NT = 2050 + 3 * 1024
for spec in os.environ.get("CASES", "FP8_E4M3:16:2048,INT4:8:8192").split(","):
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
            app = os.environ.get("APPEND", "1") == "1"
            kv.paged_decode(pool, fmt, l, qs[l], m.table, ctx, kv_scales=sc, workspace=ws,
                            k_new=kn if app else None, v_new=kn if app else None)
        ks._lib.lib.ks_probe_set_decode_trace(pool.handle, None)
    with torch.cuda.stream(st):
        step(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            step()
    for it in range(3):
        tr.zero_()
        tr[:, 2048] = 2**62
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record()
        torch.cuda.synchronize()
    t = tr.cpu().numpy()
    cta = t[:, :2048].reshape(L, -1, 8)
    cta[:, :, 0] = np.where(cta[:, :, 0] > 0, cta[:, :, 0], cta[:, :, 4])  # compute-only probes: no producer stamps
    live = cta[:, :, 0] > 0
    base = cta[:, :, 0][live].min()
    us = lambda x: (x - base) / 1e3
    print(f"{dtn} B={B} ctx={ctx0} layers={L} graph={a.elapsed_time(b)*1e3:.1f}us "
          f"({a.elapsed_time(b)*1e3/L:.1f}/layer) ctas={live[0].sum()}")
    for l in range(L):
        c = cta[l][live[l]]
        mw = us(t[l, 2048]) if t[l, 2048] < 2**62 else float("nan")
        me = us(t[l, 2049]) if t[l, 2049] > 0 else float("nan")
        print(f"  L{l}: start {us(c[:,0].min()):7.2f}-{us(c[:,0].max()):7.2f}  data {us(np.median(c[:,4])):7.2f}"
              f"  prod done {us(c[:,2].max()):7.2f}  cons done {us(np.median(c[:,5])):7.2f}/{us(c[:,5].max()):7.2f}"
              f"  merge {mw:7.2f}-{me:7.2f}")
    c = cta[1][live[1]]
    st_, dn_ = us(c[:, 0]), us(c[:, 5])
    pc4 = lambda x: "/".join("%.2f" % np.percentile(x, q) for q in (0, 10, 50, 90, 100))
    print(f"  L1 CTA start pct(0/10/50/90/100) {pc4(st_)}  done {pc4(dn_)}  corr {np.corrcoef(st_, dn_)[0,1]:.2f}")
    late = dn_ > np.percentile(dn_, 90)
    print(f"  L1 consumer loop: {np.median(c[:,6] / np.maximum(c[:,7],1)):.0f} cycles/iteration (warp 0), "
          f"{np.median((c[:,5]-c[:,4]) / np.maximum(c[:,7],1)):.0f} ns/iteration, clock "
          f"{np.median(c[:,6] / np.maximum(c[:,5]-c[:,4],1)):.2f} GHz")
    print(f"  L1 late finishers: start {pc4(st_[late])}  blocks/cta {np.median(c[:,3]):.0f}  late ids {np.nonzero(live[1])[0][late][:12]}")
    for l in (1, L - 1):
        mm = t[l, 2050:2050 + 3 * B * 8].reshape(-1, 3)
        ok = mm[:, 0] > 0
        mm = us(mm[ok])
        fin = mm[:, 2] > 0
        pc = lambda x: "%.2f/%.2f/%.2f" % (np.min(x), np.median(x), np.max(x))
        print(f"  merge L{l}: {ok.sum()} ctas, start {pc(mm[:,0])} past-wait {pc(mm[:,1])} "
              f"end(cut units: {fin.sum()}) {pc(mm[fin,2]) if fin.any() else '-'}")
    del pool

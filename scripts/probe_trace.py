"""Per-CTA timeline of one K2 launch (globaltimer stamps) -- design probe.
Columns: kernel start, producer 2nd issue, producer done, consumer first data,
consumer done (us from the earliest CTA start)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
for spec in os.environ.get("CASES", "FP16:16:2048,INT4:8:8192").split(","):
    dtn, bs, cs = spec.split(":")
    dt, B, ctx0 = KvDtype[dtn], int(bs), int(cs)
    fmt = KvFormat(dt, 8, 32, 128, 2)
    slab = fmt.key * 16
    nb = (ctx0 + 15) // 16
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 16 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    q = torch.randn(B, 32, 128, dtype=torch.float16, device="cuda")
    tr = torch.zeros(148 * 2 * 8, dtype=torch.int64, device="cuda")
    for it in range(4):
        tr.zero_()
        os.environ["KVSLAB_DECODE_TRACE"] = str(tr.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kv.paged_decode(pool, fmt, it % 2, q, m.table, ctx)
        b.record()
        torch.cuda.synchronize()
    del os.environ["KVSLAB_DECODE_TRACE"]
    t = tr.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t[:, [0, 1, 2, 4, 5]] - base) / 1e3
    q_ = lambda c: "%.2f/%.2f/%.2f" % (rel[:, c].min(), np.median(rel[:, c]), rel[:, c].max())
    print(f"{dtn} B={B} ctx={ctx0} ctas={len(t)} blocks/cta={np.median(t[:, 3]):.0f} event={a.elapsed_time(b)*1e3:.1f}us")
    print("  start", q_(0), "| prod 2nd issue", q_(1), "| prod done", q_(2), "| cons first data", q_(3), "| cons done", q_(4))
    del pool

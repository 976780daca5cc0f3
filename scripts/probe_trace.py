"""Per-warp timeline of one K2 launch (globaltimer stamps) -- design probe."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.engine import SlabModel
from paper_2509_06261_b200.kv import KvDtype, KvFormat
B, ctx0 = 16, 2048
for dt in (KvDtype.FP16, KvDtype.FP8_E4M3):
    fmt = KvFormat(dt, 8, 32, 128, 2)
    slab = fmt.key * 64
    nb = (ctx0 + 15) // 16
    pool = ks.SlabPool(ks.SlabPoolConfig((B * nb // 64 + 4) * slab, slab, [fmt.key]), device=0)
    m = SlabModel(pool, fmt, B, nb)
    for s in range(B):
        assert m.admit(s, ctx0)
    m.sync()
    ctx = torch.full((B,), ctx0, dtype=torch.int32, device="cuda")
    q = torch.randn(B, 32, 128, dtype=torch.float16, device="cuda")
    tr = torch.zeros(148 * 2 * 16 * 6, dtype=torch.int64, device="cuda")
    for it in range(3):
        tr.zero_()
        os.environ["KVSLAB_DECODE_TRACE"] = str(tr.data_ptr())
        kv.paged_decode(pool, fmt, it % 2, q, m.table, ctx)
        torch.cuda.synchronize()
    del os.environ["KVSLAB_DECODE_TRACE"]
    t = tr.view(-1, 16, 6).cpu().numpy()
    valid = t[:, :, 0] > 0
    t0 = t[:, :, 0][valid].min()
    st = (t[:, :, 0][valid] - t0) / 1e3
    lp = (t[:, :, 1][valid] - t0) / 1e3
    en = (t[:, :, 2][valid] - t0) / 1e3
    npd = t[:, :, 3][valid]
    print(dt.name, "warps", valid.sum(), "start max %.2f" % st.max(),
          "loop end min/med/max %.2f %.2f %.2f" % (lp.min(), np.median(lp), lp.max()),
          "end max %.2f" % en.max(), "merging warps", (npd > 0).sum(),
          "merge dur med/max %.2f %.2f" % (np.median((en - lp)[npd > 0]), (en - lp)[npd > 0].max()))
    at = (t[:, :, 4][valid] - t0) / 1e3
    fe = (t[:, :, 5][valid] - t0) / 1e3
    mk = npd > 0
    print("   merging warps: atomic done med %.2f, loop end med %.2f, fence done med %.2f, end med %.2f" %
          (np.median(at[mk]), np.median(lp[mk]), np.median(fe[mk]), np.median(en[mk])))
    print("   non-merging last atomic med %.2f max %.2f" % (np.median(at[~mk & (at > 0)]), at.max()))
    del pool

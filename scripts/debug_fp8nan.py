import sys, os, math
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import numpy as np, torch
import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import test_gpu_scale as T
which = [int(x) for x in os.environ.get("WHICH", "0,1,2,3").split(",")]
fmts = [KvFormat(dt, 8, 32, num_layers=32) for dt in (KvDtype.FP16, KvDtype.FP8_E4M3, KvDtype.INT8, KvDtype.INT4)]
fmts = [fmts[i] for i in which]
slab, maxb, max_ctx = 64 << 20, 64, 2048 + 16
mb = (max_ctx + 15) // 16 + 1
need = sum(maxb * mb * f.key for f in fmts)
pool = ks.SlabPool(ks.SlabPoolConfig((need * 5 // 4 // slab + 10) * slab, slab, [f.key for f in fmts], False), device=0)
ms = [T.Model(pool, f, maxb, max_ctx, 50 + i) for i, f in enumerate(fmts)]
rng = np.random.default_rng(2024)
B = int(os.environ.get("B", 64))
for m in ms:
    m.admit(list(range(B)), rng.integers(512, 2049, size=B).tolist())
torch.cuda.synchronize()
for m in ms:
    res, ctx = m.step(B)
    for layer in T.LAYERS:
        q, out = res[layer]
        bad = ~np.isfinite(out)
        print(m.fmt.kv_dtype.name, layer, "nonfinite", int(bad.sum()), "rows", sorted(set(np.nonzero(bad)[0].tolist()))[:10], "dims", sorted(set(np.nonzero(bad)[2].tolist()))[:10], flush=True)
    try:
        print("err", m.check(B, res, ctx))
    except AssertionError as e:
        print("check failed", e)

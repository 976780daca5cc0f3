"""Accuracy report (design probe): worst per-row relative error of K2 decode and
K4 prefill against the fp64 oracle for every KV format, long contexts with 1%
8-sigma outliers (the test distribution)."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np, torch
from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import oracle
from test_gpu_kernels import FORMATS, append_gpu, dev, make_world, rel_err
from test_gpu_prefill import run_prefill
for dt in FORMATS:
    fmt = KvFormat(dt, 8, 32, num_layers=1)
    ctx = [16384, 4000, 700, 9000]
    w = make_world(fmt, ctx, seed=1, fp8_scale=[1.0] * 16 if dt == KvDtype.FP8_E4M3 else None)
    append_gpu(w, fmt, 0)
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    q = w["rng"].standard_normal((len(ctx), 32, 128)).astype(np.float16)
    out = kv.paged_decode(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(w["ctx"]),
                          kv_scales=None if w["scales"] is None else dev(w["scales"]))
    f = oracle.fmt(int(dt), 8, 32, 128, 1, 16, fmt.qparams)
    ref, _ = oracle.paged_decode(img, w["pool"].slab_size(), w["pool"].blocks_per_slab(fmt.key), f, 0,
                                 q.view(np.uint16), w["table"], w["ctx"], 1 / math.sqrt(128), w["scales"],
                                 nthreads=os.cpu_count())
    e_dec = rel_err(out.cpu().numpy(), ref)
    _, _, _, _, o, _, r, _ = run_prefill(dt, 2, 8, [(3000, 1000), (700, 161)], seed=2)
    e_pre = rel_err(o, r)
    print(f"{dt.name:9s} decode ctx<=16k: {e_dec:.2e}   prefill ctx<=3k: {e_pre:.2e}", flush=True)

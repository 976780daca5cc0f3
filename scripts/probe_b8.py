"""c4 low phase (B = 8 per model) dissected (design probe): the four models'
fused append+decode layers as 8-layer graphs, each model alone at its tuned
SM share, then all four together, then each alone on the whole GPU."""
import importlib.util, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = ["bench.py"]
spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
bm = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bm)
import torch
dev = torch.device("cuda:0")
grp, targets, _ = bm.build_group("c4", dev, seed=1234)
grp.rebalance(8)
sh = grp.tune_shares(8)
print("shares", sh["split"])
kv = grp.kv
B = grp.B
bs = grp.buffers(B)[0]
main = torch.cuda.current_stream(dev)


def graph_of(models, layers=8):
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(main)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            cur = torch.cuda.current_stream(dev)
            for st in grp.streams:
                st.wait_stream(cur)
            for layer in range(layers):
                for mi in models:
                    m = grp.models[mi]
                    kv.paged_decode(grp.pool, m.fmt, layer, bs["q"][mi][layer], m.table, grp.ctx[mi][:B],
                                    out=bs["out"][mi][layer], kv_scales=grp.scales, workspace=grp.ws[mi],
                                    stream=grp.streams[mi])
            for st in grp.streams:
                cur.wait_stream(st)
    main.wait_stream(cap)
    return g


def t(g):
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main); g.replay(); b.record(main); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e3 / 8


ctx = [int(x) for x in grp.ctx[0][:B].cpu().tolist()]
for mi, n in enumerate(grp.names):
    m = grp.models[mi]
    by = m.fmt.decode_bytes([int(x) for x in grp.ctx[mi][:B].cpu().tolist()])
    print(f"{n:10s} alone at share: {t(graph_of([mi])):6.2f} us/layer  ({by/1e6:.1f} MB)")
print(f"all four together: {t(graph_of(range(4))):6.2f} us/layer")
saved = dict(grp.shares)
for m in grp.models:
    kv.set_decode_sm_share(grp.pool, m.key, 0)
for mi, n in enumerate(grp.names):
    print(f"{n:10s} alone, whole GPU: {t(graph_of([mi])):6.2f} us/layer")
print(f"all four, no shares: {t(graph_of(range(4))):6.2f} us/layer")

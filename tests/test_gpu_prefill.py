"""GPU parity of K4 chunked-prefill attention against the
fp64 oracle (oracle/kvslab_oracle.c orc_paged_prefill), through the C ABI.

Sequences mix whole prompts (chunk = context), chunks at the end of an
existing context, single-token chunks and empty chunks; blocks are scattered
by allocator churn.  Tolerance as K2: max|o-r| / max|r| per (query token,
query head) <= 1e-3 (FP16/FP8) or 1e-2 (INT8/INT4); LSE within 1e-3.
"""
import math

import numpy as np
import pytest
import torch

from paper_2509_06261_b200 import kv
from paper_2509_06261_b200.kv import KvDtype, KvFormat
import oracle
from test_gpu_kernels import FORMATS, TOL, append_gpu, dev, make_world

pytestmark = pytest.mark.gpu

# (context incl. the chunk, chunk length)
CASES = [(1, 1), (37, 37), (300, 45), (16, 16), (17, 1), (129, 0), (700, 161), (64, 33)]


def run_prefill(dt, H, Hq, cases, seed, layers=1, layer=0):
    fmt = KvFormat(dt, H, Hq, num_layers=layers)
    ctx = [c for c, _ in cases]
    nq = [n for _, n in cases]
    w = make_world(fmt, ctx, seed=seed,
                   fp8_scale=np.linspace(0.5, 2.0, 2 * H).astype(np.float32)
                   if dt == KvDtype.FP8_E4M3 else None)
    append_gpu(w, fmt, layer)
    cu = np.concatenate([[0], np.cumsum(nq)]).astype(np.int32)
    q = w["rng"].standard_normal((int(cu[-1]), Hq, 128)).astype(np.float16)
    lse = torch.zeros((int(cu[-1]), Hq), dtype=torch.float32, device="cuda")
    out = kv.paged_prefill(w["pool"], fmt, layer, dev(q), dev(w["table"]), dev(cu),
                           dev(w["ctx"]), max(nq), lse=lse,
                           kv_scales=None if w["scales"] is None else dev(w["scales"]))
    torch.cuda.synchronize()
    img = kv.kv_tensor(w["pool"]).cpu().numpy()
    f = oracle.fmt(int(dt), H, Hq, 128, layers, 16, fmt.qparams)
    ref, ref_lse = oracle.paged_prefill(img, w["pool"].slab_size(), w["pool"].blocks_per_slab(fmt.key),
                                        f, layer, q.view(np.uint16), w["table"], cu, w["ctx"],
                                        1 / math.sqrt(128), w["scales"], nthreads=8)
    return w, fmt, q, cu, out.cpu().numpy().astype(np.float64), lse.cpu().numpy(), ref, ref_lse


def rel_err(o, r):
    o = o.reshape(-1, 128)
    r = r.reshape(-1, 128)
    return (np.abs(o - r).max(1) / np.maximum(np.abs(r).max(1), 1e-30)).max() if len(r) else 0.0


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
@pytest.mark.parametrize("H,Hq", [(2, 2), (2, 8), (2, 16), (2, 32)], ids=["mha", "gqa4", "gqa8", "gqa16"])
def test_prefill_matches_oracle(dt, H, Hq):
    _, _, _, _, o, lse, r, rl = run_prefill(dt, H, Hq, CASES, seed=11 * int(dt) + Hq)
    err = rel_err(o, r)
    assert err <= TOL[dt], f"{dt.name} H={H} Hq={Hq}: rel err {err:.3e}"
    assert np.abs(lse - rl).max() <= 1e-3


def test_prefill_layer_offset_int4():
    """A non-zero layer of a multi-layer key reads its own sub-blocks."""
    _, _, _, _, o, _, r, _ = run_prefill(KvDtype.INT4, 2, 8, [(200, 77), (33, 33)], seed=5,
                                         layers=3, layer=2)
    assert rel_err(o, r) <= 1e-2


@pytest.mark.parametrize("dt", [KvDtype.FP16, KvDtype.INT8], ids=["FP16", "INT8"])
def test_prefill_last_token_equals_decode(dt):
    """A one-token chunk at the end of the context is a decode step: K4 and K2
    see the same bytes and must agree to fp16-rounding level."""
    H, Hq = 2, 8
    cases = [(513, 1), (40, 1), (1, 1), (1000, 1)]
    w, fmt, q, cu, o, _, _, _ = run_prefill(dt, H, Hq, cases, seed=3)
    dec = kv.paged_decode(w["pool"], fmt, 0, dev(q.reshape(len(cases), Hq, 128)), dev(w["table"]),
                          dev(w["ctx"]))
    torch.cuda.synchronize()
    d = dec.cpu().numpy().astype(np.float64)
    assert rel_err(o, d) <= 2e-3


@pytest.mark.parametrize("nt", ["1", "2"])
def test_prefill_mma_sync_row_tilings(nt, monkeypatch):
    """The mma.sync kernel (KVSLAB_PREFILL_TC=0), both warp tilings (8 or 16
    query rows per warp; GQA 16 always takes 16)."""
    monkeypatch.setenv("KVSLAB_PREFILL_TC", "0")
    monkeypatch.setenv("KVSLAB_PREFILL_NT", nt)
    _, _, _, _, o, _, r, _ = run_prefill(KvDtype.INT8, 2, 8, [(300, 45), (700, 161), (5, 5)], seed=21)
    assert rel_err(o, r) <= 1e-2


@pytest.mark.parametrize("dt", FORMATS, ids=[d.name for d in FORMATS])
def test_prefill_mma_sync_path_all_formats(dt, monkeypatch):
    monkeypatch.setenv("KVSLAB_PREFILL_TC", "0")
    _, _, _, _, o, _, r, _ = run_prefill(dt, 2, 8, CASES, seed=31 + int(dt))
    assert rel_err(o, r) <= TOL[dt]


def test_prefill_long_chunk_fp8():
    """A 2k-token whole-prompt chunk (many tiles, heaviest first)."""
    _, _, _, _, o, _, r, _ = run_prefill(KvDtype.FP8_E4M3, 2, 8, [(2048, 2048), (900, 300)], seed=9)
    assert rel_err(o, r) <= 1e-3


def test_prefill_rejects_bad_group():
    fmt = KvFormat(KvDtype.FP16, 1, 32)
    w = make_world(fmt, [16], churn=False)
    q = torch.zeros((16, 32, 128), dtype=torch.float16, device="cuda")
    cu = dev(np.array([0, 16], np.int32))
    with pytest.raises(Exception, match="GQA"):
        kv.paged_prefill(w["pool"], fmt, 0, q, dev(w["table"]), cu, dev(w["ctx"]), 16)


@pytest.mark.parametrize("dt", [KvDtype.FP16, KvDtype.FP8_E4M3], ids=["FP16", "FP8"])
def test_prefill_tc_long_context_and_layer(dt):
    """tcgen05 path: a chunk at the end of a 3k context (47 KV tiles, 3-stage
    ring wraps many times), layer 1 of a 2-layer key, plus a 1-token chunk."""
    _, _, _, _, o, lse, r, rl = run_prefill(dt, 2, 8, [(3000, 300), (129, 1), (64, 64)], seed=41,
                                            layers=2, layer=1)
    assert rel_err(o, r) <= TOL[dt]
    assert np.abs(lse - rl).max() <= 1e-3


def test_prefill_tc_int4_gqa1_ragged():
    """tcgen05 path, MHA (256 tokens per CTA), ragged chunks incl. empty ones."""
    _, _, _, _, o, lse, r, rl = run_prefill(KvDtype.INT4, 2, 2, [(513, 300), (40, 0), (1000, 257), (3, 3)],
                                            seed=43)
    assert rel_err(o, r) <= 1e-2
    assert np.abs(lse - rl).max() <= 1e-3



QUANT = [d for d in FORMATS if d != KvDtype.FP16]


@pytest.mark.parametrize("expand", ["0", "1"], ids=["direct", "expand"])
@pytest.mark.parametrize("dt", QUANT, ids=[d.name for d in QUANT])
def test_prefill_quantised_direct_and_expand(dt, expand, monkeypatch):
    """Both quantised K4 forms agree with the oracle: the direct tcgen05 kernel
    (dequantising loaders) and expand-once (context -> fp16 scratch blocks, then
    the FP16 kernel over an identity table), on layer 1 of a 2-layer key with
    ragged, empty and whole-prompt chunks."""
    monkeypatch.setenv("KVSLAB_PREFILL_EXPAND", expand)
    _, _, _, _, o, lse, r, rl = run_prefill(dt, 2, 8, [(1500, 700), (129, 1), (64, 64), (40, 0), (333, 333)],
                                            seed=51 + int(dt), layers=2, layer=1)
    assert rel_err(o, r) <= TOL[dt]
    assert np.abs(lse - rl).max() <= 1e-3


def test_prefill_workspace_none_and_size():
    """workspace=None runs the direct kernel; the size query is 0 for FP16 and
    batch x bt_stride fp16 blocks (+ the K scale/zero arrays) otherwise."""
    import ctypes as C
    from paper_2509_06261_b200 import _lib as L
    for dt, want in [(KvDtype.FP16, 0), (KvDtype.INT4, 3 * 10 * (2 * 4 * 16 * 128 * 2 + 4 * 128))]:
        f = KvFormat(dt, 4, 16).to_c()
        n = C.c_size_t()
        assert L.lib.ks_paged_prefill_workspace_size(C.byref(f), 3, 10, 8192, C.byref(n)) == 0
        assert n.value == want
    fmt = KvFormat(KvDtype.INT8, 2, 8)
    w = make_world(fmt, [600], seed=2)
    append_gpu(w, fmt, 0)
    q = torch.randn((600, 8, 128), dtype=torch.float16, device="cuda")
    cu = dev(np.array([0, 600], np.int32))
    a = kv.paged_prefill(w["pool"], fmt, 0, q, dev(w["table"]), cu, dev(w["ctx"]), 600, workspace=None)
    b = kv.paged_prefill(w["pool"], fmt, 0, q, dev(w["table"]), cu, dev(w["ctx"]), 600)
    torch.cuda.synchronize()
    assert (a - b).abs().max().item() <= 2e-2 * b.abs().max().item()


def test_prefill_expand_in_sequence_groups(monkeypatch):
    """A workspace for one sequence takes the batch one sequence at a time."""
    monkeypatch.setenv("KVSLAB_PREFILL_SPLIT", "0")  # same kernels both ways -> identical bits
    fmt = KvFormat(KvDtype.INT4, 2, 8)
    cases = [(700, 300), (129, 129), (1000, 256), (40, 0)]
    w, _, q, cu, o_full, _, r, _ = run_prefill(KvDtype.INT4, 2, 8, cases, seed=61)
    import ctypes as C
    from paper_2509_06261_b200 import _lib as L
    one = C.c_size_t()
    # one sequence's expand scratch only (max_q_len large enough that no split is sized)
    L.lib.ks_paged_prefill_workspace_size(C.byref(fmt.to_c()), 1, w["table"].shape[1], 1 << 16, C.byref(one))
    ws = torch.empty(one.value, dtype=torch.uint8, device="cuda")
    o = kv.paged_prefill(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(cu), dev(w["ctx"]),
                         max(n for _, n in cases), workspace=ws)
    torch.cuda.synchronize()
    o = o.cpu().numpy().astype(np.float64)
    assert rel_err(o, r) <= 1e-2
    assert np.abs(o - o_full).max() == 0.0  # the same kernels, sequence by sequence


SPLIT_CASES = [
    # (dtype, H, Hq, cases): short chunks over long contexts -> few query tiles, split-KV
    (KvDtype.FP16, 2, 8, [(3000, 16), (1500, 64), (64, 64), (900, 0)]),
    (KvDtype.FP8_E4M3, 2, 8, [(2500, 40), (333, 33)]),
    (KvDtype.INT8, 2, 16, [(2000, 64), (17, 17)]),
    (KvDtype.INT4, 2, 8, [(4100, 64), (700, 1)]),
    (KvDtype.INT4, 1, 4, [(1000, 300)]),
]


@pytest.mark.parametrize("split", ["0", "1"], ids=["nosplit", "split"])
@pytest.mark.parametrize("dt,H,Hq,cases", SPLIT_CASES,
                         ids=[f"{c[0].name}-{c[1]}x{c[2]}-{len(c[3])}" for c in SPLIT_CASES])
def test_prefill_split_kv(dt, H, Hq, cases, split, monkeypatch):
    """Split-KV K4 (query tiles x KV ranges over up to 8 CTAs, fp32 partials,
    merge kernel) and the unsplit kernel both match the oracle, including
    empty splits (ranges past a short context) and the direct / expand forms
    of the quantised formats."""
    monkeypatch.setenv("KVSLAB_PREFILL_SPLIT", split)
    monkeypatch.setenv("KVSLAB_PREFILL_TC", "1")  # tcgen05 even for the shortest chunks
    _, _, _, _, o, lse, r, rl = run_prefill(dt, H, Hq, cases, seed=71 + int(dt) + H)
    assert rel_err(o, r) <= TOL[dt]
    assert np.abs(lse - rl).max() <= 1e-3


@pytest.mark.parametrize("dt", [KvDtype.FP16, KvDtype.INT4], ids=["FP16", "INT4"])
def test_prefill_workspace_sizes_degrade_gracefully(dt):
    """Any workspace size is valid: a buffer too small for the split-KV
    partials drops the split (quantised formats then expand in sequence
    groups if they fit one sequence, else run direct); every size gives the
    oracle's answer."""
    import ctypes as C
    from paper_2509_06261_b200 import _lib as L
    cases = [(3000, 64), (700, 1)]
    w, fmt, q, cu, o_ref, _, r, _ = run_prefill(dt, 2, 8, cases, seed=81)
    nq = max(n for _, n in cases)
    full = C.c_size_t()
    L.lib.ks_paged_prefill_workspace_size(C.byref(fmt.to_c()), len(cases), w["table"].shape[1], nq,
                                          C.byref(full))
    for nbytes in (0, 4096, full.value // 3, full.value):
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        o = kv.paged_prefill(w["pool"], fmt, 0, dev(q), dev(w["table"]), dev(cu), dev(w["ctx"]), nq,
                             workspace=ws if nbytes else None)
        torch.cuda.synchronize()
        assert rel_err(o.cpu().numpy().astype(np.float64), r) <= TOL[dt], nbytes

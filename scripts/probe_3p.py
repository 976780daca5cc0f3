import time, torch
t0 = time.time()
import vllm._C  # noqa
print("vllm _C loaded", time.time() - t0)
print([n for n in dir(torch.ops._C) if 'attention' in n or 'cache' in n or 'fp8' in n][:40])
print([n for n in dir(torch.ops._C_cache_ops)])
for op in ("reshape_and_cache_flash", "reshape_and_cache"):
    try:
        print(getattr(torch.ops._C_cache_ops, op).default._schema)
    except Exception as e:
        print(op, e)
for op in ("paged_attention_v1", "paged_attention_v2"):
    try:
        print(getattr(torch.ops._C, op).default._schema)
    except Exception as e:
        print(op, e)
t0 = time.time()
try:
    import flashinfer
    H, Hq, D, ps = 8, 32, 128, 16
    B, nb = 2, 4
    kvc = torch.randn(B * nb, 2, ps, H, D, dtype=torch.float16, device="cuda")
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    indptr = torch.tensor([0, nb, 2 * nb], dtype=torch.int32, device="cuda")
    idx = torch.arange(B * nb, dtype=torch.int32, device="cuda")
    last = torch.tensor([ps, 5], dtype=torch.int32, device="cuda")
    w.plan(indptr, idx, last, Hq, H, D, ps, q_data_type=torch.float16, kv_data_type=torch.float16)
    q = torch.randn(B, Hq, D, dtype=torch.float16, device="cuda")
    o = w.run(q, kvc)
    torch.cuda.synchronize()
    print("flashinfer decode fp16 ok", o.shape, time.time() - t0)
    kv8 = kvc.to(torch.float8_e4m3fn)
    w.plan(indptr, idx, last, Hq, H, D, ps, q_data_type=torch.float16, kv_data_type=torch.float8_e4m3fn)
    o8 = w.run(q, kv8, k_scale=0.5, v_scale=0.5)
    torch.cuda.synchronize()
    print("flashinfer decode fp8 ok", time.time() - t0)
except Exception as e:
    import traceback; traceback.print_exc()
    print("flashinfer failed", time.time() - t0)

import time, torch
print("torch", torch.__version__, torch.cuda.get_device_capability())
try:
    import flash_attn
    from flash_attn import flash_attn_varlen_func
    q = torch.randn(1024, 32, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1024, 8, 128, device="cuda", dtype=torch.bfloat16)
    cu = torch.tensor([0, 512, 1024], dtype=torch.int32, device="cuda")
    o = flash_attn_varlen_func(q, k, k, cu, cu, 512, 512, causal=True)
    torch.cuda.synchronize(); print("flash_attn ok", flash_attn.__version__)
except Exception as e:
    print("flash_attn FAIL", type(e).__name__, str(e)[:200])
try:
    import flashinfer
    print("flashinfer", flashinfer.__version__)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD")
    qo = torch.tensor([0, 512, 1024], dtype=torch.int32, device="cuda")
    t0 = time.time()
    w.plan(qo, qo, 32, 8, 128, causal=True, q_data_type=torch.bfloat16)
    o = w.run(q, k, k)
    torch.cuda.synchronize(); print("flashinfer ok", time.time() - t0, "s")
except Exception as e:
    print("flashinfer FAIL", type(e).__name__, str(e)[:300])
try:
    import torch.nn.functional as F
    qq = torch.randn(1, 32, 512, 128, device="cuda", dtype=torch.bfloat16)
    kk = torch.randn(1, 32, 512, 128, device="cuda", dtype=torch.bfloat16)
    from torch.nn.attention import sdpa_kernel, SDPBackend
    for be in (SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel(be):
                F.scaled_dot_product_attention(qq, kk, kk, is_causal=True)
            torch.cuda.synchronize(); print("sdpa", be, "ok")
        except Exception as e:
            print("sdpa", be, "FAIL", str(e)[:100])
except Exception as e:
    print("sdpa FAIL", e)

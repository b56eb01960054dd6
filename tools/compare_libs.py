"""Library baselines at this framework's prefill shapes on the same B200
(reference points, not part of the product path): cuBLAS bf16 GEMMs via
torch.matmul for the four Llama-3-8B projections at 2048 rows, and
flashinfer's / flash-attn's causal GQA prefill attention (32 q heads, 8 kv
heads, head_dim 128, 2048 tokens) when they run on sm_100.

    python tools/compare_libs.py
"""
import json
import sys

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    out = {"gemm_cublas": {}, "attention": {}}
    M = 2048
    for name, (n, k) in {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096),
                         "down": (4096, 14336)}.items():
        a = torch.randn(M, k, device="cuda").bfloat16()
        b = torch.randn(n, k, device="cuda").bfloat16()
        us = timed(lambda: torch.matmul(a, b.t()))
        out["gemm_cublas"][name] = {"us": round(us, 2), "tflops": round(2 * M * n * k / us / 1e6, 1)}
    S, H, KV, D = 2048, 32, 8, 128
    flops = 4 * S * S * H * D / 2  # causal
    q = torch.randn(S, H, D, device="cuda").bfloat16()
    kk = torch.randn(S, KV, D, device="cuda").bfloat16()
    v = torch.randn(S, KV, D, device="cuda").bfloat16()
    try:
        import flashinfer
        us = timed(lambda: flashinfer.single_prefill_with_kv_cache(q, kk, v, causal=True))
        out["attention"]["flashinfer_single_prefill"] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
    except Exception as e:  # noqa: BLE001
        out["attention"]["flashinfer_single_prefill"] = {"error": str(e)[:200]}
    try:
        from flash_attn import flash_attn_func
        us = timed(lambda: flash_attn_func(q[None], kk[None], v[None], causal=True))
        out["attention"]["flash_attn2"] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
    except Exception as e:  # noqa: BLE001
        out["attention"]["flash_attn2"] = {"error": str(e)[:200]}
    try:
        us = timed(lambda: torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1)[None], kk.transpose(0, 1)[None].repeat_interleave(H // KV, 1),
            v.transpose(0, 1)[None].repeat_interleave(H // KV, 1), is_causal=True))
        out["attention"]["torch_sdpa_incl_kv_repeat"] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
    except Exception as e:  # noqa: BLE001
        out["attention"]["torch_sdpa_incl_kv_repeat"] = {"error": str(e)[:200]}
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())

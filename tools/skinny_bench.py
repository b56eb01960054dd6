"""Decode-shaped (skinny) GEMMs back to back at M = 1 and 64 for the QKV, O
and down shapes (fp32 residual epilogue, impl 4), incl. the split-K fix-up:
us per call and weight GB/s.

    python tools/skinny_bench.py
"""
import ctypes as C, sys, torch, json
sys.path.insert(0, "/root/repo")
from paper_2512_09472_b200 import _native as N
from paper_2512_09472_b200 import models  # noqa
out = {}
for M in (1, 64):
    for name, (n, k) in {"qkv": (6144, 4096), "o": (4096, 4096), "down": (4096, 14336)}.items():
        A = torch.randn(M, k, device="cuda").bfloat16(); B = (torch.randn(n, k, device="cuda") * 0.02).bfloat16()
        Cm = torch.zeros(M, n, device="cuda")
        f = lambda: N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, n, k, 2, C.c_void_p(Cm.data_ptr()), None, 4, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(3): f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): f()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        out[f"{name}_M{M}"] = (round(us, 2), round(n * k * 2 / us / 1e3))
print(json.dumps(out))

"""Decode-shaped (skinny) GEMMs back to back at M = 1, 16 and 64 for the
8B QKV, O, gate/up (SwiGLU) and down shapes (impl 4): us per call and weight
GB/s (--phi: the Phi-3-mini shapes). Env WS_SKINNY_CLUSTER=0 / WS_SKINNY_CLUSTER_MAX=C for A/B.

    python tools/skinny_bench.py [--phi] [M,M,...] [--only=qkv,o,gateup,down]
"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2512_09472_b200 import _native as N  # noqa: E402
from paper_2512_09472_b200 import models  # noqa: E402,F401  (registers ws_gemm)

SHAPES = {"qkv": (6144, 4096, 2), "o": (4096, 4096, 2), "gateup": (28672, 4096, 4), "down": (4096, 14336, 2)}
if "--phi" in sys.argv:  # Phi-3-mini
    SHAPES = {"qkv": (9216, 3072, 2), "o": (3072, 3072, 2), "gateup": (16384, 3072, 4), "down": (3072, 8192, 2)}
out = {}
MS = [int(x) for x in next((a for a in sys.argv[1:] if a[0].isdigit()), "1,16,64").split(",")]
ONLY = next((a.split("=")[1].split(",") for a in sys.argv[1:] if a.startswith("--only=")), None)
for M in MS:
    for name, (n, k, epi) in SHAPES.items():
        if ONLY and name not in ONLY:
            continue
        A = torch.randn(M, k, device="cuda").bfloat16()
        B = (torch.randn(n, k, device="cuda") * 0.02).bfloat16()
        Cm = torch.zeros(M, n // 2, device="cuda", dtype=torch.bfloat16) if epi == 4 else torch.zeros(M, n, device="cuda")
        f = lambda: N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, n, k, epi,
                           C.c_void_p(Cm.data_ptr()), None, 4, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        out[f"{name}_M{M}"] = (round(us, 2), round(n * k * 2 / us / 1e3))
print(json.dumps(out))

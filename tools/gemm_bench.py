"""Time the prefill GEMM shapes on the tcgen05 pair kernel (impl 3) with CUDA
events: back-to-back launches of one shape, TFLOP/s per shape.

    python tools/gemm_bench.py [--m 2048] [--reps 20] [--only gate_up,o] [--zero-rows=a:b] [--const-rows=a:b]
      (WS_STREAMK=0 to A/B; --zero-rows probes data-dependent epilogue cost)
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models  # noqa: F401

    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    a, _ = ap.parse_known_args()
    M = a.m
    shapes = {"qkv": (6144, 4096, 5), "o": (4096, 4096, 2), "gate_up": (28672, 4096, 4), "down": (4096, 14336, 2)}
    out = {}
    for name, (n, k, epi) in shapes.items():
        if a.only and name not in a.only.split(","):
            continue
        A = torch.randn((M + 255) // 256 * 256, k, device="cuda").bfloat16()  # rows past M: --zero-rows probes
        for arg in sys.argv:  # --zero-rows=a:b  zero rows [a, b) of A (data-dependence probe)
            if arg.startswith("--zero-rows="):
                a0, a1 = map(int, arg.split("=")[1].split(":"))
                A[a0:a1] = 0
            if arg.startswith("--const-rows="):
                a0, a1 = map(int, arg.split("=")[1].split(":"))
                A[a0:a1] = 0.01
        B = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
        if epi == 2:
            Cm = torch.zeros(M, n, device="cuda")
        else:
            Cm = torch.empty(M, n, device="cuda", dtype=torch.bfloat16)
        e = 0 if epi == 5 else epi  # RoPE needs a pool; time the plain bf16 store for QKV
        def once():
            N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, n, k, e,
                   C.c_void_p(Cm.data_ptr()), None, 3, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(3):
            once()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            once()
        t1.record()
        torch.cuda.synchronize()
        us = t0.elapsed_time(t1) / a.reps * 1e3
        out[name] = {"us": round(us, 2), "tflops": round(2.0 * M * n * k / us / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

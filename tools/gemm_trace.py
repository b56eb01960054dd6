"""Per-CTA globaltimer timeline of one pair-GEMM launch (library built with
WS_GEMM_TRACE=1, e.g. `touch csrc/kernels/gemm_tc.cu; WS_GEMM_TRACE=1 python -c
"from paper_2512_09472_b200 import build; build.build()"`).

    python tools/gemm_trace.py --shape o
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def main():
    import torch
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models  # noqa: F401

    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="o")
    ap.add_argument("--m", type=int, default=2048)
    a = ap.parse_args()
    n, k = SHAPES[a.shape]
    M = a.m
    A = torch.randn(M, k, device="cuda").bfloat16()
    B = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    Cm = torch.zeros(M, n, device="cuda")
    for _ in range(4):
        N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, n, k, 2,
               C.c_void_p(Cm.data_ptr()), None, 3, None)  # epi 2 = x += A.B^T
    torch.cuda.synchronize()
    buf = (C.c_longlong * (148 * 8))()
    N.lib.ws_gemm_trace(buf)
    t = [[buf[c * 8 + j] for j in range(8)] for c in range(148)]
    t0 = min(r[0] for r in t if r[0])
    rel = lambda x: (x - t0) / 1e3 if x else float("nan")
    ends = sorted(rel(r[7]) for r in t)
    print(f"{a.shape}: end min {ends[0]:.1f} median {ends[74]:.1f} max {ends[-1]:.1f} us")
    for c in range(0, 148, 2):
        r = t[c]
        print(f"pair {c // 2:3d} start {rel(r[0]):6.1f} ready " + " ".join(f"{rel(x):6.1f}" for x in r[1:4]) +
              " done " + " ".join(f"{rel(x):6.1f}" for x in r[4:7]) + f" end {rel(r[7]):6.1f}")


if __name__ == "__main__":
    main()

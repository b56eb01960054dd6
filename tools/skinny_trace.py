"""Per-CTA globaltimer timeline of one skinny-GEMM launch (decode shapes),
launched back to back as in a decode step (PDL overlap with the previous
launch). Needs the library built with WS_SKINNY_TRACE=1:

    WS_SKINNY_TRACE=1 python -m paper_2512_09472_b200.build -f && python tools/skinny_trace.py [--m 1] [--shape o]

Prints, per phase, the median / max over CTAs of the time since the earliest
CTA entry (us): 1 setup done, 2 past the PDL wait, 3 first stage landed,
4 last MMA committed, 5 first accumulator ready, 6 epilogue done, 7 past the
first cluster barrier, 8 reduce done, 9 exit.
"""
import argparse
import ctypes as C
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

SHAPES = {"qkv": (6144, 4096, 2), "o": (4096, 4096, 2), "gateup": (28672, 4096, 4), "down": (4096, 14336, 2)}
NAMES = ["entry", "setup", "pdl_wait", "first_stage", "last_mma", "acc_ready", "epi_done", "cluster1", "reduce",
         "exit"]


def main():
    import torch

    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models  # noqa: F401

    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--shape", default="o,down,qkv,gateup")
    a = ap.parse_args()
    for shape in a.shape.split(","):
        n, k, epi = SHAPES[shape]
        A = torch.randn(a.m, k, device="cuda").bfloat16()
        B = (torch.randn(n, k, device="cuda") * 0.02).bfloat16()
        Cm = (torch.zeros(a.m, n // 2, device="cuda", dtype=torch.bfloat16) if epi == 4
              else torch.zeros(a.m, n, device="cuda"))
        st = torch.cuda.current_stream().cuda_stream
        buf = (C.c_longlong * (148 * 10))()
        N.lib.ws_skinny_trace(buf)  # clear state read
        zero = (C.c_longlong * (148 * 10))()
        for _ in range(20):
            N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), a.m, n, k, epi,
                   C.c_void_p(Cm.data_ptr()), None, 4, C.c_void_p(st))
        torch.cuda.synchronize()
        N.lib.ws_skinny_trace(buf)
        rows = [[buf[c * 10 + j] for j in range(10)] for c in range(148)]
        rows = [r for r in rows if r[0] and r[9] and r[9] >= r[0]]
        t0 = min(r[0] for r in rows)
        t_end = max(r[9] for r in rows)
        print(f"{shape} M={a.m}: {len(rows)} CTAs, launch span {(t_end - t0) / 1e3:.2f} us")
        for j in range(10):
            v = [(r[j] - t0) / 1e3 for r in rows if r[j] >= t0]
            if v:
                print(f"  {j} {NAMES[j]:11s} median {statistics.median(v):6.2f}  max {max(v):6.2f}  min {min(v):6.2f}")
        del zero


if __name__ == "__main__":
    main()

"""clock64 timeline of the one-head attention kernel (attn_tc_kernel, WS_ATTN_PAIR=0), CTA (0,0)."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ["WS_ATTN_PAIR"] = "0"


def main():
    import torch
    from attn_bench import AttnRig

    from paper_2512_09472_b200 import _native as N

    rig = AttnRig("llama3-8b", 2048)
    q = torch.randn(2048, rig.H * rig.hd, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    for _ in range(3):
        rig.run(q, 2048, 0)
    torch.cuda.synchronize()
    buf = (C.c_longlong * 512)()
    N.lib.ws_attn_trace(buf)
    ev = lambda e, j: buf[e * 64 + j]
    t0 = ev(0, 0)
    names = ["S(j) issued", "PV(j) issued", "sm got S", "sm P done"]
    for e in range(4):
        print(names[e].ljust(14), " ".join(f"{(ev(e, j) - t0) if ev(e, j) else -1:7d}" for j in range(16)))
    for j in range(1, 16):
        print(f"j={j:2d} softmax {ev(3, j) - ev(2, j):6d}  wait S {ev(2, j) - ev(3, j - 1):6d}  S issue->got {ev(2, j) - ev(0, j):6d}")
    rig.close()


if __name__ == "__main__":
    main()

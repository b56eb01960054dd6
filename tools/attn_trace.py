"""clock64 timeline of the first work item of attention CTA 0 and per-CTA
start/end times, on the attn_bench rig (8B shape, 2048 tokens).

Needs the library built with WS_ATTN_TRACE=1:
    WS_ATTN_TRACE=1 python -m paper_2512_09472_b200.build -f && python tools/attn_trace.py
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def main():
    import torch
    from attn_bench import AttnRig

    from paper_2512_09472_b200 import _native as N

    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    rig = AttnRig("llama3-8b", rows)
    q = torch.randn(rows, rig.H * rig.hd, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    for _ in range(3):
        rig.run(q, rows, 0)
    torch.cuda.synchronize()
    buf = (C.c_longlong * 512)()
    N.lib.ws_attn_trace(buf)
    ev = lambda e, j: buf[e * 64 + j]
    t0 = ev(0, 0)
    names = ["S_A(j) issued", "PV_A(j) issued", "smA got S", "smA P done", "smA S in regs", "smA max done",
             "smA exp done", "smA O ready"]
    n = 16
    print("event".ljust(16), " ".join(f"{j:7d}" for j in range(n)))
    for e in range(8):
        print(names[e].ljust(16), " ".join(f"{(ev(e, j) - t0) if ev(e, j) else -1:7d}" for j in range(n)))
    print("MMA warp first K landed", ev(2, 63) - t0, "| CTA done", ev(1, 63) - t0)
    # per-step deltas of the softmax
    for j in range(1, n):
        if ev(2, j) and ev(3, j):
            print(f"j={j:2d} wait S {ev(2, j) - ev(3, j - 1):6d}  tmem ld {ev(4, j) - ev(2, j):5d}  max {ev(5, j) - ev(4, j):5d}"
                  f"  exp {ev(6, j) - ev(5, j):5d}  store+pvwait {ev(7, j) - ev(6, j):5d}  corr+arrive {ev(3, j) - ev(7, j):5d}"
                  f"  | S issue->got {ev(2, j) - ev(0, j):6d}  P done->PV issue {ev(1, j) - ev(3, j):6d}")
    cta = (C.c_longlong * (4096 * 3))()
    N.lib.ws_attn_cta_trace(cta)
    rows_ = [(cta[i * 3], cta[i * 3 + 1], cta[i * 3 + 2]) for i in range(148)]
    g0 = min(r[0] for r in rows_)
    d = sorted((r[1] - r[0]) / 1e3 for r in rows_)
    st = sorted((r[0] - g0) / 1e3 for r in rows_)
    print(f"CTAs: start spread {st[0]:.1f}-{st[-1]:.1f} us, duration min {d[0]:.1f} med {d[74]:.1f} max {d[-1]:.1f} us")
    rig.close()


if __name__ == "__main__":
    main()

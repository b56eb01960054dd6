"""Print the clock64 timeline of attention CTA (0,0) (build with WS_ATTN_TRACE=1)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import subprocess
    subprocess.run([sys.executable, str(Path(__file__).parent / "prefill_profile.py"), "--iters", "1"], check=True)


if __name__ == "__main__":
    import torch
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import fill_flat
    from paper_2512_09472_b200.worker import UniversalWorker
    cfg = M.LLAMA3_8B.with_(layers=1)
    w = UniversalWorker(0, pool_pages=2048, max_tokens=2048)
    w.register(cfg, None)
    w.prewarm(cfg.name, layers=1)
    fill_flat(cfg, w.slot_view(cfg.name), seed=0)
    w.switch_memory(cfg.name)
    toks = torch.randint(0, cfg.vocab, (2048,), dtype=torch.int32, device="cuda")
    for _ in range(2):
        with torch.cuda.stream(w.compute):
            s = w.open_seq(2048); w.prefill(s, toks); w.close_seq(s)
        torch.cuda.synchronize()
    buf = (C.c_longlong * 512)()
    N.lib.ws_attn_trace(buf)
    t = [[buf[e * 64 + j] for j in range(16)] for e in range(8)]
    t0 = buf[0]
    names = ["S issued", "PV issued", "softmax got S", "softmax P done", "sm S in regs", "sm max done",
             "sm exp done", "sm P stored+PV"]
    for e in range(8):
        print(f"{names[e]:16s}", " ".join(f"{(x - t0) if x else -1:7d}" for x in t[e]))
    print("CTA start 0 | Q landed", t[2][62] - t[0][0] if False else buf[2 * 64 + 62] - buf[0],
          "| K0 landed", buf[2 * 64 + 63] - buf[0], "| O complete", buf[64 + 62] - buf[0],
          "| epilogue stored", buf[64 + 63] - buf[0])
    cta = (C.c_longlong * (4096 * 3))()
    N.lib.ws_attn_cta_trace(cta)
    import os
    persistent = os.environ.get("WS_ATTN_PAIR") != "0"
    nh = 32
    n = 148 if persistent else 32 * 16
    rows = [(cta[i * 3], cta[i * 3 + 1], cta[i * 3 + 2]) for i in range(n)]
    g0 = min(r[0] for r in rows)
    ends = sorted((r[1] - g0) / 1e3 for r in rows)
    print(f"CTAs: last end {ends[-1]:.1f} us; median end {ends[len(ends) // 2]:.1f}")
    per_sm = {}
    for (a, b, sm) in rows:
        per_sm.setdefault(sm, []).append(((a - g0) / 1e3, (b - g0) / 1e3))
    busy = sorted(sum(b - a for a, b in v) for v in per_sm.values())
    last = sorted(max(b for a, b in v) for v in per_sm.values())
    print(f"SMs used {len(per_sm)}; busy us min {busy[0]:.1f} med {busy[len(busy)//2]:.1f} max {busy[-1]:.1f}; "
          f"last end min {last[0]:.1f} max {last[-1]:.1f}")
    if persistent:
        d = sorted((r[1] - r[0]) / 1e3 for r in rows)
        print(f"persistent CTAs: duration min {d[0]:.1f} median {d[74]:.1f} max {d[-1]:.1f} us")
        sys.exit(0)
    for qt in range(16):
        durs = [(rows[qt * nh + h][1] - rows[qt * nh + h][0]) / 1e3 for h in range(nh)]
        st = [(rows[qt * nh + h][0] - g0) / 1e3 for h in range(nh)]
        print(f"grid row {qt:2d} (q tile {15 - qt:2d}): start {min(st):6.1f}-{max(st):6.1f} dur {min(durs):5.1f}-{max(durs):5.1f} us")

"""Warm prefill back to back with nvidia-smi sampling: per-iteration device
time next to SM clock / power, to separate kernel efficiency from the power
cap under sustained tensor-core load.

    python tools/prefill_power.py [--model llama3-8b] [--tokens 2048] [--iters 40] [--gap-ms 0]
"""

from __future__ import annotations

import argparse
import json
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import fill_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--gap-ms", type=float, default=0.0)
    ap.add_argument("--pool-pages", type=int, default=9216)
    ap.add_argument("--tp", type=int, default=1,
                    help="time one rank's shard (tp.shard_config) on this GPU: the per-rank compute of a "
                         "TP prefill, allreduce excluded; the lm_head stays whole")
    a = ap.parse_args()
    cfg = M.ALL[a.model]
    if a.tp > 1:
        from paper_2512_09472_b200.tp import shard_config
        cfg = shard_config(cfg, a.tp).with_(lm_head_rows=0)
    w = UniversalWorker(0, pool_pages=a.pool_pages, max_tokens=max(a.tokens, 256))
    w.register(cfg, None)
    w.prewarm(cfg.name, layers=cfg.layers)
    fill_flat(cfg, w.slot_view(cfg.name), seed=0)
    w.slot(cfg.name).layers_loaded = cfg.layers
    w.switch_memory(cfg.name)
    toks = torch.randint(0, cfg.vocab, (a.tokens,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits", "-lms", "50", "-i", "0"],
                           stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    evs = []
    with torch.cuda.stream(w.compute):
        for i in range(a.iters):
            s = w.open_seq(a.tokens)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(w.compute)
            w.prefill(s, toks)
            e1.record(w.compute)
            w.close_seq(s)
            evs.append((e0, e1))
            if a.gap_ms:
                torch.cuda.synchronize()
                time.sleep(a.gap_ms / 1e3)
    torch.cuda.synchronize()
    time.sleep(0.2)
    smi.terminate()
    out, _ = smi.communicate()
    ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    clk = [float(r.split(",")[1]) for r in out.strip().splitlines() if r.count(",") >= 3]
    pw = [float(r.split(",")[2]) for r in out.strip().splitlines() if r.count(",") >= 3]
    res = {"model": cfg.name, "tp": a.tp, "tokens": a.tokens, "gap_ms": a.gap_ms, "ms": [round(x, 3) for x in ms],
           "ms_first3": ms[:3], "ms_median_last_half": sorted(ms[len(ms) // 2:])[len(ms) // 4],
           "sm_mhz": clk, "power_w": pw}
    print(json.dumps(res))
    w.release()
    w.close()


if __name__ == "__main__":
    main()

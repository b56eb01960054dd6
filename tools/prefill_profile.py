"""Warm prefill of a model on one GPU, for ncu launch lists / captures.

    python tools/prefill_profile.py [--model llama3-8b] [--tokens 2048] [--iters 2] [--gemm 0|1]

Weights are synthesized straight into the slot (all layers resident); no
pinned host image is built, so the process stays small under ncu replay.
"""

from __future__ import annotations

import argparse
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
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--gemm", type=int, default=0)
    ap.add_argument("--pool-pages", type=int, default=9216)
    a = ap.parse_args()
    cfg = M.ALL[a.model]
    w = UniversalWorker(0, pool_pages=a.pool_pages, max_tokens=max(a.tokens, 256))
    w.register(cfg, None)
    w.prewarm(cfg.name, layers=cfg.layers)  # maps every page; no host source
    fill_flat(cfg, w.slot_view(cfg.name), seed=0)
    w.slot(cfg.name).layers_loaded = cfg.layers
    w.set_gemm_impl(a.gemm)
    w.switch_memory(cfg.name)
    toks = torch.randint(0, cfg.vocab, (a.tokens,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    dev_ms = []
    for i in range(a.iters):
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(w.compute):
            s = w.open_seq(a.tokens)
            e0.record(w.compute)
            w.prefill(s, toks)
            e1.record(w.compute)
            w.close_seq(s)
        torch.cuda.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
        print(f"prefill {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms wall, {dev_ms[-1]:.3f} ms device", flush=True)
    if len(dev_ms) > 2:
        tail = sorted(dev_ms[2:])
        print(f"device median {tail[len(tail) // 2]:.3f} ms min {tail[0]:.3f} ms over {len(tail)}", flush=True)
    w.release()
    w.close()


if __name__ == "__main__":
    main()

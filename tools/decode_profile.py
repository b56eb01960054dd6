"""Warm decode throughput of a model on one GPU (HBM roofline check).

    python tools/decode_profile.py [--model llama3-8b] [--batch 1,8,32,64] [--ctx 2048] [--steps 20]

Every sequence is prefilled to --ctx tokens once, then decode steps run with
all sequences advancing one token per step. Device time per step (CUDA events
on the compute stream) and the algorithmic bytes per step — every weight byte
except the embedding table (only B rows are gathered) plus each sequence's K/V
for every layer — give the achieved HBM bandwidth.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import fill_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--batch", default="1,8,32,64")
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--pool-pages", type=int, default=24576)
    ap.add_argument("--json", default="")
    ap.add_argument("--graphed", action="store_true", help="CUDA-graph replay (UniversalWorker.decode_graphed)")
    ap.add_argument("--back-to-back", action="store_true", help="time all steps between two events (as bench.py)")
    a = ap.parse_args()
    cfg = M.ALL[a.model]
    batches = [int(b) for b in a.batch.split(",")]
    bmax = max(batches)
    w = UniversalWorker(0, pool_pages=a.pool_pages, max_seqs=max(64, bmax), max_tokens=max(a.ctx, 256))
    w.register(cfg, None)
    w.prewarm(cfg.name, layers=cfg.layers)
    fill_flat(cfg, w.slot_view(cfg.name), seed=0)
    w.slot(cfg.name).layers_loaded = cfg.layers
    w.switch_memory(cfg.name)
    lay = w.models[cfg.name].layout
    embed_bytes = cfg.vocab * cfg.hidden * 2
    weight_bytes = lay.total - embed_bytes
    kv_tok = cfg.kv_geometry()[1]

    g = torch.Generator().manual_seed(0)
    seqs = []
    for _ in range(bmax):
        s = w.open_seq(a.ctx + a.steps + 8)
        toks = torch.randint(0, cfg.vocab, (a.ctx,), generator=g, dtype=torch.int32).cuda()
        with torch.cuda.stream(w.compute):
            w.prefill(s, toks)
        seqs.append(s)
    torch.cuda.synchronize()

    out = []
    for B in batches:
        sd = torch.tensor(seqs[:B], dtype=torch.int32, device="cuda")
        tok = torch.randint(0, cfg.vocab, (B,), generator=g, dtype=torch.int32).cuda()
        times = []
        for i in range(a.steps):
            # rewrite the same position each step so every batch size sees ctx = a.ctx
            pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(w.compute):
                e0.record(w.compute)
                torch.cuda.nvtx.range_push(f"decode_b{B}")
                step = w.decode_graphed if a.graphed else w.decode
                _, nt = step(sd, pos, tok, a.ctx + 1)
                torch.cuda.nvtx.range_pop()
                e1.record(w.compute)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            tok = nt.clone()
        t = sorted(times[3:])
        ms = t[len(t) // 2]
        if a.back_to_back:
            step = w.decode_graphed if a.graphed else w.decode
            with torch.cuda.stream(w.compute):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(w.compute)
                for i in range(a.steps):
                    pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
                    _, tok = step(sd, pos, tok, a.ctx + 1)
                e1.record(w.compute)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
        nbytes = weight_bytes + B * (a.ctx + 1) * kv_tok
        r = {"batch": B, "ctx": a.ctx, "ms_per_step": ms, "min_ms": t[0], "tokens_per_s": B / ms * 1e3,
             "algorithmic_gb": nbytes / 1e9, "achieved_gbs": nbytes / ms / 1e6}
        print(json.dumps(r), flush=True)
        out.append(r)
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))
    w.release()
    w.close()


if __name__ == "__main__":
    main()

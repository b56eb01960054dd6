"""Small workloads that launch every hand-written sm_100a kernel once or a
few times, sized for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck slow kernels down 10-1000x). tools/sanitize.sh runs this under each
tool and keeps the logs under profiles/.

Covered kernels: gemm_tc2 (CTA pair; bf16 / SwiGLU / RoPE+KV-append / TMA
reduce-add epilogues), gemm_tc (1-CTA), gemm_skinny (+ fix-up, folded norm,
fused RoPE fix-up), attn_tc2 (paired heads, TMA page rows), attn_tc
(odd GQA group; head_dim 96 cp.async gather), attn_decode (+ cluster merge /
combine), rmsnorm / rope_kv / embed / argmax, switch_kernel (promote,
reclaim with live-block migration), unpack_huff (packed stream), the layer
streamer's copies.

    python tools/sanitize_cases.py [case ...]   (default: all)
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _worker(cfg, pool_pages, max_tokens=1024):
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    w = UniversalWorker(0, pool_pages=pool_pages, max_tokens=max_tokens)
    flat = synth_flat(cfg, seed=3, device="cuda")
    host = pinned_host_copy(flat)
    w.register(cfg, host)
    return w, flat, host


def _prompt(cfg, n, seed=0):
    import torch

    return torch.randint(0, cfg.vocab, (n,), generator=torch.Generator().manual_seed(seed), dtype=torch.int32)


def _decode(w, cfg, seqs, pos, steps=2, graphed=False):
    import torch

    B = len(seqs)
    sd = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    tok = torch.randint(0, cfg.vocab, (B,), dtype=torch.int32, device="cuda")
    for i in range(steps):
        p = torch.tensor([x + i for x in pos], dtype=torch.int32, device="cuda")
        fn = w.decode_graphed if graphed else w.decode
        _, tok = fn(sd, p, tok, max(pos) + i + 1)
    torch.cuda.synchronize()


def case_tiny_cold():
    """tiny: packed cold activation (streamer + unpack + switch), decode,
    reclaim with live blocks (migration), release."""
    import torch

    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pack_stream

    cfg = M.TINY
    w, flat, _ = _worker(cfg, 64)
    try:
        w.set_packed(cfg.name, pack_stream(cfg, flat))
        w.prewarm(cfg.name, layers=1, full=False)
        w.activate_instance(cfg.name, _prompt(cfg, 512).pin_memory())
        s = w.open_seq(300)
        with torch.cuda.stream(w.compute):
            w.prefill(s, _prompt(cfg, 256, 1).cuda())
        torch.cuda.synchronize()
        _decode(w, cfg, [s], [256], steps=2)
        _decode(w, cfg, [s], [258], steps=2, graphed=True)
        w.reclaim(1)  # live blocks of s stay; the KV pool shrinks around them
        torch.cuda.synchronize()
        w.release()
    finally:
        w.close()


def _wide(name, **kw):
    from paper_2512_09472_b200 import models as M

    return M.TINY.with_(name=name, layers=1, vocab=4096, **kw)


def case_llama_width():
    """Llama-3-8B widths, 1 layer: pair GEMMs + fused epilogues, attn_tc2<128>,
    decode B = 1 / 4 / 24 (folded norm, fused RoPE fix-up, split decode)."""
    import torch

    cfg = _wide("w8b", hidden=4096, heads=32, kv_heads=8, head_dim=128, ffn=14336)
    w, _, _ = _worker(cfg, 400, max_tokens=1024)
    try:
        w.prewarm(cfg.name, layers=cfg.layers)
        w.switch_memory(cfg.name)
        seqs = []
        for b in range(24):
            n = 384 if b == 0 else 40 + 8 * b
            s = w.open_seq(n + 8)
            with torch.cuda.stream(w.compute):
                w.prefill(s, _prompt(cfg, n, b).cuda())
            seqs.append((s, n))
        torch.cuda.synchronize()
        for B in (1, 4, 24):
            _decode(w, cfg, [s for s, _ in seqs[:B]], [n for _, n in seqs[:B]], steps=1)
        w.release()
    finally:
        w.close()


def case_odd_groups():
    """Qwen2.5 widths (GQA group 7, QKV bias: attn_tc TMA one-head kernel) and
    Phi-3 widths (head_dim 96: attn_tc cp.async gather), 1 layer each."""
    import torch

    for cfg in (_wide("wq", hidden=3584, heads=28, kv_heads=4, head_dim=128, ffn=18944, qkv_bias=True),
                _wide("wp", hidden=3072, heads=32, kv_heads=32, head_dim=96, ffn=8192)):
        w, _, _ = _worker(cfg, 400, max_tokens=512)
        try:
            w.prewarm(cfg.name, layers=cfg.layers)
            w.switch_memory(cfg.name)
            s = w.open_seq(300)
            with torch.cuda.stream(w.compute):
                w.prefill(s, _prompt(cfg, 288).cuda())
            torch.cuda.synchronize()
            _decode(w, cfg, [s], [288], steps=1)
            w.release()
        finally:
            w.close()


CASES = {"tiny_cold": case_tiny_cold, "llama_width": case_llama_width, "odd_groups": case_odd_groups}


def main():
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n} ok", flush=True)


if __name__ == "__main__":
    main()

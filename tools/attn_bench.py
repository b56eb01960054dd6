"""Prefill attention alone (ws_attn_prefill) on the paged pool: a parity
harness against a torch fp32 causal GQA reference, and a timing loop.

    python tools/attn_bench.py [--shape llama3-8b] [--rows 2048] [--pos0 0] [--iters 50] [--impl 0]

K/V are written straight into the sequence's pool pages (layout
[layer][k|v][kv_head][tpb][head_dim] per page, ws_model_kv_geometry), q is
random; no RoPE / projections involved. Prints µs per launch and TFLOP/s
(algorithmic causal FLOPs: 4 * hd * H * sum over queries of visible keys).
"""

from __future__ import annotations

import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SHAPES = {  # name: hidden, heads, kv_heads, head_dim, layers (sets tokens per KV block)
    "llama3-8b": (4096, 32, 8, 128, 32),       # 16 tokens per 2 MiB block
    "qwen2.5-7b": (3584, 28, 4, 128, 28),      # 36
    "phi3-mini": (3072, 32, 32, 96, 32),       # 5
    "tiny": (256, 4, 2, 64, 2),                # 4096
    "llama3-70b-tp8": (1024, 8, 1, 128, 80),   # 51 (not a multiple of 16: cp.async gather)
}


class AttnRig:
    """A 1-layer model of the given attention shape on a worker whose KV pool
    holds one sequence of `n_keys` tokens filled with seeded random K/V."""

    def __init__(self, shape: str, n_keys: int, seed: int = 0, device: int = 0):
        import torch

        from paper_2512_09472_b200 import _native as N
        from paper_2512_09472_b200 import models as M
        from paper_2512_09472_b200.devmem import view
        from paper_2512_09472_b200.worker import UniversalWorker

        d, H, KV, hd, layers = SHAPES[shape]
        self.H, self.KV, self.hd = H, KV, hd
        cfg = M.TINY.with_(name=f"attn-{shape}", hidden=d, heads=H, kv_heads=KV, head_dim=hd, ffn=256, layers=layers,
                           vocab=256, max_positions=max(8192, n_keys + 8))
        self.cfg = cfg
        tpb, _ = cfg.kv_geometry()
        pages = (n_keys + tpb - 1) // tpb + 8 + cfg.layout().total // M.PAGE + 2
        self.w = w = UniversalWorker(device, pool_pages=pages, max_tokens=max(n_keys, 256))
        w.register(cfg, None)
        w.prewarm(cfg.name, layers=0)  # slot pages only: attention reads no weights
        w.switch_memory(cfg.name)
        self.seq = w.open_seq(n_keys)
        nb = (n_keys + tpb - 1) // tpb
        ids = (C.c_int32 * nb)()
        n = C.c_int32()
        N.call("ws_seq_blocks", w.gpu.pool, self.seq, ids, nb, C.byref(n))
        base = C.c_void_p()
        N.call("ws_pool_window", w.gpu.pool, C.byref(base))
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.K = torch.randn(KV, n_keys, hd, generator=g).bfloat16()
        self.V = torch.randn(KV, n_keys, hd, generator=g).bfloat16()
        page_elems = M.PAGE // 2
        for b in range(n.value):
            pg = view(base.value + ids[b] * M.PAGE, (page_elems,), torch.bfloat16, device)
            lo, hi = b * tpb, min(n_keys, (b + 1) * tpb)
            planes = pg[: 2 * KV * tpb * hd].view(2, KV, tpb, hd)  # layer 0 (the first planes of the page)
            planes[0, :, : hi - lo] = self.K[:, lo:hi].to(pg.device)
            planes[1, :, : hi - lo] = self.V[:, lo:hi].to(pg.device)
        torch.cuda.synchronize()
        self.n_keys = n_keys

    def run(self, q, rows, pos0, impl=0, stream=None):
        """q: bf16 [rows, H*hd] on the device -> out bf16 [rows, H*hd]."""
        import torch

        from paper_2512_09472_b200 import _native as N

        qkv = torch.zeros(rows, (self.H + 2 * self.KV) * self.hd, dtype=torch.bfloat16, device=q.device)
        qkv[:, : self.H * self.hd] = q
        out = torch.empty(rows, self.H * self.hd, dtype=torch.bfloat16, device=q.device)
        self.launch(qkv, out, rows, pos0, impl, stream)
        return out

    def launch(self, qkv, out, rows, pos0, impl=0, stream=None):
        import torch

        from paper_2512_09472_b200 import _native as N

        st = stream if stream is not None else torch.cuda.current_stream()
        N.call("ws_attn_prefill", self.w.models[self.cfg.name].handle, self.w.gpu.pool, 0, self.seq,
               C.c_void_p(qkv.data_ptr()), rows, pos0, C.c_void_p(out.data_ptr()), impl, C.c_void_p(st.cuda_stream))

    def reference(self, q, rows, pos0):
        """fp32 causal GQA attention of queries pos0..pos0+rows-1 (CPU)."""
        import torch

        H, KV, hd = self.H, self.KV, self.hd
        qf = q.float().cpu().view(rows, H, hd).transpose(0, 1)  # [H, rows, hd]
        n = pos0 + rows
        k = self.K[:, :n].float().repeat_interleave(H // KV, 0)
        v = self.V[:, :n].float().repeat_interleave(H // KV, 0)
        s = qf @ k.transpose(1, 2) / hd**0.5
        qpos = torch.arange(pos0, pos0 + rows)[:, None]
        s = s.masked_fill(torch.arange(n)[None, :] > qpos, float("-inf"))
        return (s.softmax(-1) @ v).transpose(0, 1).reshape(rows, H * hd)

    def flops(self, rows, pos0):
        vis = sum(pos0 + i + 1 for i in range(rows))
        return 4.0 * self.hd * self.H * vis

    def close(self):
        self.w.close()


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama3-8b")
    ap.add_argument("--rows", type=int, default=2048)
    ap.add_argument("--pos0", type=int, default=0)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--impl", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    rig = AttnRig(a.shape, a.pos0 + a.rows)
    q = torch.randn(a.rows, rig.H * rig.hd, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    qkv = torch.zeros(a.rows, (rig.H + 2 * rig.KV) * rig.hd, dtype=torch.bfloat16, device="cuda")
    qkv[:, : rig.H * rig.hd] = q
    out = torch.empty(a.rows, rig.H * rig.hd, dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        rig.launch(qkv, out, a.rows, a.pos0, a.impl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        rig.launch(qkv, out, a.rows, a.pos0, a.impl)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / a.iters * 1e3
    tf = rig.flops(a.rows, a.pos0) / (us * 1e-6) / 1e12
    line = f"{a.shape} rows {a.rows} pos0 {a.pos0} impl {a.impl}: {us:.1f} us/launch, {tf:.0f} TFLOP/s"
    if a.check:
        ref = rig.reference(q, a.rows, a.pos0)
        rel = ((out.float().cpu() - ref).norm() / ref.norm()).item()
        line += f", rel err {rel:.2e}"
    print(line, flush=True)
    rig.close()


if __name__ == "__main__":
    main()

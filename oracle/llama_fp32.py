"""TEST INFRASTRUCTURE ONLY — CPU fp32 logits oracle for the worker's forward.

The reference has no model forward (logits are "parity
unpinned" with respect to the reference). This oracle restates a
Llama-family decoder in fp32 on the CPU — RMSNorm, rotate_half RoPE, causal
GQA attention, SwiGLU — reading the SAME bf16 weight bytes the GPU uses,
upcast to fp32, laid out by ``ws_model_layout``. It is pinned against
HF ``transformers`` LlamaForCausalLM in tests/test_oracle_llama.py.

The RoPE angle for pair i at position p is p * theta**(-2i/head_dim) in
float64, rounded to fp32 cos/sin (the same table the device uses).
"""

from __future__ import annotations

import math

import numpy as np
import torch


def rope_table(head_dim: int, theta: float, n_pos: int) -> tuple[torch.Tensor, torch.Tensor]:
    half = head_dim // 2
    inv = np.array([float(theta) ** (-2.0 * i / head_dim) for i in range(half)], dtype=np.float64)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def unpack(cfg, layout, flat_bf16: torch.Tensor) -> dict:
    """Slice the flat bf16 weight image into fp32 tensors by name."""
    out = {}
    for name, off, shape in layout.tensors():
        n = int(np.prod(shape))
        out[name] = flat_bf16[off // 2: off // 2 + n].view(*shape).float()
    return out


def split_gate_up(wgu: torch.Tensor, ffn: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Wgu stores gate and up rows interleaved in 128-row blocks
    ([gate 0:128][up 0:128][gate 128:256]...), so a 256-wide GEMM tile holds
    matching gate/up columns (SwiGLU fused in the epilogue)."""
    blocks = wgu.view(ffn // 128, 2, 128, -1)
    return blocks[:, 0].reshape(ffn, -1), blocks[:, 1].reshape(ffn, -1)


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    # x: [S, heads, hd]; rotate_half pairs (i, i + hd/2)
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1)


def forward_tp(cfg_shard, w: dict, tokens, allreduce, allgather):
    """Tensor-parallel restatement for one rank: local heads / ffn slice /
    vocab slice; ``allreduce(t)`` sums a tensor over ranks in place,
    ``allgather(t)`` returns the rank tensors concatenated on the last dim.
    Mathematically equal to ``forward`` of the full model (Megatron split)."""
    tokens = torch.as_tensor(tokens, dtype=torch.long)
    S = tokens.numel()
    H, KV, hd = cfg_shard.heads, cfg_shard.kv_heads, cfg_shard.head_dim
    cos, sin = rope_table(hd, cfg_shard.rope_theta, S)
    x = w["embed"][tokens]
    for l in range(cfg_shard.layers):
        h = _rms(x, w[f"l{l}.attn_norm"], cfg_shard.rms_eps)
        qkv = h @ w[f"l{l}.wqkv"].T
        if f"l{l}.bqkv" in w:
            qkv = qkv + w[f"l{l}.bqkv"]
        q = _rope(qkv[:, : H * hd].view(S, H, hd), cos, sin)
        k = _rope(qkv[:, H * hd: (H + KV) * hd].view(S, KV, hd), cos, sin)
        v = qkv[:, (H + KV) * hd:].view(S, KV, hd)
        g = H // KV
        sc = torch.einsum("shd,thd->hst", q, k.repeat_interleave(g, 1)) / math.sqrt(hd)
        sc = sc.masked_fill(torch.ones(S, S, dtype=torch.bool).triu(1)[None], float("-inf"))
        o = torch.einsum("hst,thd->shd", torch.softmax(sc, -1), v.repeat_interleave(g, 1)).reshape(S, H * hd)
        part = o @ w[f"l{l}.wo"].T
        allreduce(part)
        x = x + part
        h = _rms(x, w[f"l{l}.ffn_norm"], cfg_shard.rms_eps)
        wg, wu = split_gate_up(w[f"l{l}.wgu"], cfg_shard.ffn)
        part = (torch.nn.functional.silu(h @ wg.T) * (h @ wu.T)) @ w[f"l{l}.wdown"].T
        allreduce(part)
        x = x + part
    h = _rms(x, w["final_norm"], cfg_shard.rms_eps)
    return allgather(h @ w["lm_head"].T)


def forward(cfg, w: dict, tokens, pos0: int = 0, past: list | None = None):
    """Logits [S, vocab] for tokens at positions pos0.. with optional past
    K/V (list per layer of (k [P, kvh, hd], v)). Returns (logits, new_past)."""
    tokens = torch.as_tensor(tokens, dtype=torch.long)
    S = tokens.numel()
    H, KV, hd = cfg.heads, cfg.kv_heads, cfg.head_dim
    cos, sin = rope_table(hd, cfg.rope_theta, pos0 + S)
    cos, sin = cos[pos0:], sin[pos0:]
    x = w["embed"][tokens]
    new_past = []
    for l in range(cfg.layers):
        h = _rms(x, w[f"l{l}.attn_norm"], cfg.rms_eps)
        qkv = h @ w[f"l{l}.wqkv"].T
        if f"l{l}.bqkv" in w:
            qkv = qkv + w[f"l{l}.bqkv"]
        q = qkv[:, : H * hd].view(S, H, hd)
        k = qkv[:, H * hd: (H + KV) * hd].view(S, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(S, KV, hd)
        q, k = _rope(q, cos, sin), _rope(k, cos, sin)
        if past is not None:
            k = torch.cat([past[l][0], k], 0)
            v = torch.cat([past[l][1], v], 0)
        new_past.append((k, v))
        T = k.shape[0]
        g = H // KV
        kk = k.repeat_interleave(g, dim=1)  # [T, H, hd]
        vv = v.repeat_interleave(g, dim=1)
        sc = torch.einsum("shd,thd->hst", q, kk) / math.sqrt(hd)
        qpos = torch.arange(pos0, pos0 + S)[:, None]
        kpos = torch.arange(T)[None, :]
        sc = sc.masked_fill((kpos > qpos)[None], float("-inf"))
        p = torch.softmax(sc, dim=-1)
        o = torch.einsum("hst,thd->shd", p, vv).reshape(S, H * hd)
        x = x + o @ w[f"l{l}.wo"].T
        h = _rms(x, w[f"l{l}.ffn_norm"], cfg.rms_eps)
        wg, wu = split_gate_up(w[f"l{l}.wgu"], cfg.ffn)
        x = x + (torch.nn.functional.silu(h @ wg.T) * (h @ wu.T)) @ w[f"l{l}.wdown"].T
    h = _rms(x, w["final_norm"], cfg.rms_eps)
    return h @ w["lm_head"].T, new_past


def forward_streamed(cfg, layout, flat_bf16: torch.Tensor, tokens, heads_per_chunk: int = 8,
                     emulate_bf16: bool = False) -> torch.Tensor:
    """Last-row logits [vocab] of ``forward`` without materialising the whole
    fp32 model: each tensor is upcast from the bf16 image when its layer runs
    (a full-size Llama-3-8B needs ~1 GB of fp32 weights at a time instead of
    32 GB). Same math, same order of operations as ``forward`` with pos0 = 0;
    attention runs ``heads_per_chunk`` heads at a time to bound the S x S
    score buffers.

    ``emulate_bf16=True`` is the *bf16 floor*: the same fp32 math with every
    tensor a bf16 kernel path must hold in bf16 rounded to bf16 — the
    normalised activations fed to the QKV and gate/up GEMMs, q/k/v after
    RoPE (the KV cache), the unnormalised softmax numerators exp(s - max)
    fed to the PV product (normalised in fp32 afterwards), the attention
    output fed to O, the SwiGLU output fed to down, and the final normalised
    row fed to the lm_head; the residual stream and every accumulation stay
    fp32. Any bf16 implementation carries at least this rounding; its
    distance to the fp32 logits is the accuracy a bf16 forward can reach on
    these weights."""
    tokens = torch.as_tensor(tokens, dtype=torch.long)
    S = tokens.numel()
    H, KV, hd, d = cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.hidden
    cos, sin = rope_table(hd, cfg.rope_theta, S)
    R = (lambda v: v.bfloat16().float()) if emulate_bf16 else (lambda v: v)

    def t(off, *shape):
        n = int(np.prod(shape))
        return flat_bf16[off // 2: off // 2 + n].view(*shape).float()

    x = flat_bf16[layout.embed // 2: layout.embed // 2 + cfg.vocab * d].view(cfg.vocab, d)[tokens].float()
    causal = torch.ones(S, S, dtype=torch.bool).triu(1)[None]
    for L in layout.layers:
        h = R(_rms(x, t(L["attn_norm"], d), cfg.rms_eps))
        qkv = h @ t(L["wqkv"], cfg.qkv_dim, d).T
        if L["bqkv"] >= 0:
            qkv = qkv + t(L["bqkv"], cfg.qkv_dim)
        q = R(_rope(qkv[:, : H * hd].view(S, H, hd), cos, sin))
        k = R(_rope(qkv[:, H * hd: (H + KV) * hd].view(S, KV, hd), cos, sin))
        v = R(qkv[:, (H + KV) * hd:].view(S, KV, hd))
        g = H // KV
        o = torch.empty(S, H, hd)
        for h0 in range(0, H, heads_per_chunk):
            h1 = min(H, h0 + heads_per_chunk)
            kk = k[:, torch.arange(h0, h1) // g]
            vv = v[:, torch.arange(h0, h1) // g]
            sc = torch.einsum("shd,thd->hst", q[:, h0:h1], kk) / math.sqrt(hd)
            sc = sc.masked_fill(causal, float("-inf"))
            if emulate_bf16:
                e = torch.exp(sc - sc.amax(-1, keepdim=True))
                o[:, h0:h1] = (torch.einsum("hst,thd->hsd", R(e), vv) / e.sum(-1, keepdim=True)).transpose(0, 1)
            else:
                o[:, h0:h1] = torch.einsum("hst,thd->shd", torch.softmax(sc, dim=-1), vv)
        x = x + R(o.reshape(S, H * hd)) @ t(L["wo"], d, H * hd).T
        h = R(_rms(x, t(L["ffn_norm"], d), cfg.rms_eps))
        wg, wu = split_gate_up(t(L["wgu"], 2 * cfg.ffn, d), cfg.ffn)
        x = x + R(torch.nn.functional.silu(h @ wg.T) * (h @ wu.T)) @ t(L["wdown"], d, cfg.ffn).T
    h = R(_rms(x[-1:], t(layout.final_norm, d), cfg.rms_eps))
    rows = cfg.lm_head_rows or cfg.vocab
    out = torch.empty(rows)
    step = 16384
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        out[r0:r1] = (h @ t(layout.lm_head + r0 * d * 2, r1 - r0, d).T)[0]
    return out

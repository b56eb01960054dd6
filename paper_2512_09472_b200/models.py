"""Model shapes of the BASELINE configs and the in-slot weight layout.

Shapes are the public HF configs. The byte layout of a
model inside its prewarm slot comes from the native ``ws_model_layout`` (single
source of truth for kernels, loader and oracle): embedding, then each decoder
layer contiguously, then final norm and lm_head — so a prewarmed prefix is
``[0, layer_begin(k))`` and the streamed remainder is one suffix range.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

from . import _native as N

PAGE = 2 * 1024 * 1024


class ModelConfigC(C.Structure):
    _fields_ = [
        ("layers", C.c_int32), ("hidden", C.c_int32), ("ffn", C.c_int32), ("heads", C.c_int32),
        ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("vocab", C.c_int32),
        ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("qkv_bias", C.c_int32),
        ("max_positions", C.c_int32), ("lm_head_rows", C.c_int32),
    ]


N.register({
    "ws_model_layout": [C.POINTER(ModelConfigC), C.POINTER(C.c_int64), C.c_int64],
    "ws_model_kv_geometry": [C.POINTER(ModelConfigC), C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int64)],
    "ws_model_create": [C.POINTER(ModelConfigC), C.c_int32, C.POINTER(C.c_void_p)],
    "ws_model_destroy": [C.c_void_p],
    "ws_model_workspace_bytes": [C.c_void_p, C.c_int32, C.POINTER(C.c_int64)],
    "ws_model_set_gemm": [C.c_void_p, C.c_int32],
    "ws_model_set_prune_last": [C.c_void_p, C.c_int32],
    "ws_model_set_tp_dtype": [C.c_void_p, C.c_int32],
    "ws_model_prefill": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                         C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "ws_model_decode": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                        C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "ws_gemm": [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                C.c_void_p, C.c_int32, C.c_void_p],
    "ws_attn_prefill": [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                        C.c_void_p, C.c_int32, C.c_void_p],
    "ws_nccl_unique_id": [C.POINTER(C.c_uint8), C.c_int32],
    "ws_comm_create": [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)],
    "ws_comm_destroy": [C.c_void_p],
    "ws_model_set_comm": [C.c_void_p, C.c_void_p],
})


@dataclass(frozen=True)
class ModelConfig:
    name: str
    layers: int
    hidden: int
    ffn: int
    heads: int
    kv_heads: int
    head_dim: int
    vocab: int
    rope_theta: float = 500_000.0
    rms_eps: float = 1e-5
    qkv_bias: bool = False
    max_positions: int = 8192
    lm_head_rows: int = 0  # vocab-parallel lm_head shard (TP rank); 0 = full vocab

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.layers, self.hidden, self.ffn, self.heads, self.kv_heads, self.head_dim,
                            self.vocab, self.rope_theta, self.rms_eps, int(self.qkv_bias), self.max_positions,
                            self.lm_head_rows)

    @property
    def qkv_dim(self) -> int:
        return (self.heads + 2 * self.kv_heads) * self.head_dim

    def layout(self) -> "Layout":
        n = 4 + 9 * self.layers
        buf = (C.c_int64 * n)()
        N.call("ws_model_layout", C.byref(self.c()), buf, n)
        return Layout(self, list(buf))

    def kv_geometry(self, page_size: int = PAGE) -> tuple[int, int]:
        tpb, per_tok = C.c_int32(), C.c_int64()
        N.call("ws_model_kv_geometry", C.byref(self.c()), page_size, C.byref(tpb), C.byref(per_tok))
        return tpb.value, per_tok.value

    def prefill_flops(self, tokens: int) -> float:
        """Algorithmic prefill FLOPs: 2 * params_in_layers * S
        + causal attention 2*S^2*H*hd per layer (QK^T and PV, half masked),
        + the last-row logits 2*V*d."""
        d, o = self.hidden, self.heads * self.head_dim
        per_layer = self.qkv_dim * d + d * o + 2 * self.ffn * d + d * self.ffn
        dense = 2.0 * per_layer * self.layers * tokens
        attn = 2.0 * tokens * tokens * o * self.layers  # 4*S^2*o/2 (causal)
        return dense + attn + 2.0 * self.vocab * d

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


class Layout:
    """Byte offsets of every tensor inside the slot (see include/warmserve.h)."""

    def __init__(self, cfg: ModelConfig, flat: list[int]):
        self.cfg = cfg
        self.embed, self.final_norm, self.lm_head, self.total = flat[:4]
        self.layers = [dict(zip(("begin", "attn_norm", "wqkv", "bqkv", "wo", "ffn_norm", "wgu", "wdown", "end"),
                                flat[4 + 9 * l: 13 + 9 * l])) for l in range(cfg.layers)]

    def tensors(self):
        """(name, offset, shape) of every weight tensor, in layout order."""
        c = self.cfg
        d, o = c.hidden, c.heads * c.head_dim
        out = [("embed", self.embed, (c.vocab, d))]
        for i, L in enumerate(self.layers):
            out.append((f"l{i}.attn_norm", L["attn_norm"], (d,)))
            out.append((f"l{i}.wqkv", L["wqkv"], (c.qkv_dim, d)))
            if L["bqkv"] >= 0:
                out.append((f"l{i}.bqkv", L["bqkv"], (c.qkv_dim,)))
            out.append((f"l{i}.wo", L["wo"], (d, o)))
            out.append((f"l{i}.ffn_norm", L["ffn_norm"], (d,)))
            out.append((f"l{i}.wgu", L["wgu"], (2 * c.ffn, d)))
            out.append((f"l{i}.wdown", L["wdown"], (d, c.ffn)))
        out.append(("final_norm", self.final_norm, (d,)))
        out.append(("lm_head", self.lm_head, (c.lm_head_rows or c.vocab, d)))
        return out

    def prefix_bytes(self, k: int) -> int:
        """Bytes of embedding + layers [0, k)."""
        return self.layers[k]["begin"] if k < len(self.layers) else self.final_norm

    def stream_ranges(self, k: int) -> list[tuple[int, int, int]]:
        """(dst, src, bytes) per streamed unit: layers k..L-1, then final
        norm + lm_head as one tail range (offsets identical in slot and source)."""
        out = [(L["begin"], L["begin"], L["end"] - L["begin"]) for L in self.layers[k:]]
        out.append((self.final_norm, self.final_norm, self.total - self.final_norm))
        return out


# BASELINE.json configs (SURVEY.md §8 shapes).
TINY = ModelConfig("tiny", 2, 256, 768, 4, 2, 64, 4096)
LLAMA3_8B = ModelConfig("llama3-8b", 32, 4096, 14336, 32, 8, 128, 128256)
QWEN25_7B = ModelConfig("qwen2.5-7b", 28, 3584, 18944, 28, 4, 128, 152064, rope_theta=1_000_000.0,
                        rms_eps=1e-6, qkv_bias=True)
MISTRAL_7B = ModelConfig("mistral-7b", 32, 4096, 14336, 32, 8, 128, 32000, rope_theta=1_000_000.0)
PHI3_MINI = ModelConfig("phi3-mini", 32, 3072, 8192, 32, 32, 96, 32064, rope_theta=10_000.0)
LLAMA3_70B = ModelConfig("llama3-70b", 80, 8192, 28672, 64, 8, 128, 128256)

ALL = {m.name: m for m in (TINY, LLAMA3_8B, QWEN25_7B, MISTRAL_7B, PHI3_MINI, LLAMA3_70B)}


def model_spec(cfg: ModelConfig, parallelism: int = 1, max_batch: int = 32, **kw):
    """Reference ModelSpec (cluster.py:52-94) for this model: weight_bytes is
    the exact slot layout size, kv_bytes_per_token the paged-KV footprint."""
    from .cluster import ModelSpec

    _, per_tok = cfg.kv_geometry()
    return ModelSpec(cfg.name, cfg.layout().total, parallelism, max_batch=max_batch, layers=cfg.layers,
                     kv_bytes_per_token=per_tok, **kw)

"""Tensor parallelism for the large-model config (BASELINE config 4,
Llama-3-70B at TP 2/4/8).

Megatron-style sharding of one model's weight image into TP rank shards, the
layout a rank's prewarm slot holds:

  Wqkv   column-parallel: the rank's q heads, k heads and v heads (rows)
  Wo     row-parallel:    the matching input columns   -> allreduce after
  Wgu    column-parallel: the rank's ffn slice (the 128-row gate/up blocks
                          of that slice are contiguous in the interleaved layout)
  Wdown  row-parallel:    the matching input columns   -> allreduce after
  lm_head vocab-parallel: vocab/TP rows                -> allgather
  embedding and norms:    replicated

The reference only models TP as a ceil-divided weight partition on one server
(cluster.py:58, 79-80, 305-306) plus a constant sync cost (engine.py:110-113).
Here a rank's physical shard is ``Layout(shard_config).total`` bytes and the
rank's ``ModelSpec.weight_bytes`` is TP x that, so the reference's
``partition_bytes`` equals the physical shard exactly.

Communicator: ``TpGroup`` wraps the native NCCL communicator (created once at
prewarm time — the paper's pre-established group); the
unique id is exchanged with ``torch.distributed`` (plumbing only).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .models import ModelConfig


def shard_config(cfg: ModelConfig, tp: int) -> ModelConfig:
    """The per-rank model config: heads/TP, kv_heads/TP, ffn/TP, vocab/TP
    lm_head rows (every divisibility the shapes need is checked)."""
    if tp == 1:
        return cfg
    for name, v, unit in (("heads", cfg.heads, 1), ("kv_heads", cfg.kv_heads, 1), ("ffn", cfg.ffn, 128),
                          ("vocab", cfg.vocab, 1)):
        if v % (tp * unit):
            raise ValueError(f"{cfg.name}: {name}={v} not divisible by TP={tp} (x{unit})")
    return cfg.with_(name=f"{cfg.name}-tp{tp}", heads=cfg.heads // tp, kv_heads=cfg.kv_heads // tp,
                     ffn=cfg.ffn // tp, lm_head_rows=cfg.vocab // tp)


def _views(cfg: ModelConfig, flat: torch.Tensor) -> dict:
    out = {}
    for name, off, shape in cfg.layout().tensors():
        n = 1
        for s in shape:
            n *= s
        out[name] = flat[off // 2: off // 2 + n].view(*shape)
    return out


def shard_tensor(cfg: ModelConfig, name: str, full: torch.Tensor, tp: int, rank: int) -> torch.Tensor:
    """Rank ``rank``'s slice of full tensor ``name`` (layout.tensors() naming)."""
    hd = cfg.head_dim
    hr, kr = cfg.heads // tp, cfg.kv_heads // tp
    fr = cfg.ffn // tp
    base = name.split(".")[-1]
    if base in ("attn_norm", "ffn_norm") or name in ("embed", "final_norm"):
        return full
    if base in ("wqkv", "bqkv"):
        q = full[rank * hr * hd:(rank + 1) * hr * hd]
        k0 = cfg.heads * hd
        k = full[k0 + rank * kr * hd:k0 + (rank + 1) * kr * hd]
        v0 = (cfg.heads + cfg.kv_heads) * hd
        v = full[v0 + rank * kr * hd:v0 + (rank + 1) * kr * hd]
        return torch.cat([q, k, v], 0)
    if base == "wo":
        return full[:, rank * hr * hd:(rank + 1) * hr * hd]
    if base == "wgu":  # interleaved 128-row gate/up blocks: the rank's blocks are contiguous
        return full[2 * rank * fr:2 * (rank + 1) * fr]
    if base == "wdown":
        return full[:, rank * fr:(rank + 1) * fr]
    if name == "lm_head":
        v = cfg.vocab // tp
        return full[rank * v:(rank + 1) * v]
    raise KeyError(name)


def shard_flat(cfg: ModelConfig, full_flat: torch.Tensor, tp: int, rank: int) -> torch.Tensor:
    """Rank shard image (bf16 flat in the shard layout) of a full image."""
    scfg = shard_config(cfg, tp)
    out = torch.zeros(scfg.layout().total // 2, dtype=full_flat.dtype, device=full_flat.device)
    src, dst = _views(cfg, full_flat), _views(scfg, out)
    for name, t in dst.items():
        t.copy_(shard_tensor(cfg, name, src[name], tp, rank))
    return out


def synth_shard(cfg: ModelConfig, tp: int, rank: int, seed: int = 0, device="cuda") -> torch.Tensor:
    """Rank shard of ``weights.synth_flat(cfg, seed)`` without materialising
    the full image (one full tensor at a time: 70B fits a rank)."""
    from .weights import _fill_tensor

    scfg = shard_config(cfg, tp)
    out = torch.zeros(scfg.layout().total // 2, dtype=torch.bfloat16, device=device)
    dst = _views(scfg, out)
    for idx, (name, off, shape) in enumerate(cfg.layout().tensors()):
        full = torch.empty(shape, dtype=torch.bfloat16, device=device)
        _fill_tensor(full.view(-1), name, idx, seed)
        dst[name].copy_(shard_tensor(cfg, name, full, tp, rank))
        del full
    return out


class TpGroup:
    """Native NCCL communicator for one TP group (one rank per GPU)."""

    def __init__(self, rank: int, size: int, device: int, unique_id: bytes):
        self.rank, self.size, self.device = rank, size, device
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        N.call("ws_comm_create", buf, rank, size, device, C.byref(h))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        N.call("ws_nccl_unique_id", buf, 128)
        return bytes(buf)

    @classmethod
    def from_torch_dist(cls, device: int) -> "TpGroup":
        """Rank 0 makes the NCCL id; torch.distributed broadcasts it."""
        import torch.distributed as dist

        obj = [cls.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(dist.get_rank(), dist.get_world_size(), device, obj[0])

    @classmethod
    def peer_only(cls, device: int, max_count: int, group=None) -> "TpGroup":
        """A TP group whose allreduces and allgathers all run on the
        peer-memory kernels (csrc/peer.cu) — no NCCL communicator. Collectives
        above max_count floats fail."""
        import torch.distributed as dist

        from .peer import PeerAllreduce

        self = cls.__new__(cls)
        self.rank, self.size, self.device = dist.get_rank(group), dist.get_world_size(group), device
        self.peer = PeerAllreduce(max_count, group)
        h = C.c_void_p()
        N.call("ws_comm_create_peer", self.rank, self.size, device, self.peer._h, self.peer.max_count, C.byref(h))
        self.handle = h
        return self

    def attach_peer(self, max_count: int, group=None) -> None:
        """Route the row-parallel allreduces (<= max_count floats) through the
        peer-memory allreduce (csrc/peer.cu) instead of NCCL."""
        from .peer import PeerAllreduce

        self.peer = PeerAllreduce(max_count, group)
        N.call("ws_comm_set_peer", self.handle, self.peer._h, self.peer.max_count)

    def close(self):
        if getattr(self, "peer", None) is not None:
            N.call("ws_comm_set_peer", self.handle, None, 0)
            self.peer.close()
            self.peer = None
        if self.handle:
            N.fns["ws_comm_destroy"](self.handle)
            self.handle = None

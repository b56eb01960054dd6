"""Seeded synthetic weights in the slot layout (no checkpoints are reachable).

Linear/embedding weights ~ N(0, 0.02), norm gains ~ N(1, 0.1), biases ~
N(0, 0.02); each tensor has its own seed (seed, tensor index) so any prefix
or suffix can be regenerated independently. Generated on the GPU (Philox) in
fp32 and rounded to bf16; the CPU oracle upcasts the same bf16 bytes.
"""

from __future__ import annotations

import torch

from .models import ModelConfig


def fill_flat(cfg: ModelConfig, out: torch.Tensor, seed: int = 0) -> torch.Tensor:
    """Fill a flat bf16 tensor of layout.total/2 elements (any device)."""
    layout = cfg.layout()
    assert out.dtype == torch.bfloat16 and out.numel() * 2 >= layout.total
    for idx, (name, off, shape) in enumerate(layout.tensors()):
        n = 1
        for s in shape:
            n *= s
        _fill_tensor(out[off // 2: off // 2 + n], name, idx, seed)
    return out


def _fill_tensor(dst: torch.Tensor, name: str, idx: int, seed: int) -> None:
    """Fill one flat bf16 tensor (index ``idx`` in layout order) from its own seed."""
    gen = torch.Generator(device=dst.device)
    gen.manual_seed(seed * 1_000_003 + idx)
    is_norm = name.endswith("norm")
    chunk = 1 << 26
    n = dst.numel()
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        v = torch.randn(m, generator=gen, device=dst.device, dtype=torch.float32)
        if is_norm:
            v.mul_(0.1).add_(1.0)
        else:
            v.mul_(0.02)
        dst[i:i + m].copy_(v)


def synth_flat(cfg: ModelConfig, seed: int = 0, device: str | torch.device = "cuda") -> torch.Tensor:
    layout = cfg.layout()
    out = torch.zeros(layout.total // 2, dtype=torch.bfloat16, device=device)
    return fill_flat(cfg, out, seed)


def pinned_host_copy(flat_dev: torch.Tensor) -> torch.Tensor:
    """Pinned host image of the weights: the cold-start source (PCIe DMA)."""
    host = torch.empty(flat_dev.numel(), dtype=flat_dev.dtype, pin_memory=True)
    host.copy_(flat_dev)
    return host

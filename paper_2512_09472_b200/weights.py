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


# ---------------------------------------------------------------- packed stream
def _align(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def packed_sections(n: int, n_esc: int) -> tuple[int, int, int, int]:
    """(codes, idx, exp, total) byte offsets of a packed range — the layout
    ws::packed_sections uses (csrc/kernels/unpack.cu)."""
    codes = _align(n, 16)
    idx = _align(codes + (n + 1) // 2, 16)
    exp = _align(idx + 4 * n_esc, 16)
    return codes, idx, exp, _align(exp + n_esc, 16)


class PackedImage:
    """Losslessly packed host image of a model's streamable ranges (every
    decoder layer, then final norm + lm_head), for the packed cold-start
    stream (ws_streamer_start_packed). Per bf16 weight: one byte of
    sign|mantissa plus a 4-bit exponent code relative to the range's densest
    15-exponent window; values outside it are escapes (position + exponent).
    Random-init and trained bf16 weights both sit in a few exponents, so a
    range packs to ~12 bits per weight: ~25% fewer bytes over PCIe."""

    def __init__(self, blob: torch.Tensor, desc: list[list[int]], ranges: list[tuple[int, int, int]]):
        self.blob = blob      # pinned uint8
        self.desc = desc      # per range: [dst_off, packed_off, n_values, e_base, n_escapes, packed_bytes]
        self.ranges = ranges  # layout.stream_ranges(0): layers 0..L-1, then the tail

    def rows(self, first_layer: int) -> list[list[int]]:
        """desc rows streamed when layers [0, first_layer) are resident."""
        return self.desc[first_layer:]

    @property
    def max_range_bytes(self) -> int:
        return max(d[5] for d in self.desc)


def pack_range(v: torch.Tensor) -> tuple[torch.Tensor, int, int]:
    """Pack one range of bf16 values (1-D tensor, any device): returns the
    packed bytes (same device), the exponent base and the escape count."""
    u = v.view(torch.int16).to(torch.int32) & 0xFFFF
    n = u.numel()
    e = (u >> 7) & 0xFF
    hist = torch.bincount(e, minlength=256).cpu()
    cs = torch.cat([torch.zeros(1, dtype=hist.dtype), hist.cumsum(0)])
    base = int(torch.argmax(cs[15:256] - cs[0:241]))  # window [base, base + 15), base <= 240
    code = e - base
    esc = (code < 0) | (code > 14)
    code = code.masked_fill(esc, 15)
    lo = (((u >> 8) & 0x80) | (u & 0x7F)).to(torch.uint8)
    if n % 2:
        code = torch.cat([code, code.new_zeros(1)])
    codes = (code[0::2] | (code[1::2] << 4)).to(torch.uint8)
    idx = esc.nonzero().flatten().to(torch.int32)
    exps = e[idx.long()].to(torch.uint8)
    n_esc = idx.numel()
    c_off, i_off, e_off, total = packed_sections(n, n_esc)
    out = torch.zeros(total, dtype=torch.uint8, device=v.device)
    out[:n] = lo
    out[c_off:c_off + codes.numel()] = codes
    out[i_off:i_off + 4 * n_esc] = idx.view(torch.uint8)
    out[e_off:e_off + n_esc] = exps
    return out, base, n_esc


def pack_stream(cfg: ModelConfig, flat: torch.Tensor) -> PackedImage:
    """PackedImage of every streamable range of ``flat`` (the bf16 slot image;
    packing runs where ``flat`` lives — on the GPU it takes seconds)."""
    ranges = cfg.layout().stream_ranges(0)
    parts, desc, off = [], [], 0
    for dst, src, nbytes in ranges:
        blob, base, n_esc = pack_range(flat[src // 2: (src + nbytes) // 2])
        desc.append([dst, off, nbytes // 2, base, n_esc, blob.numel()])
        parts.append(blob)
        off += _align(blob.numel(), 256)
    host = torch.empty(off, dtype=torch.uint8, pin_memory=True)
    for d, p in zip(desc, parts):
        host[d[1]:d[1] + p.numel()].copy_(p)
    return PackedImage(host, desc, ranges)

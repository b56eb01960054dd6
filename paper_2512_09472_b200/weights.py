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
    sign|mantissa plus the exponent, either as a canonical Huffman code
    (format 1, default: ~10.6 bits per weight, 34% fewer PCIe bytes) or as a
    4-bit code relative to the range's densest 15-exponent window with
    escapes (format 0: ~12 bits). Random-init and trained bf16 weights both
    sit in a few exponents (~2.6 bits of exponent entropy)."""

    def __init__(self, blob: torch.Tensor, desc: list[list[int]], ranges: list[tuple[int, int, int]]):
        self.blob = blob      # pinned uint8
        self.desc = desc      # per range: [dst_off, packed_off, n_values, e_base (-1: Huffman), n_escapes, packed_bytes]
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


HUFF_BLOCK, HUFF_BITS = 1024, 12  # csrc/kernels/unpack.cu kHuffBlock / kHuffBits


def huff_sections(n: int) -> tuple[int, int, int]:
    """(lut, block offsets, words) byte offsets of a Huffman-packed range."""
    lut = _align(n, 16)
    offs = lut + 2 * (1 << HUFF_BITS)
    return lut, offs, _align(offs + 4 * (-(-n // HUFF_BLOCK)), 16)


def huff_lengths(hist, lmax: int = HUFF_BITS) -> list[int]:
    """Code length per symbol (0 = unused) of a Huffman code limited to
    ``lmax`` bits: rebuild with flattened frequencies until it fits."""
    import heapq

    f = [float(x) for x in hist]
    while True:
        live = [i for i, x in enumerate(f) if x > 0]
        lens = [0] * len(f)
        if len(live) == 1:
            lens[live[0]] = 1
            return lens
        heap = [(f[i], i, [i]) for i in live]
        heapq.heapify(heap)
        tie = len(f)
        while len(heap) > 1:
            a, b = heapq.heappop(heap), heapq.heappop(heap)
            for s_ in a[2] + b[2]:
                lens[s_] += 1
            heapq.heappush(heap, (a[0] + b[0], tie, a[2] + b[2]))
            tie += 1
        if max(lens) <= lmax:
            return lens
        top = max(f)
        f = [x + top * 1e-3 if x > 0 else 0.0 for x in f]


def pack_range_huff(v: torch.Tensor) -> torch.Tensor:
    """Huffman-pack one range of bf16 values (format 1; see unpack.cu):
    returns the packed bytes on v's device."""
    dev = v.device
    u = v.view(torch.int16).to(torch.int32) & 0xFFFF
    n = u.numel()
    e = ((u >> 7) & 0xFF).long()
    lens = huff_lengths(torch.bincount(e, minlength=256).cpu().tolist())
    # canonical codes, stored bit-reversed for LSB-first reading
    code_of, code, prev = [0] * 256, 0, 0
    for sym in sorted((s_ for s_ in range(256) if lens[s_]), key=lambda s_: (lens[s_], s_)):
        code <<= lens[sym] - prev
        prev = lens[sym]
        code_of[sym] = int(format(code, f"0{prev}b")[::-1], 2)
        code += 1
    lut = torch.zeros(1 << HUFF_BITS, dtype=torch.int32)
    for sym in range(256):
        if lens[sym]:
            lut[code_of[sym]::1 << lens[sym]] = sym | (lens[sym] << 8)
    L = torch.tensor(lens, dtype=torch.int64, device=dev)[e]
    Cd = torch.tensor(code_of, dtype=torch.int64, device=dev)[e]
    nb = -(-n // HUFF_BLOCK)
    pad = nb * HUFF_BLOCK - n
    Lb = torch.cat([L, L.new_zeros(pad)]).view(nb, HUFF_BLOCK)
    block_words = (Lb.sum(1) + 31) // 32
    word_off = torch.cumsum(block_words, 0) - block_words        # first word of each block
    pos = (torch.cumsum(Lb, 1) - Lb).flatten()[:n] + word_off.repeat_interleave(HUFF_BLOCK)[:n] * 32
    total_words = int(block_words.sum()) + 2                      # +2: the decoder's refill may read ahead
    words = torch.zeros(total_words + 1, dtype=torch.int64, device=dev)
    w, sh = pos >> 5, pos & 31
    words.scatter_add_(0, w, (Cd << sh) & 0xFFFFFFFF)
    words.scatter_add_(0, w + 1, Cd >> (32 - sh))                 # the part spilling into the next word
    lut_off, offs_off, words_off = huff_sections(n)
    out = torch.zeros(words_off + 4 * total_words, dtype=torch.uint8, device=dev)
    out[:n] = (((u >> 8) & 0x80) | (u & 0x7F)).to(torch.uint8)
    out[lut_off:lut_off + 2 * (1 << HUFF_BITS)] = lut.to(torch.int16).view(torch.uint8).to(dev)
    out[offs_off:offs_off + 4 * nb] = word_off.to(torch.int32).view(torch.uint8)
    out[words_off:] = words[:total_words].to(torch.int32).view(torch.uint8)  # low 32 bits (two's complement)
    return out


def pack_stream(cfg: ModelConfig, flat: torch.Tensor, huffman: bool = True) -> PackedImage:
    """PackedImage of every streamable range of ``flat`` (the bf16 slot image;
    packing runs where ``flat`` lives — on the GPU it takes seconds)."""
    ranges = cfg.layout().stream_ranges(0)
    parts, desc, off = [], [], 0
    for dst, src, nbytes in ranges:
        v = flat[src // 2: (src + nbytes) // 2]
        if huffman:
            blob, base, n_esc = pack_range_huff(v), -1, 0
        else:
            blob, base, n_esc = pack_range(v)
        desc.append([dst, off, nbytes // 2, base, n_esc, blob.numel()])
        parts.append(blob)
        off += _align(blob.numel(), 256)
    host = torch.empty(off, dtype=torch.uint8, pin_memory=True)
    for d, p in zip(desc, parts):
        host[d[1]:d[1] + p.numel()].copy_(p)
    return PackedImage(host, desc, ranges)

"""Packed cold-start stream: the lossless bf16 packing format (host side,
CPU) and the device unpack + packed activation (GPU) reproduce the weight
bytes exactly."""

import numpy as np
import pytest
import torch

from paper_2512_09472_b200.weights import pack_range, packed_sections


def _unpack_numpy(blob: np.ndarray, n: int, base: int, n_esc: int) -> np.ndarray:
    """Reference decoder of the packed layout (the one csrc/kernels/unpack.cu implements)."""
    c_off, i_off, e_off, _ = packed_sections(n, n_esc)
    lo = blob[:n].astype(np.uint32)
    codes = blob[c_off:c_off + (n + 1) // 2]
    code = np.empty(2 * codes.size, dtype=np.uint32)
    code[0::2] = codes & 0xF
    code[1::2] = codes >> 4
    code = code[:n]
    e = (base + code) & 0xFF
    idx = blob[i_off:i_off + 4 * n_esc].view(np.uint32)
    e[idx] = blob[e_off:e_off + n_esc]
    return (((lo & 0x80) << 8) | (e << 7) | (lo & 0x7F)).astype(np.uint16)


@pytest.mark.parametrize("n", [1, 15, 16, 33, 4096 * 3 + 5])
def test_pack_roundtrip_cpu(n):
    g = torch.Generator().manual_seed(n)
    v = (torch.randn(n, generator=g) * 0.02).bfloat16()
    if n > 20:  # escapes: exact zeros, norm-like gains, huge and tiny values, inf
        v[3] = 0.0
        v[7] = 1.0
        v[11] = -3.0e4
        v[13] = 1e-30
        v[17] = float("inf")
    blob, base, n_esc = pack_range(v)
    assert 0 <= base <= 240
    if n > 20:
        assert n_esc >= 3  # zero, 1e-30, -3e4 and inf cannot share one 15-exponent window
    got = _unpack_numpy(blob.numpy(), n, base, n_esc)
    assert np.array_equal(got, v.view(torch.int16).numpy().view(np.uint16))
    assert blob.numel() <= 2 * n * 0.80 + 64 + 5 * n_esc  # ~12 bits per value


def test_pack_ratio_on_weight_like_values():
    v = (torch.randn(1 << 20, generator=torch.Generator().manual_seed(3)) * 0.02).bfloat16()
    blob, _, n_esc = pack_range(v)
    assert n_esc < 1e-3 * v.numel()
    assert blob.numel() / (2 * v.numel()) < 0.76


@pytest.mark.gpu
@pytest.mark.parametrize("huffman,shape", [(True, "llama"), (False, "llama"), (True, "qwen"), (True, "phi")])
def test_packed_activation_matches_plain(cuda_device, huffman, shape):
    """Cold activation of the tiny model from the packed stream: the slot
    holds exactly the bf16 image afterwards and the logits equal the plain
    (unpacked) stream's bit for bit."""
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    cfg = {"llama": M.TINY,
           "qwen": M.TINY.with_(name="tq", qkv_bias=True, rope_theta=1e6, rms_eps=1e-6),
           "phi": M.TINY.with_(name="tp", heads=4, kv_heads=4, head_dim=96, hidden=384, rope_theta=1e4)}[shape]
    w = UniversalWorker(cuda_device, pool_pages=64, max_tokens=1024)
    try:
        flat = synth_flat(cfg, seed=5, device="cuda")
        host = pinned_host_copy(flat)
        w.register(cfg, host)
        prompt = torch.randint(0, cfg.vocab, (300,), generator=torch.Generator().manual_seed(1),
                               dtype=torch.int32).pin_memory()
        w.prewarm(cfg.name, layers=1, full=False)
        plain = w.activate_instance(cfg.name, prompt)
        ref_logits = w.logits[: cfg.vocab].clone()
        w.release()
        w.set_packed(cfg.name, pack_stream(cfg, flat, huffman=huffman))
        w.drop_suffix(cfg.name, 1)
        w.slot_view(cfg.name)[cfg.layout().prefix_bytes(1) // 2:].zero_()  # the suffix must come from the stream
        packed = w.activate_instance(cfg.name, prompt)
        assert packed.streamed_layers == cfg.layers - 1
        assert packed.streamed_bytes < (0.7 if huffman else 0.8) * plain.streamed_bytes
        assert torch.equal(w.slot_view(cfg.name)[: host.numel()].cpu().view(torch.int16), host.view(torch.int16))
        assert torch.equal(w.logits[: cfg.vocab], ref_logits)
        assert packed.token == plain.token
        w.release()
    finally:
        w.close()


def _unhuff_numpy(blob: np.ndarray, n: int) -> np.ndarray:
    """Reference decoder of the Huffman layout (format 1, csrc/kernels/unpack.cu)."""
    from paper_2512_09472_b200.weights import HUFF_BITS, HUFF_BLOCK, huff_sections

    lut_off, offs_off, words_off = huff_sections(n)
    lo = blob[:n].astype(np.uint32)
    lut = blob[lut_off:lut_off + 2 * (1 << HUFF_BITS)].view(np.uint16)
    nb = -(-n // HUFF_BLOCK)
    offs = blob[offs_off:offs_off + 4 * nb].view(np.uint32)
    words = blob[words_off:].view(np.uint32)
    out = np.empty(n, dtype=np.uint16)
    for b in range(nb):
        bits = int(words[offs[b]]) | (int(words[offs[b] + 1]) << 32)
        have, nxt = 64, offs[b] + 2
        for v in range(b * HUFF_BLOCK, min(n, (b + 1) * HUFF_BLOCK)):
            ent = int(lut[bits & ((1 << HUFF_BITS) - 1)])
            ln = ent >> 8
            bits >>= ln
            have -= ln
            if have < 32:
                bits |= int(words[nxt]) << have
                nxt += 1
                have += 32
            e = ent & 0xFF
            out[v] = ((lo[v] & 0x80) << 8) | (e << 7) | (lo[v] & 0x7F)
    return out


@pytest.mark.parametrize("n", [1, 7, 1024, 1025, 3000])
def test_huffman_roundtrip_cpu(n):
    from paper_2512_09472_b200.weights import pack_range_huff

    g = torch.Generator().manual_seed(100 + n)
    v = (torch.randn(n, generator=g) * 0.02).bfloat16()
    if n > 20:
        v[3] = 0.0
        v[7] = 1.0
        v[11] = -3.0e4
        v[17] = float("inf")
    blob = pack_range_huff(v)
    got = _unhuff_numpy(blob.numpy(), n)
    assert np.array_equal(got, v.view(torch.int16).numpy().view(np.uint16))


def test_huffman_ratio_on_weight_like_values():
    from paper_2512_09472_b200.weights import pack_range_huff

    v = (torch.randn(1 << 20, generator=torch.Generator().manual_seed(4)) * 0.02).bfloat16()
    blob = pack_range_huff(v)
    assert blob.numel() / (2 * v.numel()) < 0.68  # ~10.6 bits per weight + block offsets + LUT

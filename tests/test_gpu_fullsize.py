"""Parity of the BENCHMARKED configuration against the CPU fp32 oracle.

BASELINE configs[1] exactly as bench.py runs it: Llama-3-8B at full depth
(32 layers, vocab 128256), first 4 layers prewarmed, 2048-token prompts,
cold ``activate_instance`` with layers 4..31 + lm_head streamed over PCIe —
once through the plain bf16 stream and once through the packed (Huffman
exponent) stream — then a warm activation. The three activations must give
bit-identical logits (same kernels, same bytes, the stream only changes when
bytes land), and match the fp32 oracle (oracle/llama_fp32.forward_streamed,
reading the same bf16 bytes): greedy token equal, and the logits error
||gpu - ref|| / ||ref|| no larger than the bf16 floor — the same oracle run
with every bf16-held tensor rounded to bf16 (``emulate_bf16``) — plus 25%.

Why not the flat 2e-2 at full depth: on these random-init weights a 32-layer
forward amplifies bf16 rounding chaotically. The ideal bf16 forward sits at
4.3e-2 from fp32 at 32 layers (1.5e-2 at 4, 2.2e-2 at 8, 2.9e-2 at 16;
DESIGN.md §2), so no bf16 implementation meets 2e-2 there; the measured GPU
error equals that floor. The flat 2e-2 bar is asserted at the depths where
the floor permits it (the 2- and 4-layer full-width tests below).

Also the other co-prewarmed families of configs[2] at FULL width (hidden,
heads, GQA groups, head_dim, vocab, qkv bias, RoPE theta / eps of the public
configs) with 2 decoder layers and 2048-token prompts, plus one decode step
over the KV the prefill appended.

Reference: the prefill these replace is LatencyModel.prefill_ms
(engine.py:107-108); catch-up semantics at k=4 are cluster.py:169-182.
"""

from __future__ import annotations

import json
import os
import time

import pytest
import torch

from oracle import llama_fp32 as O

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 2e-2
S = 2048


def _rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / b.norm()).item()


def _prompt(vocab, seed, n=S):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (n,), generator=g, dtype=torch.int32)


def _report(name, payload):
    out = os.environ.get("WS_REPORT_DIR", "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, name), "w") as f:
            json.dump(payload, f, indent=1)
    except OSError:
        pass


@pytest.fixture(scope="module")
def llama8b(cuda_device):
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    torch.cuda.set_device(cuda_device)
    cfg = M.LLAMA3_8B
    flat = synth_flat(cfg, seed=0, device="cuda")
    host = pinned_host_copy(flat)
    packed = pack_stream(cfg, flat)
    del flat
    torch.cuda.empty_cache()
    w = UniversalWorker(0, pool_pages=8192, max_tokens=S)
    w.register(cfg, host)
    w.prewarm(cfg.name, layers=4, full=False)
    yield cfg, w, host, packed
    w.release()
    w.close()


def test_llama3_8b_full_depth_cold_k4_plain_and_packed_match_oracle(llama8b):
    from paper_2512_09472_b200 import _native as N

    cfg, w, host, packed = llama8b
    fb0 = N.fallback_counts()
    results = []
    for seed in (7, 8):
        prompt = _prompt(cfg.vocab, seed).pin_memory()
        # cold, plain bf16 stream: layers 4..31 + lm_head over PCIe
        w.drop_suffix(cfg.name, 4)
        cold = w.activate_instance(cfg.name, prompt)
        assert cold.streamed_layers == cfg.layers - 4
        plain = w.logits[: cfg.vocab].clone()
        w.release()
        # cold, packed stream (GPU unpack of the Huffman-coded exponents)
        w.set_packed(cfg.name, packed)
        w.drop_suffix(cfg.name, 4)
        coldp = w.activate_instance(cfg.name, prompt)
        w.models[cfg.name].packed = None
        packed_logits = w.logits[: cfg.vocab].clone()
        w.release()
        # warm: every layer resident
        warm = w.activate_instance(cfg.name, prompt)
        assert warm.streamed_layers == 0
        warm_logits = w.logits[: cfg.vocab].clone()
        w.release()
        assert torch.equal(plain, packed_logits), "packed stream changed the weights"
        assert torch.equal(plain, warm_logits), "cold and warm forwards differ"
        assert cold.token == coldp.token == warm.token
        t0 = time.perf_counter()
        ref = O.forward_streamed(cfg, cfg.layout(), host, prompt.long())
        oracle_s = time.perf_counter() - t0
        emu = O.forward_streamed(cfg, cfg.layout(), host, prompt.long(), emulate_bf16=True)
        floor = _rel(emu, ref)
        rel = _rel(plain, ref)
        top2 = ref.topk(2)
        results.append({"seed": seed, "rel": rel, "bf16_floor_rel": floor, "gpu_token": cold.token,
                        "ref_token": int(top2.indices[0]), "bf16_floor_token": int(emu.argmax()),
                        "ref_margin": float(top2.values[0] - top2.values[1]),
                        "cold_plain_ttft_ms": cold.ttft_ms, "cold_packed_ttft_ms": coldp.ttft_ms,
                        "warm_ttft_ms": warm.ttft_ms, "oracle_cpu_s": oracle_s,
                        "cpu_threads": torch.get_num_threads()})
        print(f"\nseed {seed}: rel {rel:.2e} (bf16 floor {floor:.2e}), token gpu {cold.token} ref {int(top2.indices[0])} "
              f"(margin {results[-1]['ref_margin']:.3e}); TTFT cold {cold.ttft_ms:.1f} / packed "
              f"{coldp.ttft_ms:.1f} / warm {warm.ttft_ms:.1f} ms; oracle {oracle_s:.0f} s")
    assert N.fallback_counts() == fb0, "the benchmarked path fell back to a legacy kernel"
    _report("r2_llama8b_full_parity.json", {"config": "llama3-8b, 32 layers, k=4, 2048 tokens", "rows": results})
    for r in results:
        assert r["rel"] <= 1.25 * r["bf16_floor_rel"], r
        assert r["gpu_token"] == r["ref_token"], r


@pytest.mark.parametrize("layers", [4])
def test_llama3_8b_full_width_depth_within_2e2(cuda_device, layers):
    """The flat north_star bar (2e-2) at full Llama-3-8B width and vocab, at
    the deepest prefix where the bf16 floor permits it (4 layers: floor
    ~1.5e-2), cold-started from 1 resident layer over 2048 tokens."""
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    torch.cuda.set_device(cuda_device)
    cfg = M.LLAMA3_8B.with_(layers=layers)
    host = pinned_host_copy(synth_flat(cfg, seed=1, device="cuda"))
    torch.cuda.empty_cache()
    w = UniversalWorker(0, pool_pages=-(-cfg.layout().total // M.PAGE) + 160, max_tokens=S)
    try:
        w.register(cfg, host)
        w.prewarm(cfg.name, layers=1, full=False)
        rows = []
        for seed in (3, 4):
            prompt = _prompt(cfg.vocab, seed).pin_memory()
            w.drop_suffix(cfg.name, 1)
            r = w.activate_instance(cfg.name, prompt)
            got = w.logits[: cfg.vocab].clone()
            w.release()
            ref = O.forward_streamed(cfg, cfg.layout(), host, prompt.long())
            rows.append((seed, _rel(got, ref), r.token, int(ref.argmax())))
        print(f"\n8B width, {layers} layers: {rows}")
        for seed, rel, tg, tr in rows:
            assert rel < LOGIT_RTOL and tg == tr, (seed, rel, tg, tr)
    finally:
        w.close()


@pytest.mark.parametrize("name", ["qwen2.5-7b", "mistral-7b", "phi3-mini", "llama3-8b"])
def test_full_width_families_two_layers_match_oracle(cuda_device, name):
    """Full-width shapes of the configs[2] families, 2 decoder layers, 2048
    tokens, real vocab; cold activation (layer 1 + lm_head streamed), then one
    decode step over the appended KV."""
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    torch.cuda.set_device(cuda_device)
    cfg = M.ALL[name].with_(layers=2)
    flat = synth_flat(cfg, seed=5, device="cuda")
    host = pinned_host_copy(flat)
    del flat
    pages = -(-cfg.layout().total // M.PAGE)
    tpb, _ = cfg.kv_geometry()
    w = UniversalWorker(0, pool_pages=pages + -(-(S + 8) // tpb) + 16, max_tokens=S)
    try:
        w.register(cfg, host)
        w.prewarm(cfg.name, layers=1, full=False)
        prompt = _prompt(cfg.vocab, 21).pin_memory()
        res = w.activate_instance(cfg.name, prompt, keep_seq=True)
        assert res.streamed_layers == 1
        got = w.logits[: cfg.vocab].clone()
        weights = O.unpack(cfg, cfg.layout(), host)
        ref, past = O.forward(cfg, weights, prompt.long())
        rel = _rel(got, ref[-1])
        tok = int(ref[-1].argmax())
        print(f"\n{name} (2 layers, full width): prefill rel {rel:.2e}, token gpu {res.token} ref {tok}")
        assert rel < LOGIT_RTOL
        assert res.token == tok
        logits, _ = w.decode(torch.tensor([res.seq], dtype=torch.int32, device="cuda"),
                             torch.tensor([S], dtype=torch.int32, device="cuda"),
                             torch.tensor([tok], dtype=torch.int32, device="cuda"), S + 1)
        ref2, _ = O.forward(cfg, weights, [tok], pos0=S, past=past)
        rel2 = _rel(logits[0], ref2[0])
        print(f"{name}: decode rel {rel2:.2e}")
        assert rel2 < LOGIT_RTOL
        w.close_seq(res.seq)
        w.release()
    finally:
        w.close()

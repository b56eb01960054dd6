"""Background prewarm to full residency (engine.py:885-919, 658-686):
"ready" once k layers have landed, "full" at L, ``layers_loaded`` /
``weight_bytes_loaded`` following the per-layer copy events; an activation
during the load rides it layer by layer; a promote that evicts a slot whose
load is still in flight must not let those copies land on the new KV pages;
reclaim reads KV usage from the pool's live blocks (engine.py:391-404)."""

import pytest
import torch

from oracle import llama_fp32 as O

pytestmark = pytest.mark.gpu

S = 1024


def _rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / b.norm()).item()


def _setup(names):
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    base = M.TINY.with_(hidden=4096, heads=32, kv_heads=8, head_dim=128, ffn=14336, layers=6, vocab=8192)
    cfgs = [base.with_(name=n) for n in names]
    pages = sum(-(-c.layout().total // M.PAGE) for c in cfgs)
    w = UniversalWorker(0, pool_pages=pages + 256, max_tokens=S)
    hosts = {}
    for i, c in enumerate(cfgs):
        hosts[c.name] = pinned_host_copy(synth_flat(c, seed=40 + i, device="cuda"))
        w.register(c, hosts[c.name])
    torch.cuda.empty_cache()
    return w, cfgs, hosts


def test_background_prewarm_ready_then_full(cuda_device):
    w, (cfg,), hosts = _setup(["bg"])
    try:
        slot = w.prewarm(cfg.name, layers=2, wait="ready")
        assert slot.required_prewarm_layers == 2
        seen = [w.residency(cfg.name)]
        assert seen[0] >= 2  # "ready": k layers resident on return
        while seen[-1] < cfg.layers:
            seen.append(w.residency(cfg.name))
        assert seen == sorted(seen)  # monotone, layer by layer
        w.wait_resident(cfg.name)
        assert slot.layers_loaded == cfg.layers
        assert slot.weight_bytes_loaded == float(cfg.layout().total)
        assert slot.load_finish is not None
        got = w.slot_view(cfg.name).cpu()
        assert torch.equal(got, hosts[cfg.name])  # every byte landed
    finally:
        w.close()


def test_activation_rides_inflight_prewarm_and_eviction_fences_copies(cuda_device):
    """Model b is prewarmed in the background and activated at once: its
    prefill waits per layer on that load (same logits as a warm run). Then
    model a's load is left in flight and b is re-promoted (a evicted, its
    pages become KV): b's KV and next decode step must match the oracle."""
    w, (ca, cb), hosts = _setup(["a", "b"])
    try:
        g = torch.Generator().manual_seed(3)
        prompt = torch.randint(0, cb.vocab, (S,), generator=g, dtype=torch.int32).pin_memory()
        w.prewarm(cb.name, layers=1, wait=None)
        r1 = w.activate_instance(cb.name, prompt)
        assert r1.streamed_layers == 0 and w.slot(cb.name).layers_loaded == cb.layers
        l1 = w.logits[: cb.vocab].clone()
        w.release()
        r2 = w.activate_instance(cb.name, prompt)  # warm
        assert torch.equal(w.logits[: cb.vocab], l1) and r2.token == r1.token
        w.release()
        wb = O.unpack(cb, cb.layout(), hosts[cb.name])
        ref, past = O.forward(cb, wb, prompt.long())
        assert _rel(l1, ref[-1]) < 2e-2 and r1.token == int(ref[-1].argmax())
        # a's load in flight while b is promoted again: a is evicted
        w.prewarm(ca.name, layers=1, wait=None)
        r3 = w.activate_instance(cb.name, prompt, keep_seq=True)
        assert [m for _, m in r3.evicted] == [ca.name]
        tok = int(ref[-1].argmax())
        logits, _ = w.decode(torch.tensor([r3.seq], dtype=torch.int32, device="cuda"),
                             torch.tensor([S], dtype=torch.int32, device="cuda"),
                             torch.tensor([tok], dtype=torch.int32, device="cuda"), S + 1)
        ref2, _ = O.forward(cb, wb, [tok], pos0=S, past=past)
        assert _rel(logits[0], ref2[0]) < 2e-2
        # reclaim from device truth: the live blocks of the open sequence
        tpb, per_tok = cb.kv_geometry()
        used = w.kv_used_bytes()
        assert used == -(-(S + 1) // tpb) * w.page_size
        freed = w.reclaim(inflight=1)
        cap = w.gpu.kv_capacity_pages
        assert w.gpu.kv_pages_mapped * w.page_size >= used and freed > 0 and cap > 0
        w.release()
    finally:
        w.close()


def test_prefix_prewarm_with_head_streams_only_layers(cuda_device):
    """prewarm(k, full=False, head=True): embedding, layers [0, k) and the
    final norm + lm_head resident; a cold activation streams only layers
    k..L-1 (no tail range) and matches a warm run bit for bit."""
    w, (cfg,), hosts = _setup(["hd"])
    try:
        g = torch.Generator().manual_seed(5)
        prompt = torch.randint(0, cfg.vocab, (S,), generator=g, dtype=torch.int32).pin_memory()
        slot = w.prewarm(cfg.name, layers=2, full=False, head=True, wait="full")
        lay = cfg.layout()
        assert w.residency(cfg.name) == 2 and slot.head_resident
        assert slot.weight_bytes_loaded == float(lay.prefix_bytes(2) + lay.total - lay.final_norm)
        cold = w.activate_instance(cfg.name, prompt)
        assert cold.streamed_layers == cfg.layers - 2
        assert cold.streamed_bytes == lay.final_norm - lay.prefix_bytes(2)
        l1 = w.logits[: cfg.vocab].clone()
        w.release()
        warm = w.activate_instance(cfg.name, prompt)
        assert warm.streamed_bytes == 0 and torch.equal(w.logits[: cfg.vocab], l1)
        w.release()
    finally:
        w.close()

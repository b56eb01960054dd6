"""__graft_entry__.smoke(): one cold activation of the tiny model (BASELINE
config 1: layer 0 + embedding prewarmed, 512-token prompt) through the worker
API on cuda:0 over the packed (Huffman) layer stream, checked against the CPU
fp32 oracle; plus one memory switch whose ledger is checked against the
reference-pinned ledger oracle."""

from __future__ import annotations


def run_smoke() -> None:
    import torch

    from oracle import ledger as OL
    from oracle import llama_fp32 as O
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    assert torch.cuda.is_available(), "smoke needs cuda:0"
    cfg = M.TINY
    w = UniversalWorker(0, pool_pages=64, max_tokens=1024)
    flat = synth_flat(cfg, seed=1, device="cuda")
    host = pinned_host_copy(flat)
    w.register(cfg, host)
    w.set_packed(cfg.name, pack_stream(cfg, flat))
    w.prewarm(cfg.name, layers=1, full=False)  # embedding + layer 0 resident: layer 1 + head stream
    prompt = torch.randint(0, cfg.vocab, (512,), generator=torch.Generator().manual_seed(0),
                           dtype=torch.int32).pin_memory()
    res = w.activate_instance(cfg.name, prompt)
    ref, _ = O.forward(cfg, O.unpack(cfg, cfg.layout(), host.clone()), prompt.long())
    got = w.logits[: cfg.vocab].double().cpu()
    rel = ((got - ref[-1].double()).norm() / ref[-1].double().norm()).item()
    assert rel < 2e-2, f"logits rel err {rel}"
    assert res.token == int(ref[-1].argmax()), (res.token, int(ref[-1].argmax()))
    # ledger after the switch == oracle ledger for the same op
    cl = OL.new_cluster(1, 1, 64, M.PAGE)
    OL.begin_prewarm(cl, 0, cfg.name, w.models[cfg.name].spec.partition_pages(M.PAGE), 1)
    OL.promote(cl, [0], cfg.name, 1, w.models[cfg.name].spec.weight_bytes, 32, 1)
    want = OL.snapshot(cl)[0]
    c = w.gpu.counts()
    assert [w.gpu.role.value, c.free_pages, c.kv_pages_mapped, c.kv_capacity_pages] == \
        [want[0], want[1], want[2], want[4]], (want, c.free_pages, c.kv_pages_mapped)
    w.release()
    w.close()
    assert res.streamed_layers == cfg.layers - 1
    print(f"smoke ok: cold TTFT {res.ttft_ms:.2f} ms (packed stream {res.streamed_bytes} B), token {res.token}, "
          f"logits rel err {rel:.2e}, "
          f"switch {res.switch_ms*1e3:.0f} us host / {res.switch_kernel_ms*1e3:.1f} us kernel")

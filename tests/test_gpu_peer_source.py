"""Peer-HBM weight source: a worker process exports its
slot's physical handles (POSIX fds over a Unix socket), another worker
process maps them and cold-starts with layers k..L streamed device-to-device
from that mapping — no host staging. On one GPU both processes share it (the
copy stays in HBM); with >= 2 GPUs the exporter sits on cuda:1 and the copy
crosses NVLink (skipped below 2 GPUs). The cold logits must equal a warm
activation's bit for bit, and the oracle's."""

from __future__ import annotations

import os

import pytest
import torch

pytestmark = pytest.mark.gpu

S = 1024


def _cfg():
    from paper_2512_09472_b200 import models as M

    return M.TINY.with_(name="peer", hidden=4096, heads=32, kv_heads=8, head_dim=128, ffn=14336, layers=4,
                        vocab=8192)


def _exporter(device, tag, q_ready, q_done):
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.peer_source import serve_export
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    torch.cuda.set_device(device)
    cfg = _cfg()
    host = pinned_host_copy(synth_flat(cfg, seed=9, device=f"cuda:{device}"))
    w = UniversalWorker(device, pool_pages=-(-cfg.layout().total // M.PAGE) + 64, max_tokens=S)
    w.register(cfg, host)
    w.prewarm(cfg.name, layers=cfg.layers, wait="full")
    q_ready.put("ready")
    serve_export(w, cfg.name, tag)
    q_done.get(timeout=300)  # keep the slot resident until the importer is done
    w.close()


def _run(exporter_device):
    import torch.multiprocessing as mp

    from oracle import llama_fp32 as O
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.peer_source import PeerSource
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    ctx = mp.get_context("spawn")
    q_ready, q_done = ctx.Queue(), ctx.Queue()
    tag = f"t{os.getpid()}-{exporter_device}"
    p = ctx.Process(target=_exporter, args=(exporter_device, tag, q_ready, q_done))
    p.start()
    try:
        assert q_ready.get(timeout=300) == "ready"
        cfg = _cfg()
        host = pinned_host_copy(synth_flat(cfg, seed=9, device="cuda:0"))
        w = UniversalWorker(0, pool_pages=-(-cfg.layout().total // M.PAGE) + 64, max_tokens=S)
        try:
            w.register(cfg, host)
            w.prewarm(cfg.name, layers=1, full=False)
            ps = PeerSource(0, tag)
            prompt = torch.randint(0, cfg.vocab, (S,), generator=torch.Generator().manual_seed(4),
                                   dtype=torch.int32).pin_memory()
            w.slot_view(cfg.name)[cfg.layout().prefix_bytes(1) // 2:].zero_()  # the suffix must come from the peer
            cold = w.activate_instance(cfg.name, prompt, source=ps)
            assert cold.streamed_layers == cfg.layers - 1
            got = w.logits[: cfg.vocab].clone()
            w.release()
            warm = w.activate_instance(cfg.name, prompt)
            assert torch.equal(w.logits[: cfg.vocab], got) and warm.token == cold.token
            w.release()
            assert torch.equal(w.slot_view(cfg.name).cpu(), host)
            ref, _ = O.forward(cfg, O.unpack(cfg, cfg.layout(), host), prompt.long())
            rel = ((got.double().cpu() - ref[-1].double()).norm() / ref[-1].double().norm()).item()
            assert rel < 2e-2 and cold.token == int(ref[-1].argmax())
            gbs = cold.streamed_bytes / (cold.stream_ms / 1e3) / 1e9
            print(f"\npeer source (exporter cuda:{exporter_device}): {cold.streamed_bytes / 1e9:.2f} GB in "
                  f"{cold.stream_ms:.2f} ms = {gbs:.0f} GB/s; cold TTFT {cold.ttft_ms:.1f} ms, warm {warm.ttft_ms:.1f} ms")
            ps.close()
        finally:
            w.close()
    finally:
        q_done.put("done")
        p.join(120)
        if p.exitcode is None:
            p.kill()
    assert p.exitcode == 0


def test_peer_source_same_gpu_two_processes(cuda_device):
    _run(0)


def test_peer_source_over_nvlink(cuda_device):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (exporter on cuda:1, importer on cuda:0)")
    from paper_2512_09472_b200.peer_source import can_access_peer

    assert can_access_peer(0, 1), "no P2P between cuda:0 and cuda:1"
    _run(1)

"""Debug driver: prefill a small head_dim-128 model at several prompt lengths
and compare last-row logits with the CPU oracle (prints as it goes, so a hang
is localised). Usage: python tools/attn_debug.py [hd] [lens...]"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from oracle import llama_fp32 as O
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    hd = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    heads = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    kvh = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    lens = [int(x) for x in sys.argv[4:]] or [128, 256, 640, 2048]
    cfg = M.TINY.with_(name="dbg", head_dim=hd, hidden=heads * hd, heads=heads, kv_heads=kvh)
    w = UniversalWorker(0, pool_pages=1024, max_tokens=max(lens))
    host = pinned_host_copy(synth_flat(cfg, seed=2, device="cuda"))
    w.register(cfg, host)
    weights = O.unpack(cfg, cfg.layout(), host.clone())
    w.prewarm(cfg.name, layers=cfg.layers)
    import os
    w.set_gemm_impl(int(os.environ.get('WS_IMPL', '0')))
    w.switch_memory(cfg.name)
    for n in lens:
        prompt = torch.randint(0, cfg.vocab, (n,), generator=torch.Generator().manual_seed(n), dtype=torch.int32)
        s = w.open_seq(n)
        print(f"len {n}: launching", flush=True)
        w.prefill(s, prompt.cuda())
        torch.cuda.synchronize()
        got = w.logits[: cfg.vocab].double().cpu()
        w.close_seq(s)
        ref, _ = O.forward(cfg, weights, prompt.long())
        rel = ((got - ref[-1].double()).norm() / ref[-1].double().norm()).item()
        print(f"len {n}: rel err {rel:.3e} argmax {int(got.argmax())} vs {int(ref[-1].argmax())}", flush=True)
    w.release()
    w.close()


if __name__ == "__main__":
    main()

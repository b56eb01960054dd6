"""Greedy-token diagnosis at full Llama-3-8B depth for one prompt seed: the
kernel's argmax token, torch's argmax of the same GPU logits, and the top-5
of the GPU logits, the fp32 oracle and the bf16-floor oracle emulation.

    python tools/token_diag.py [seed]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import llama_fp32 as O  # noqa: E402
from paper_2512_09472_b200 import models as M  # noqa: E402
from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat  # noqa: E402
from paper_2512_09472_b200.worker import UniversalWorker  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = M.LLAMA3_8B
flat = synth_flat(cfg, seed=0, device="cuda")
host = pinned_host_copy(flat)
del flat
torch.cuda.empty_cache()
w = UniversalWorker(0, pool_pages=8192, max_tokens=2048)
w.register(cfg, host)
w.prewarm(cfg.name, layers=cfg.layers, wait="full")
prompt = torch.randint(0, cfg.vocab, (2048,), generator=torch.Generator().manual_seed(seed), dtype=torch.int32)
r = w.activate_instance(cfg.name, prompt.pin_memory())
gpu = w.logits[: cfg.vocab].float().cpu()
w.release()
w.close()


def top(x, k=5):
    v, i = x.double().topk(k)
    return [(int(a), round(float(b), 4)) for a, b in zip(i, v)]


print("kernel token", r.token, "torch argmax", int(gpu.argmax()))
print("gpu  ", top(gpu))
ref = O.forward_streamed(cfg, cfg.layout(), host, prompt.long())
print("fp32 ", top(ref))
emu = O.forward_streamed(cfg, cfg.layout(), host, prompt.long(), emulate_bf16=True)
print("bf16 ", top(emu))
print("rel gpu-ref", float((gpu.double() - ref.double()).norm() / ref.double().norm()),
      "rel emu-ref", float((emu.double() - ref.double()).norm() / ref.double().norm()),
      "rel gpu-emu", float((gpu.double() - emu.double()).norm() / emu.double().norm()))

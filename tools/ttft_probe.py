"""Probe cold TTFT decomposition for a given resident prefix (k layers, with or
without the lm_head resident): host TTFT, device time, stream time."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_09472_b200 import models as M  # noqa: E402
from paper_2512_09472_b200.weights import pinned_host_copy, synth_flat  # noqa: E402
from paper_2512_09472_b200.worker import UniversalWorker  # noqa: E402

cfg = M.LLAMA3_8B
flat = synth_flat(cfg, seed=0, device="cuda")
host = pinned_host_copy(flat)
del flat
torch.cuda.empty_cache()
w = UniversalWorker(0, pool_pages=12288, max_tokens=2048)
w.register(cfg, host)
w.prewarm(cfg.name, layers=cfg.layers, wait="full")
prompt = torch.randint(0, cfg.vocab, (2048,), generator=torch.Generator().manual_seed(1), dtype=torch.int32).pin_memory()
for k, head in [(32, True), (30, False), (29, False), (29, True), (28, True), (4, False), (4, True)]:
    rows = []
    for i in range(8):
        if k < cfg.layers:
            w.drop_suffix(cfg.name, k, head=head)
        r = w.activate_instance(cfg.name, prompt)
        w.release()
        rows.append((r.ttft_ms, r.device_ms, r.stream_ms, r.streamed_bytes))
    rows = rows[2:]
    med = [statistics.median(x[j] for x in rows) for j in range(4)]
    print(f"k={k} head={head}: ttft {med[0]:.1f} device {med[1]:.1f} stream {med[2]:.1f} ms, {med[3]/1e9:.2f} GB", flush=True)
w.close()

"""Distribution of cold TTFT at one resident prefix (k layers): per activation
host TTFT, device time, stream time and the per-range landing times, to find
where slow activations lose their time.

    python tools/ttft_dist.py [--k 30] [--n 40] [--packed] [--pool-pages 0]
"""
import argparse
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_09472_b200 import _native as N  # noqa: E402
from paper_2512_09472_b200 import models as M  # noqa: E402
from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat  # noqa: E402
from paper_2512_09472_b200.worker import UniversalWorker  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=30)
ap.add_argument("--n", type=int, default=40)
ap.add_argument("--packed", action="store_true")
ap.add_argument("--pool-pages", type=int, default=0)
a = ap.parse_args()
cfg = M.LLAMA3_8B
flat = synth_flat(cfg, seed=0, device="cuda")
host = pinned_host_copy(flat)
packed = pack_stream(cfg, flat) if a.packed else None
del flat
torch.cuda.empty_cache()
pages = a.pool_pages or int((torch.cuda.mem_get_info(0)[0] - 24 * (1 << 30)) // M.PAGE)
w = UniversalWorker(0, pool_pages=pages, max_tokens=2048)
w.register(cfg, host)
if packed is not None:
    w.set_packed(cfg.name, packed)
w.prewarm(cfg.name, layers=cfg.layers, wait="full")
gp = torch.Generator().manual_seed(1234)
rows = []
for i in range(a.n + 3):
    prompt = torch.randint(0, cfg.vocab, (2048,), generator=gp, dtype=torch.int32).pin_memory()
    w.drop_suffix(cfg.name, a.k)
    t0 = time.perf_counter()
    r = w.activate_instance(cfg.name, prompt)
    w.release()
    n_r = cfg.layers - a.k + 1
    times = (C.c_float * n_r)()
    N.call("ws_streamer_times", w.streamer, times, n_r)
    if i >= 3:
        rows.append((r.ttft_ms, r.device_ms, r.stream_ms, list(times)))
        print(f"{i - 3:3d} ttft {r.ttft_ms:6.1f} device {r.device_ms:6.1f} stream {r.stream_ms:6.1f} ranges "
              + " ".join(f"{t:5.1f}" for t in times), flush=True)
tt = sorted(x[0] for x in rows)
print(f"k={a.k} packed={a.packed}: ttft p50 {statistics.median(tt):.1f} min {tt[0]:.1f} max {tt[-1]:.1f}")
w.close()

"""Cold activation of Llama-3-8B (k = 4) with the suffix streamed from an
HBM-resident copy (bench.py's "cold hbm" leg), a few times, with a Python
stack dump if one activation takes longer than --stall seconds.

    python tools/hbm_leg_probe.py [--n 5] [--stall 60] [--plain-first]
"""

from __future__ import annotations

import argparse
import faulthandler
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=5)
    ap.add_argument("--stall", type=float, default=60.0)
    ap.add_argument("--plain-first", action="store_true")
    ap.add_argument("--pool-pages", type=int, default=0)
    ap.add_argument("--first-n", type=int, default=4, help="activations per plain / packed leg")
    ap.add_argument("--smi", action="store_true", help="nvidia-smi -lms 200 into an unread pipe (as bench.py)")
    a = ap.parse_args()
    cfg = M.ALL["llama3-8b"]
    flat = synth_flat(cfg, seed=0, device="cuda")
    host = pinned_host_copy(flat)
    packed = pack_stream(cfg, flat)
    del flat
    torch.cuda.empty_cache()
    pages = a.pool_pages
    if pages <= 0:
        free_b, _ = torch.cuda.mem_get_info(0)
        pages = int((free_b - 24 * (1 << 30)) // M.PAGE)
    w = UniversalWorker(0, pool_pages=pages, max_tokens=2048)
    w.register(cfg, host)
    w.prewarm(cfg.name, layers=4, full=False)
    prompt = torch.randint(0, cfg.vocab, (2048,), generator=torch.Generator().manual_seed(7),
                           dtype=torch.int32).pin_memory()
    print(f"setup done, pool pages {pages}", flush=True)

    if a.smi:
        import subprocess
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm", "--format=csv,noheader,nounits",
                                "-lms", "200", "-i", "0"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                               text=True)

    def run(src, tag, n=None):
        for i in range(a.n if n is None else n):
            w.drop_suffix(cfg.name, 4, head=False)
            faulthandler.dump_traceback_later(a.stall, exit=True)
            t0 = time.perf_counter()
            r = w.activate_instance(cfg.name, prompt, source=src)
            w.release()
            torch.cuda.synchronize()
            faulthandler.cancel_dump_traceback_later()
            print(f"{tag} {i}: ttft {r.ttft_ms:.2f} ms wall {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)

    if a.plain_first:
        run(None, "plain", a.first_n)
        w.set_packed(cfg.name, packed)
        run(None, "packed", a.first_n)
        w.models[cfg.name].packed = None
    dev_src = host.to("cuda:0")
    torch.cuda.synchronize()
    print("device source ready", flush=True)
    run(dev_src, "hbm")
    w.close()


if __name__ == "__main__":
    main()

"""BASELINE config 3: four models co-prewarmed on one B200, weight<->KV memory
switch under a seeded burst.

Llama-3-8B, Qwen2.5-7B, Mistral-7B and Phi-3-mini are prewarmed into four
slots of one device pool (windowed slots over the page window). The burst is
a seeded sequence of switches, each one:

  activate(m)   promote_to_dedicated (cluster.py:291-342): the other slots are
                evicted, every free page becomes KV via the switch kernel
  prefill       a short prompt on the paged pool (exercises the new KV pages)
  grace+reclaim reclaim_on_completion (cluster.py:351-365) frees KV pages
                above Eq. 1's target (cluster.py:185-197)
  proactive     begin_prewarm of another model into the reclaimed pages
                (Fig. 4b), weights copied from a device-resident image
  release       release_instance (cluster.py:367-387): back to universal,
                holding m and the proactively loaded model

`run_burst` takes an ``on_op(kind, args)`` observer called after every ledger
op; tests/test_gpu_config3.py replays each op on the reference-pinned oracle
(oracle/ledger.py) and compares the ledger, bench.py reports the latencies.
This module never imports the oracle.

    python tools/config3_switch_burst.py [--switches 1000] [--pool-pages 32768]
"""

from __future__ import annotations

import argparse
import json
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = (len(xs) - 1) * q / 100.0
    f = int(k)
    c = min(f + 1, len(xs) - 1)
    return xs[f] + (xs[c] - xs[f]) * (k - f)


def run_burst(switches: int = 1000, pool_pages: int = 32768, prompt: int = 128, seed: int = 7, device: int = 0,
              on_op=None, progress=None) -> dict:
    """Run the config-3 burst on a fresh UniversalWorker; return the summary
    dict (latencies in µs / ms, counts). ``on_op(kind, worker, **info)`` is
    called after every ledger-changing op with the op's arguments."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.cluster import InstanceState
    from paper_2512_09472_b200.weights import synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    op = on_op or (lambda *a, **k: None)
    cfgs = [M.LLAMA3_8B, M.QWEN25_7B, M.MISTRAL_7B, M.PHI3_MINI]
    t0 = time.perf_counter()
    w = UniversalWorker(device, pool_pages=pool_pages, max_tokens=max(prompt, 256), max_seqs=8)
    init_s = time.perf_counter() - t0
    try:
        src = {}
        for c in cfgs:
            src[c.name] = synth_flat(c, seed=1, device=f"cuda:{device}")  # device-resident image (peer stand-in)
            w.register(c, None)
        torch.cuda.synchronize()
        spec = {c.name: w.models[c.name].spec for c in cfgs}

        def prewarm(name):
            w.prewarm(name, layers=spec[name].layers, source=src[name])
            op("prewarm", w, model=name, pages=spec[name].partition_pages(M.PAGE),
               required=max(1, spec[name].layers))

        prewarm_ms = []
        for c in cfgs:
            t = time.perf_counter()
            prewarm(c.name)
            prewarm_ms.append((time.perf_counter() - t) * 1e3)
        rng = random.Random(seed)
        lat = {"promote": [], "reclaim": [], "release": [], "prefill": [], "proactive_prewarm": []}
        kernel_us, evicted_n = [], []
        for i in range(switches):
            if progress and i % 100 == 0:
                progress(f"switch {i}")
            m = rng.choice(sorted(w.gpu.slots))
            # ---- activate: weight -> KV switch
            t = time.perf_counter()
            inst, evicted, host_ms, kms = w.switch_memory(m)
            w.compute.synchronize()
            lat["promote"].append((time.perf_counter() - t) * 1e6)
            kernel_us.append(kms * 1e3)
            evicted_n.append(len(evicted))
            op("promote", w, model=m, evicted=evicted, weight_bytes=spec[m].weight_bytes,
               max_batch=spec[m].max_batch, required=w.slot(m).required_prewarm_layers)
            # ---- a short prefill on the fresh KV pool
            toks = torch.randint(0, w.models[m].cfg.vocab, (prompt,), dtype=torch.int32, device=f"cuda:{device}")
            t = time.perf_counter()
            with torch.cuda.stream(w.compute):
                s = w.open_seq(prompt)
                w.prefill(s, toks)
            w.compute.synchronize()
            lat["prefill"].append((time.perf_counter() - t) * 1e3)
            used_pages = w.gpu.counts().kv_pages_allocated
            w.close_seq(s)
            # ---- grace + reclaim: KV -> free pages (Eq. 1)
            inst.state = InstanceState.ACTIVE
            w.cluster.enter_grace(inst)
            op("grace", w, instance=inst.instance_id)
            inflight = rng.randint(0, 3)
            used = float(used_pages * M.PAGE) * rng.random()
            t = time.perf_counter()
            freed = w.reclaim(inflight, used)
            w.compute.synchronize()
            lat["reclaim"].append((time.perf_counter() - t) * 1e6)
            op("reclaim", w, inflight=inflight, max_batch=inst.max_batch, used=used, freed=freed)
            # ---- proactive prewarm of a non-resident model into the reclaimed pages
            missing = [c.name for c in cfgs if c.name not in w.gpu.slots]
            rng.shuffle(missing)
            for name in missing:
                if spec[name].partition_pages(M.PAGE) <= w.gpu.free_pages:
                    t = time.perf_counter()
                    prewarm(name)
                    lat["proactive_prewarm"].append((time.perf_counter() - t) * 1e3)
                    break
            # ---- release: KV pages back to free, slots kept
            t = time.perf_counter()
            w.cluster.release_instance(inst)
            w.compute.synchronize()
            lat["release"].append((time.perf_counter() - t) * 1e6)
            w.instance = None
            w.active_model = None
            op("release", w, instance=inst.instance_id)
            # keep every model reachable: re-prewarm evicted ones while pages allow
            for c in cfgs:
                if c.name not in w.gpu.slots and spec[c.name].partition_pages(M.PAGE) <= w.gpu.free_pages:
                    prewarm(c.name)
        host = w.gpu.owner_map()
        dev = np.empty_like(host)
        N.call("ws_pool_device_owner_map", w.gpu.pool, dev.ctypes.data_as(C.POINTER(C.c_int32)), dev.size)
        owner_map_equal = bool(np.array_equal(host, dev))
        N.call("ws_pool_sync_unmaps", w.gpu.pool)
        ti, mp, up = C.c_double(), C.c_double(), C.c_double()
        N.call("ws_pool_timing", w.gpu.pool, C.byref(ti), C.byref(mp), C.byref(up))
        return {
            "config": "BASELINE configs[2]: 4 models co-prewarmed on one B200, weight<->KV switch under burst",
            "models": [c.name for c in cfgs], "pool_pages": pool_pages, "switches": switches, "seed": seed,
            "switch_us": {k: {"p50": pct(v, 50), "p99": pct(v, 99), "max": max(v) if v else None, "n": len(v)}
                          for k, v in lat.items() if k in ("promote", "reclaim", "release")},
            "switch_kernel_us": {"p50": pct(kernel_us, 50), "p99": pct(kernel_us, 99)},
            "slots_evicted_per_promote_mean": sum(evicted_n) / max(1, len(evicted_n)),
            "prefill_ms": {"p50": pct(lat["prefill"], 50), "tokens": prompt},
            "proactive_prewarm_ms": {"p50": pct(lat["proactive_prewarm"], 50),
                                     "p99": pct(lat["proactive_prewarm"], 99), "n": len(lat["proactive_prewarm"])},
            "initial_prewarm_ms": prewarm_ms, "pool_init_s": init_s,
            "vmm_map_us_per_page": mp.value * 1e3, "vmm_unmap_us_per_page": up.value * 1e3,
            "device_owner_map_equals_ledger": owner_map_equal,
            "target_us": 1000.0,
        }
    finally:
        w.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--switches", type=int, default=1000)
    ap.add_argument("--pool-pages", type=int, default=32768)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    t0 = time.perf_counter()
    out = run_burst(a.switches, a.pool_pages, a.prompt, a.seed,
                    progress=lambda s: print(f"[{time.perf_counter() - t0:8.1f}s] {s}", file=sys.stderr, flush=True))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

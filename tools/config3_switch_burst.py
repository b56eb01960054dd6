"""BASELINE config 3: four models co-prewarmed on one B200, weight<->KV memory
switch under a seeded burst.

Llama-3-8B, Qwen2.5-7B, Mistral-7B and Phi-3-mini are prewarmed into four
slots of one device pool (real VMM pages, slot VAs, page window). The burst is
a seeded sequence of switches, each one:

  activate(m)   promote_to_dedicated: the other slots are evicted (pages to
                the free list now, VMM unmap on the background thread), every
                free page becomes KV via the switch kernel
  prefill       a short prompt on the paged pool (exercises the new KV pages)
  grace+reclaim reclaim_on_completion frees KV pages above Eq. 1's target
  proactive     begin_prewarm of another model into the reclaimed pages
                (Fig. 4b), weights copied from a device-resident image
  release       back to universal, holding m and the proactively loaded model

Every op's ledger is replayed on the reference-pinned oracle (oracle/ledger.py)
and compared (counts) plus device owner map == host ledger at the end.
Prints one JSON line with switch latency p50/p99 per op kind.

    python tools/config3_switch_burst.py [--switches 1000] [--pool-pages 40960]
"""

from __future__ import annotations

import argparse
import json
import random
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pct(xs, q):
    xs = sorted(xs)
    k = (len(xs) - 1) * q / 100.0
    f = int(k)
    c = min(f + 1, len(xs) - 1)
    return xs[f] + (xs[c] - xs[f]) * (k - f)


def main():
    import numpy as np
    import torch

    from oracle import ledger as OL
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.cluster import InstanceState, Role
    from paper_2512_09472_b200.weights import synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    ap = argparse.ArgumentParser()
    ap.add_argument("--switches", type=int, default=1000)
    ap.add_argument("--pool-pages", type=int, default=40960)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()

    cfgs = [M.LLAMA3_8B, M.QWEN25_7B, M.MISTRAL_7B, M.PHI3_MINI]
    t0 = time.perf_counter()
    w = UniversalWorker(0, pool_pages=a.pool_pages, max_tokens=max(a.prompt, 256), max_seqs=8)
    init_s = time.perf_counter() - t0
    src = {}
    for c in cfgs:
        src[c.name] = synth_flat(c, seed=1, device="cuda")  # device-resident image (stands in for a peer's HBM)
        w.register(c, None)
    torch.cuda.synchronize()
    # oracle ledger mirrors every op (counts parity)
    ol = OL.new_cluster(1, 1, a.pool_pages, M.PAGE)
    spec = {c.name: w.models[c.name].spec for c in cfgs}

    def oracle_check(tag):
        g = ol["gpus"][0]
        cnt = w.gpu.counts()
        got = (w.gpu.role.value, cnt.free_pages, cnt.kv_pages_mapped, cnt.kv_capacity_pages, cnt.kv_pages_used,
               sorted(w.gpu.slots))
        want = (g["role"], OL.free_pages(g), g["kv_mapped"], g["kv_cap"], g["kv_used"],
                sorted(s["model"] for s in g["slots"]))
        assert got == want, (tag, got, want)

    def prewarm(name):
        w.prewarm(name, layers=spec[name].layers, source=src[name])
        OL.begin_prewarm(ol, 0, name, spec[name].partition_pages(M.PAGE), max(1, spec[name].layers))
        oracle_check(f"prewarm {name}")

    prewarm_ms = []
    for c in cfgs:
        t = time.perf_counter()
        prewarm(c.name)
        prewarm_ms.append((time.perf_counter() - t) * 1e3)
    rng = random.Random(a.seed)
    lat = {"promote": [], "reclaim": [], "release": [], "prefill": [], "proactive_prewarm": []}
    kernel_us = []
    import ctypes as C

    from paper_2512_09472_b200 import _native as NN

    def progress(tag):
        rm, ru = C.c_int64(), C.c_int64()
        NN.call("ws_pool_map_stats", w.gpu.pool, C.byref(rm), C.byref(ru))
        print(f"[{time.perf_counter() - t0:8.1f}s] {tag}: remapped {rm.value} reused {ru.value} pages",
              file=sys.stderr, flush=True)

    progress(f"init {init_s:.1f}s, initial prewarm {[round(x) for x in prewarm_ms]} ms")
    for i in range(a.switches):
        if i % 10 == 0:
            progress(f"switch {i}")
        resident = sorted(w.gpu.slots)
        m = rng.choice(resident)
        # ---- activate: weight -> KV switch
        t = time.perf_counter()
        inst, evicted, host_ms, kms = w.switch_memory(m)
        w.compute.synchronize()
        lat["promote"].append((time.perf_counter() - t) * 1e6)
        kernel_us.append(kms * 1e3)
        OL.promote(ol, [0], m, 1, spec[m].weight_bytes, spec[m].max_batch, w.slot(m).required_prewarm_layers)
        oracle_check(f"promote {m}")
        # ---- a short prefill on the fresh KV pool
        prompt = torch.randint(0, w.models[m].cfg.vocab, (a.prompt,), dtype=torch.int32, device="cuda")
        t = time.perf_counter()
        with torch.cuda.stream(w.compute):
            s = w.open_seq(a.prompt)
            w.prefill(s, prompt)
        w.compute.synchronize()
        lat["prefill"].append((time.perf_counter() - t) * 1e3)
        used_pages = w.gpu.counts().kv_pages_allocated
        w.close_seq(s)
        # ---- grace + reclaim: KV -> free pages (Eq. 1)
        inst.state = InstanceState.ACTIVE
        w.cluster.enter_grace(inst)
        OL.enter_grace(ol, inst.instance_id)
        inflight = rng.randint(0, 3)
        used = float(used_pages * M.PAGE) * rng.random()
        t = time.perf_counter()
        freed = w.reclaim(inflight, used)
        w.compute.synchronize()
        lat["reclaim"].append((time.perf_counter() - t) * 1e6)
        assert freed == OL.reclaim(ol, 0, inflight, inst.max_batch, used)
        oracle_check("reclaim")
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
        OL.release(ol, inst.instance_id)
        oracle_check("release")
        # keep every model reachable: re-prewarm evicted ones while pages allow
        for c in cfgs:
            if c.name not in w.gpu.slots and spec[c.name].partition_pages(M.PAGE) <= w.gpu.free_pages:
                prewarm(c.name)
    N = __import__("paper_2512_09472_b200._native", fromlist=["x"])
    host = w.gpu.owner_map()
    dev = np.empty_like(host)
    import ctypes as C

    N.call("ws_pool_device_owner_map", w.gpu.pool, dev.ctypes.data_as(C.POINTER(C.c_int32)), dev.size)
    assert np.array_equal(host, dev), "device owner map diverged from the host ledger"
    N.call("ws_pool_sync_unmaps", w.gpu.pool)
    ti, mp, up = C.c_double(), C.c_double(), C.c_double()
    N.call("ws_pool_timing", w.gpu.pool, C.byref(ti), C.byref(mp), C.byref(up))
    out = {
        "config": "BASELINE configs[2]: 4 models co-prewarmed on one B200, weight<->KV switch under burst",
        "models": [c.name for c in cfgs], "pool_pages": a.pool_pages, "switches": a.switches,
        "switch_us": {k: {"p50": pct(v, 50), "p99": pct(v, 99), "n": len(v)} for k, v in lat.items()
                      if k in ("promote", "reclaim", "release")},
        "switch_kernel_us": {"p50": pct(kernel_us, 50), "p99": pct(kernel_us, 99)},
        "prefill_ms": {"p50": pct(lat["prefill"], 50), "tokens": a.prompt},
        "proactive_prewarm_ms": {"p50": pct(lat["proactive_prewarm"], 50), "n": len(lat["proactive_prewarm"])}
        if lat["proactive_prewarm"] else None,
        "initial_prewarm_ms": prewarm_ms, "pool_init_s": init_s,
        "vmm_map_us_per_page": mp.value * 1e3, "vmm_unmap_us_per_page": up.value * 1e3,
        "ledger_parity": "every op == oracle/ledger.py counts; device owner map == host ledger",
        "target_us": 1000.0,
    }
    print(json.dumps(out))
    w.close()


if __name__ == "__main__":
    main()

"""BASELINE config 5 on real workers: the reference engine's decision log
(tests/golden/config5_trace.json.gz, recorded by oracle/gen_config5_trace.py:
prewarmsim.engine on this framework's Cluster with B200-measured latency
terms) replayed op by op on real UniversalWorkers, one per logical GPU.

Per logical GPU, in the engine's order (one sequence counter over ops and
admissions):
  prewarm   UniversalWorker.prewarm(model, k, full) — background layer copies
            from pinned host memory over PCIe ("ready" at k, "full" at L)
  evict     UniversalWorker.evict(model) — in-flight copies fenced, pages freed
  promote   UniversalWorker.activate_instance(model, prompt) — memory switch,
            streaming of whatever is not resident, prefill of the instance's
            first request, first token to the host (cold or warm as it comes)
  admission a real prefill of the request's tokens on the active instance
            (device time, CUDA events)
  grace / release   enter_grace / release (KV pages back, slots kept)
  reclaim   UniversalWorker.reclaim(inflight, engine's KV bytes)
After every op the worker's ledger — role, free / KV-mapped / KV-capacity /
KV-used pages, resident slots in insertion order, evicted models, freed bytes
— must equal the engine's (exact).

Time is compressed: ops run back to back. The engine's gaps between a prewarm
and the next op on that GPU are >= seconds, so a background load that would
have finished by then is waited for first (``settle``). TTFT per request =
the engine's queueing + the measured startup of its instance (activation
TTFT minus a warm prefill of the same prompt) when it waited for the
activation + its measured prefill.

    python tools/config5_live.py [--policy warmserve] [--gpus 0,1,...]
"""

from __future__ import annotations

import argparse
import gzip
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
TRACE = ROOT / "tests" / "golden" / "config5_trace.json.gz"


def load_trace(path: Path = TRACE) -> dict:
    with gzip.open(path, "rt") as f:
        return json.load(f)


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = (len(xs) - 1) * q / 100.0
    f = int(k)
    c = min(f + 1, len(xs) - 1)
    return xs[f] + (xs[c] - xs[f]) * (k - f)


class HostImages:
    """Pinned host images of the config-5 models (seeded synthetic weights)."""

    def __init__(self, names, device: int, packed: bool = True):
        import torch

        from paper_2512_09472_b200 import models as M
        from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat

        self.cfgs = {n: M.ALL[n] for n in names}
        self.host, self.packed = {}, {}
        for i, n in enumerate(names):
            flat = synth_flat(self.cfgs[n], seed=100 + i, device=f"cuda:{device}")
            self.host[n] = pinned_host_copy(flat)
            if packed:  # the lossless packed stream cold activations use (bench e2e path)
                self.packed[n] = pack_stream(self.cfgs[n], flat)
            del flat
            torch.cuda.empty_cache()


def replay_gpu(trace: dict, policy: str, gid: int, device: int, images: HostImages, log=None) -> dict:
    import torch

    from paper_2512_09472_b200.cluster import InstanceState
    from paper_2512_09472_b200.worker import UniversalWorker

    pol = trace["policies"][policy]
    ops = [o for o in pol["ops"] if o["gpu"] == gid]
    adm = [a for a in pol["admissions"] if a["gpu"] == gid]
    events = sorted([(o["seq"], "op", o) for o in ops] + [(a["seq"], "adm", a) for a in adm], key=lambda e: e[0])
    first_act = {}
    for a in adm:
        if a["activation"] and a["instance"] not in first_act:
            first_act[a["instance"]] = a["request"]
    max_tok = max([a["tokens"] for a in adm] + [256])
    w = UniversalWorker(device, pool_pages=trace["pages_per_gpu"], max_tokens=max_tok)
    out = {"gpu": gid, "ops": len(ops), "admissions": len(adm), "ledger_checks": 0, "mismatches": [],
           "activations": [], "prefill_ms": {}, "startup_ms": {}, "op_us": {}}
    try:
        for n, host in images.host.items():
            w.register(images.cfgs[n], host)
            if n in images.packed:
                w.set_packed(n, images.packed[n])
        gen = torch.Generator().manual_seed(gid)
        prewarm_t = {}

        def check(o, extra=None):
            c = w.gpu.counts()
            got = [w.gpu.role.value, c.free_pages, c.kv_pages_mapped, c.kv_capacity_pages, c.kv_pages_used,
                   list(w.gpu.slots)]
            out["ledger_checks"] += 1
            if got != o["ledger"] or (extra and extra[0] != extra[1]):
                out["mismatches"].append({"seq": o["seq"], "op": o["op"], "got": got, "want": o["ledger"],
                                          "extra": extra})

        def settle(t):
            # compressed time: a background prewarm the engine would have
            # finished by trace time t is completed before the next op
            for name, t0 in list(prewarm_t.items()):
                if name in w.gpu.slots and t - t0 > 1000.0:
                    w.wait_resident(name)
                    del prewarm_t[name]

        def timed(kind, fn, sync=True):
            t0 = time.perf_counter()
            r = fn()
            if sync:
                torch.cuda.synchronize(device)
            out["op_us"].setdefault(kind, []).append((time.perf_counter() - t0) * 1e6)
            return r

        def prompt(n):
            return torch.randint(0, 32000, (n,), generator=gen, dtype=torch.int32).pin_memory()

        for _, kind, e in events:
            if kind == "adm":
                if first_act.get(e["instance"]) == e["request"]:
                    continue  # served by activate_instance (its prefill is in the activation's TTFT)
                p = prompt(e["tokens"])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(w.compute):
                    toks = p.to(f"cuda:{device}", non_blocking=True)
                    s = w.open_seq(e["tokens"] + 1)
                    e0.record(w.compute)
                    w.prefill(s, toks)
                    e1.record(w.compute)
                e1.synchronize()
                w.close_seq(s)
                out["prefill_ms"][e["request"]] = e0.elapsed_time(e1)
                continue
            o = e
            settle(o["t"])
            op = o["op"]
            if op == "prewarm":
                # host cost of the call (slot + copy queueing): the copies land
                # in the background, as the engine's prewarm does
                timed("prewarm_issue", lambda: w.prewarm(o["model"], layers=o["required"], full=True, wait=None),
                      sync=False)
                prewarm_t[o["model"]] = o["t"]
                check(o)
            elif op == "evict":
                timed("evict", lambda: w.evict(o["model"]))
                prewarm_t.pop(o["model"], None)
                check(o)
            elif op == "promote":
                req = first_act.get(o["instance"])
                n = next((a["tokens"] for a in adm if a["request"] == req), 64)
                p = prompt(n)
                slot = w.slot(o["model"])
                resident = w.residency(o["model"]) if slot is not None else 0
                r = w.activate_instance(o["model"], p, keep_seq=False)
                # warm prefill of the same prompt: the activation's startup is the rest
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(w.compute):
                    toks = p.to(f"cuda:{device}", non_blocking=True)
                    s = w.open_seq(n + 1)
                    e0.record(w.compute)
                    w.prefill(s, toks)
                    e1.record(w.compute)
                e1.synchronize()
                w.close_seq(s)
                warm_ms = e0.elapsed_time(e1)
                startup = max(0.0, r.ttft_ms - warm_ms)
                out["startup_ms"][o["instance"]] = startup
                if req is not None:
                    out["prefill_ms"][req] = warm_ms
                out["activations"].append({"instance": o["instance"], "model": o["model"], "warm": o["warm"],
                                           "layers_resident": resident, "ttft_ms": r.ttft_ms,
                                           "switch_us": r.switch_ms * 1e3, "streamed_layers": r.streamed_layers,
                                           "stream_ms": r.stream_ms, "startup_ms": startup, "tokens": n})
                check(o, ([m for _, m in r.evicted], [m for _, m in o["evicted"]]))
            elif op == "grace":
                if w.instance.state == InstanceState.STARTING:
                    w.instance.state = InstanceState.ACTIVE
                timed("grace", lambda: w.cluster.enter_grace(w.instance))
                check(o)
            elif op == "reclaim":
                freed = timed("reclaim", lambda: w.reclaim(o["inflight"], o["used"]))
                check(o, (freed, o["freed"]))
            elif op == "release":
                timed("release", lambda: w.release())
                check(o)
            else:
                raise ValueError(f"unknown op {op}")
            if log:
                log(f"gpu {gid} seq {o['seq']} {op} {o.get('model', '')}")
        return out
    finally:
        w.close()


def summarize(trace: dict, policy: str, results: list[dict]) -> dict:
    pol = trace["policies"][policy]
    prefill, startup, acts = {}, {}, []
    for r in results:
        prefill.update(r["prefill_ms"])
        startup.update({int(k): v for k, v in r["startup_ms"].items()})
        acts += r["activations"]
    gpus = {r["gpu"] for r in results}
    ttft = []
    for a in pol["admissions"]:
        if a["gpu"] not in gpus:
            continue
        t = a["queue_ms"] + prefill[a["request"]]
        if a["activation"]:
            t += startup[a["instance"]]
        ttft.append(t)
    engine_ttft = [a["ttft_ms"] for a in pol["admissions"] if a["gpu"] in gpus]
    op_us = {}
    for r in results:
        for k, v in r["op_us"].items():
            op_us.setdefault(k, []).extend(v)
    cold = [a for a in acts if not a["warm"]]
    warm = [a for a in acts if a["warm"]]
    return {
        "policy": policy, "gpus": sorted(gpus), "requests": len(ttft),
        "ledger_checks": sum(r["ledger_checks"] for r in results),
        "ledger_mismatches": sum(len(r["mismatches"]) for r in results),
        "first_mismatches": [m for r in results for m in r["mismatches"]][:5],
        "ttft_ms": {"p50": pct(ttft, 50), "p99": pct(ttft, 99), "mean": statistics.fmean(ttft) if ttft else None},
        "engine_modeled_ttft_ms": {"p50": pct(engine_ttft, 50), "p99": pct(engine_ttft, 99)},
        "activations": {"n": len(acts), "cold": len(cold), "warm": len(warm),
                        "cold_ttft_ms_p50": pct([a["ttft_ms"] for a in cold], 50),
                        "warm_ttft_ms_p50": pct([a["ttft_ms"] for a in warm], 50),
                        "startup_ms_p50": pct([a["startup_ms"] for a in acts], 50),
                        "startup_ms_p99": pct([a["startup_ms"] for a in acts], 99),
                        "switch_us_p50": pct([a["switch_us"] for a in acts], 50),
                        "switch_us_p99": pct([a["switch_us"] for a in acts], 99)},
        "op_us": {k: {"p50": pct(v, 50), "p99": pct(v, 99), "n": len(v)} for k, v in op_us.items()},
        "prefill_ms_p50": pct(list(prefill.values()), 50),
    }


def run_live(policy: str = "warmserve", gpus=None, device: int = 0, trace=None, images=None, log=None) -> dict:
    trace = trace or load_trace()
    gpus = list(range(trace["gpus"])) if gpus is None else list(gpus)
    if images is None:
        images = HostImages(sorted(trace["models"]), device)
    t0 = time.perf_counter()
    results = [replay_gpu(trace, policy, g, device, images, log) for g in gpus]
    out = summarize(trace, policy, results)
    out["wall_s"] = time.perf_counter() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--policy", default="warmserve,no_prewarm")
    ap.add_argument("--gpus", default="")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args()
    trace = load_trace()
    gpus = [int(x) for x in a.gpus.split(",") if x] or None
    images = HostImages(sorted(trace["models"]), a.device)
    for pol in a.policy.split(","):
        print(json.dumps(run_live(pol, gpus, a.device, trace, images)), flush=True)


if __name__ == "__main__":
    main()

"""Record BASELINE config 5's decision log for the live replay (test/bench
infrastructure; imports the unmodified reference from /root/reference, so it
runs only in the build container).

The reference's own event loop, placement and autoscaler
(prewarmsim.engine.Simulation, engine.py:168-998) run the config-5 trace
(tools/config5_replay.build_config5: 8 universal workers, periodic
4-model trace) on this framework's Cluster with the B200-measured latency
terms (engine_adapter.run_measured). A recording subclass of the Cluster logs
every top-level ledger op the engine issues — begin_prewarm
(engine.py:889-892), evict_slot (engine.py:612, 727), promote_to_dedicated
(engine.py:283, 499), enter_grace (engine.py:695), reclaim_on_completion
(engine.py:374), release_instance (engine.py:721) — with the engine clock, its
arguments, its result (evicted pairs, freed bytes) and the GPU's ledger right
after it (role, free / KV-mapped / KV-capacity / KV-used pages, resident slots
in insertion order). Every admission (engine.py:330-348) is logged with its
instance and the TTFT phases the engine assigns.

tools/config5_live.py replays each GPU's ops on a real UniversalWorker and
checks the worker's ledger against these snapshots after every op.

    python oracle/gen_config5_trace.py [--pages-per-gpu 76800] [--days 3]
      -> tests/golden/config5_trace.json.gz
"""

from __future__ import annotations

import argparse
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")


def main():
    from config5_replay import build_config5

    from paper_2512_09472_b200 import cluster as ours
    from paper_2512_09472_b200.engine_adapter import Measured, run_measured

    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default=str(ROOT / "profiles" / "r2a_bench_session_start.json"))
    ap.add_argument("--days", type=int, default=3)
    # 150 GiB of 2 MiB pages: a universal worker's pool fits one B200 next to
    # its workspace (the model images stay in pinned host memory)
    ap.add_argument("--pages-per-gpu", type=int, default=76_800)
    ap.add_argument("--policies", default="warmserve,no_prewarm")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "config5_trace.json.gz"))
    a = ap.parse_args()

    engine, cfg, reqs, shapes = build_config5(a.days, a.pages_per_gpu)
    measured = Measured.from_bench(json.loads(Path(a.bench).read_text()))
    ops, admits = [], []
    state = {"sim": None, "depth": 0, "seq": 0}

    def snap(cl, gid):
        g = cl.gpu(gid)
        c = g.counts()
        return [g.role.value, c.free_pages, c.kv_pages_mapped, c.kv_capacity_pages, c.kv_pages_used, list(g.slots)]

    class Recording(ours.Cluster):
        def _rec(self, kind, gid, **kw):
            if state["depth"] == 1:  # top-level engine calls only
                ops.append({"seq": state["seq"], "t": state["sim"].now if state["sim"] else 0.0, "op": kind,
                            "gpu": gid, **kw, "ledger": snap(self, gid)})
                state["seq"] += 1

        def begin_prewarm(self, gpu, spec, pages, required_layers):
            state["depth"] += 1
            try:
                slot = super().begin_prewarm(gpu, spec, pages, required_layers)
                self._rec("prewarm", gpu.gpu_id, model=spec.model_id, pages=pages, required=required_layers)
                return slot
            finally:
                state["depth"] -= 1

        def evict_slot(self, gpu, model_id):
            state["depth"] += 1
            try:
                slot = super().evict_slot(gpu, model_id)
                if slot is not None:
                    self._rec("evict", gpu.gpu_id, model=model_id)
                return slot
            finally:
                state["depth"] -= 1

        def promote_to_dedicated(self, gpu_ids, spec, required_layers):
            state["depth"] += 1
            try:
                assert len(gpu_ids) == 1, "config 5 models run on one GPU each"
                warm = spec.model_id in self.gpu(gpu_ids[0]).slots
                inst, evicted = super().promote_to_dedicated(gpu_ids, spec, required_layers)
                self._rec("promote", gpu_ids[0], model=spec.model_id, required=required_layers, warm=warm,
                          instance=inst.instance_id, max_batch=inst.max_batch,
                          evicted=[list(e) for e in evicted])
                return inst, evicted
            finally:
                state["depth"] -= 1

        def enter_grace(self, inst):
            state["depth"] += 1
            try:
                super().enter_grace(inst)
                self._rec("grace", inst.gpu_ids[0], instance=inst.instance_id)
            finally:
                state["depth"] -= 1

        def reclaim_on_completion(self, gpu, inflight, max_batch, kv_used_bytes):
            state["depth"] += 1
            try:
                freed = super().reclaim_on_completion(gpu, inflight, max_batch, kv_used_bytes)
                self._rec("reclaim", gpu.gpu_id, inflight=inflight, max_batch=max_batch, used=kv_used_bytes,
                          freed=freed, instance=gpu.instance_id)
                return freed
            finally:
                state["depth"] -= 1

        def release_instance(self, inst):
            state["depth"] += 1
            try:
                out = super().release_instance(inst)
                self._rec("release", inst.gpu_ids[0], instance=inst.instance_id)
                return out
            finally:
                state["depth"] -= 1

    sim_cls = engine.Simulation
    orig_init, orig_admit = sim_cls.__init__, sim_cls._admit

    def init(self, *args, **kw):
        orig_init(self, *args, **kw)
        state["sim"] = self

    def admit(self, rs, inst, t, activation):
        orig_admit(self, rs, inst, t, activation)
        admits.append({"seq": state["seq"], "t": t, "request": rs.req.id, "model": rs.req.model_id, "instance": inst.instance_id,
                       "gpu": inst.gpu_ids[0], "activation": activation, "tokens": rs.req.input_tokens})
        state["seq"] += 1

    out = {
        "what": "BASELINE configs[4] decision logs: the reference engine (prewarmsim.engine) on this framework's "
                "Cluster with B200-measured latency terms; every top-level ledger op with the ledger after it, "
                "every admission with its TTFT phases; ops and admissions share one sequence counter",
        "generator": "oracle/gen_config5_trace.py", "days": a.days, "gpus": 8, "pages_per_gpu": a.pages_per_gpu,
        "page_size": 2 * 1024 * 1024, "measured_inputs": measured.__dict__,
        "models": {n: {"layers": s.layers, "weight_bytes": s.layout().total} for n, s in shapes.items()},
        "ledger_fields": ["role", "free_pages", "kv_pages_mapped", "kv_capacity_pages", "kv_pages_used", "slots"],
        "policies": {},
    }
    sim_cls.__init__, sim_cls._admit = init, admit
    try:
        for policy in a.policies.split(","):
            ops.clear()
            admits.clear()
            state.update(sim=None, depth=0, seq=0)
            report = run_measured(engine, cfg, reqs, policy, measured, shapes, cluster_cls=Recording)
            recs = {r.request_id: r for r in report.records}
            for ad in admits:
                r = recs[ad["request"]]
                ad.update(queue_ms=r.queue_ms, startup_ms=r.startup_ms, load_stall_ms=r.load_stall_ms,
                          prefill_ms=r.prefill_ms, ttft_ms=r.ttft_ms)
            out["policies"][policy] = {"ops": list(ops), "admissions": list(admits),
                                       "summary": report.overall_summary(),
                                       "invariant_violations": len(report.invariant_violations)}
            kinds = {}
            for o in ops:
                kinds[o["op"]] = kinds.get(o["op"], 0) + 1
            sm = report.overall_summary()["ttft_ms"]
            print(f"{policy}: {len(ops)} ops {kinds}, {len(admits)} admissions, ttft p50/p99 "
                  f"{sm['p50']:.2f}/{sm['p99']:.2f} ms")
    finally:
        sim_cls.__init__, sim_cls._admit = orig_init, orig_admit
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    with gzip.open(a.out, "wt") as f:
        json.dump(out, f)
    print("wrote", a.out)


if __name__ == "__main__":
    main()

"""TEST INFRASTRUCTURE ONLY — generate golden vectors by running the REFERENCE.

Run in the build container (where ``/root/reference`` exists):

    python oracle/gen_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``) and
its own test helpers (``pkg/tests/lifecycle_walker.py``, ``conftest.py``) and
records, for every Cluster operation issued by (a) the reference's randomized
lifecycle walks, (b) the reference engine on the reference's own desk and
acceptance workloads, and (c) the config-3 page-scale scenario, the full page
ledger after the op, its return value, its error text and its role transitions.
It also records the planning math (cluster.py:145-197, memswitch.py:59-122) on
grids that include every known-answer value of the reference tests.

Outputs (committed, small): ``tests/golden/ledger_traces.json.gz`` and
``tests/golden/plan_math.json``. Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import gzip
import json
import math
import os
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import prewarmsim.cluster as rc  # noqa: E402
import prewarmsim.engine as reng  # noqa: E402
import prewarmsim.memswitch as rms  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
PAGE = 2 * 1024 * 1024
GIB = 1024**3


def _snap(cl):
    out = []
    for g in cl.gpus:
        out.append(
            [
                g.role.value,
                g.free_pages,
                g.kv_pages_mapped,
                g.kv_pages_used,
                g.kv_capacity_pages,
                g.instance_id,
                [[s.model_id, s.slot_id, s.mapped_pages, bool(s.active)] for s in g.slots.values()],
            ]
        )
    return out


class Recorder:
    """Wraps the reference Cluster class; logs top-level ops only."""

    traces: list = []

    @classmethod
    def make_class(cls):
        rec = cls

        class RecordingCluster(rc.Cluster):
            def __init__(self, n_servers, gpus_per_server, pages_per_gpu, page_size, bandwidth):
                super().__init__(n_servers, gpus_per_server, pages_per_gpu, page_size, bandwidth)
                self._depth = 0
                self._roles = []
                self._trace = dict(
                    init=[n_servers, gpus_per_server, pages_per_gpu, page_size, bandwidth],
                    ops=[],
                )
                rec.traces.append(self._trace)

            def _set_role(self, gpu, new):
                old = gpu.role
                super()._set_role(gpu, new)
                if old != new:
                    self._roles.append([gpu.gpu_id, old.value, new.value])

            def _run(self, entry, fn):
                top = self._depth == 0
                self._depth += 1
                if top:
                    self._roles = []
                try:
                    ret = fn()
                    if top:
                        entry["ret"] = _ret(ret)
                    return ret
                except rc.ClusterError as e:
                    if top:
                        entry["err"] = str(e)
                    raise
                except ValueError as e:
                    if top:
                        entry["err"] = "ValueError: " + str(e)
                    raise
                finally:
                    self._depth -= 1
                    if top:
                        entry["roles"] = self._roles
                        entry["state"] = _snap(self)
                        self._trace["ops"].append(entry)

            def begin_prewarm(self, gpu, spec, pages, required_layers):
                e = dict(op="begin_prewarm", gpu=gpu.gpu_id, model=spec.model_id, pages=pages,
                         required=required_layers)
                return self._run(e, lambda: super(RecordingCluster, self).begin_prewarm(
                    gpu, spec, pages, required_layers))

            def evict_slot(self, gpu, model_id):
                e = dict(op="evict_slot", gpu=gpu.gpu_id, model=model_id)
                return self._run(e, lambda: super(RecordingCluster, self).evict_slot(gpu, model_id))

            def promote_to_dedicated(self, gpu_ids, spec, required_layers):
                e = dict(op="promote", gpus=list(gpu_ids), model=spec.model_id,
                         weight=spec.weight_bytes, parallelism=spec.parallelism,
                         max_batch=spec.max_batch, layers=spec.layers, required=required_layers)
                return self._run(e, lambda: super(RecordingCluster, self).promote_to_dedicated(
                    gpu_ids, spec, required_layers))

            def enter_grace(self, inst):
                e = dict(op="enter_grace", inst=inst.instance_id)
                return self._run(e, lambda: super(RecordingCluster, self).enter_grace(inst))

            def reclaim_on_completion(self, gpu, inflight, max_batch, kv_used_bytes):
                e = dict(op="reclaim", gpu=gpu.gpu_id, inflight=inflight, max_batch=max_batch,
                         used=float(kv_used_bytes))
                return self._run(e, lambda: super(RecordingCluster, self).reclaim_on_completion(
                    gpu, inflight, max_batch, kv_used_bytes))

            def release_instance(self, inst):
                e = dict(op="release", inst=inst.instance_id, inflight=len(inst.inflight))
                return self._run(e, lambda: super(RecordingCluster, self).release_instance(inst))

        return RecordingCluster


def _ret(ret):
    if ret is None:
        return None
    if isinstance(ret, rc.PrewarmSlot):
        return ret.slot_id
    if isinstance(ret, tuple) and len(ret) == 2 and isinstance(ret[0], rc.Instance):
        return [ret[0].instance_id, [list(p) for p in ret[1]]]
    if isinstance(ret, int):
        return ret
    if isinstance(ret, list):
        return [g.gpu_id for g in ret]
    raise TypeError(type(ret))


def gen_walks(RC, n, base_seed):
    import lifecycle_walker as lw

    lw.Cluster = RC
    start = len(Recorder.traces)
    lw.run_walks(n_sequences=n, base_seed=base_seed)
    for t in Recorder.traces[start:]:
        t["name"] = "walk"
    return Recorder.traces[start:]


def gen_engine(RC):
    from conftest import desk_config, desk_model, periodic_trace
    from prewarmsim.trace import Request

    reng.Cluster = RC

    def merge(*parts):
        merged = sorted((r for p in parts for r in p), key=lambda r: r.arrival)
        return [Request(f"r{i:06d}", r.model_id, r.arrival, r.input_tokens, r.output_tokens)
                for i, r in enumerate(merged)]

    runs = []
    # Light load — test_acceptance.py:336-347
    ma, mb = desk_model("a", initial_instances=1), desk_model("b", initial_instances=1)
    cfg = desk_config([ma, mb])
    cfg.cluster.gpus_per_server = 8
    reqs = merge(periodic_trace("a", 3, cfg.sim.day_ms, 60_000, (1, 3, 5, 7), 2, ma, slack_ms=700.0),
                 periodic_trace("b", 3, cfg.sim.day_ms, 60_000, (2, 3, 4), 3, mb, slack_ms=700.0))
    runs.append(("engine_light_warmserve", cfg, reqs, "warmserve"))
    # Heavy load — test_acceptance.py:349-359
    models = [desk_model(m) for m in "abcd"]
    cfg = desk_config(models)
    cfg.cluster.gpus_per_server = 3
    windows = {"a": (0, 1, 4, 5), "b": (2, 3), "c": (6, 7), "d": (8, 9)}
    reqs = merge(*[periodic_trace(m.model_id, 3, cfg.sim.day_ms, 60_000, windows[m.model_id], 3, m,
                                  slack_ms=700.0) for m in models])
    for pol in ("warmserve", "sllm_gpu", "no_prewarm"):
        runs.append((f"engine_heavy_{pol}", cfg, reqs, pol))
    # Grace reclaim with long decodes — test_engine.py:401-421
    cfg = desk_config([desk_model(initial_instances=2)])
    reqs = [Request("r0", "s", 0.0, 16, 2000), Request("r1", "s", 1.0, 16, 2000)]
    runs.append(("engine_grace", cfg, reqs, "warmserve"))
    out = []
    for name, cfg, reqs, pol in runs:
        start = len(Recorder.traces)
        rep = reng.run(cfg, reqs, pol)
        assert not rep.invariant_violations, name
        for t in Recorder.traces[start:]:
            t["name"] = name
            out.append(t)
    return out


def gen_scenarios(RC):
    """Hand-written sequences: the reference KAT ledger cases
    (test_cluster.py:124-328) plus the config-3 page-scale scenario."""
    out = []

    def spec(mid, weight, par=1, layers=4, **kw):
        return rc.ModelSpec(mid, weight, par, layers=layers, **kw)

    def attempt(fn):
        try:
            return fn()
        except (rc.ClusterError, ValueError):
            return None

    # KAT ledger — test_cluster.py:124-328 (page_size 1, 1000 pages)
    cl = RC(1, 4, 1000, 1, 1.0)
    a, b = spec("a", 950), spec("b", 100)
    cl.begin_prewarm(cl.gpu(0), a, 950, 1)
    attempt(lambda: cl.begin_prewarm(cl.gpu(0), b, 100, 1))  # insufficient pages
    attempt(lambda: cl.begin_prewarm(cl.gpu(0), a, 10, 1))  # already holds
    cl.evict_slot(cl.gpu(0), "a")
    cl.begin_prewarm(cl.gpu(0), spec("a", 100), 100, 1)
    cl.begin_prewarm(cl.gpu(0), spec("b", 200), 200, 1)
    inst, _ = cl.promote_to_dedicated((0,), spec("a", 100), 1)
    attempt(lambda: cl.begin_prewarm(cl.gpu(0), spec("c", 10), 10, 1))  # dedicated
    attempt(lambda: cl.evict_slot(cl.gpu(0), "a"))  # active slot
    attempt(lambda: cl.promote_to_dedicated((0,), spec("b", 10), 1))  # dedicated to instance
    s4 = spec("q", 400, par=4)
    for gid in (1, 2):
        cl.begin_prewarm(cl.gpu(gid), s4, 100, 1)
    attempt(lambda: cl.promote_to_dedicated((1, 2, 3), s4, 1))  # needs 4 GPUs
    attempt(lambda: cl.release_instance(inst))  # not in grace
    cl.enter_grace(inst)
    inst.inflight.add("r1")
    attempt(lambda: cl.release_instance(inst))  # inflight
    inst.inflight.clear()
    attempt(lambda: cl.reclaim_on_completion(cl.gpu(1), 0, 4, 0))  # not draining
    for inflight, used in zip(range(7, -1, -1), [500, 380, 240, 140, 60, 20, 10, 0]):
        cl.reclaim_on_completion(cl.gpu(0), min(inflight, 32), 32, used)
    cl.begin_prewarm(cl.gpu(0), spec("z", 200), 200, 1)  # proactive prewarm into freed KV
    cl.release_instance(inst)
    cl.promote_to_dedicated((0,), spec("z", 200), 1)
    Recorder.traces[-1]["name"] = "kat_ledger"
    out.append(Recorder.traces[-1])

    cl = RC(2, 2, 1000, 1, 1.0)
    attempt(lambda: cl.promote_to_dedicated((1, 2), spec("a", 100, par=2), 1))  # one server
    attempt(lambda: cl.promote_to_dedicated((0,), spec("a", 100, par=1), 1))
    Recorder.traces[-1]["name"] = "kat_servers"
    out.append(Recorder.traces[-1])

    # Config 3: one B200 of 89,600 2 MiB pages, four
    # co-prewarmed 7-8B models, promote Mistral, drain with a reclaim sequence.
    models = {
        "llama3-8b": 16_060_522_496,
        "qwen2.5-7b": 15_231_233_024,
        "mistral-7b": 14_483_464_192,
        "phi3-mini": 7_642_159_104,
    }
    cl = RC(1, 8, 89_600, PAGE, 128 * GIB / 1000.0)
    specs = {m: spec(m, w, layers=32, max_batch=32) for m, w in models.items()}
    for m, s in specs.items():
        cl.begin_prewarm(cl.gpu(0), s, s.partition_pages(PAGE), 1)
    inst, _ = cl.promote_to_dedicated((0,), specs["mistral-7b"], 1)
    inst.state = rc.InstanceState.ACTIVE
    cl.enter_grace(inst)
    for inflight, used in [(31, 60 * GIB), (8, 10 * GIB), (1, 1 * GIB), (0, 0.0)]:
        cl.reclaim_on_completion(cl.gpu(0), inflight, 32, float(used))
    cl.begin_prewarm(cl.gpu(0), specs["llama3-8b"], specs["llama3-8b"].partition_pages(PAGE), 1)
    cl.release_instance(inst)
    # Switch burst: seeded promote/reclaim/release cycle over the 4 models.
    rng = random.Random(7)
    for _ in range(60):
        g = cl.gpu(rng.randrange(8))
        if g.role == rc.Role.IDLE or g.role == rc.Role.UNIVERSAL:
            m = rng.choice(sorted(specs))
            if m not in g.slots and g.role == rc.Role.UNIVERSAL:
                if attempt(lambda: cl.begin_prewarm(g, specs[m], specs[m].partition_pages(PAGE), 1)) is None:
                    continue
                continue
            inst, _ = cl.promote_to_dedicated((g.gpu_id,), specs[m], 1)
            inst.state = rc.InstanceState.ACTIVE
        elif g.role == rc.Role.DEDICATED:
            cl.enter_grace(cl.instances[g.instance_id])
        else:
            inst = cl.instances[g.instance_id]
            cap = g.kv_capacity_pages * PAGE
            used = rng.uniform(0, cap)
            cl.reclaim_on_completion(g, rng.randint(0, 32), 32, used)
            if rng.random() < 0.5:
                cl.release_instance(inst)
    Recorder.traces[-1]["name"] = "config3"
    out.append(Recorder.traces[-1])
    return out


def gen_math():
    """Planning math on grids that include every reference KAT input."""
    rows = dict(required=[], stall=[], reservation=[], pipeline=[], kvmap=[], pages=[])
    # required_prewarm_layers / catchup_stall: test_cluster.py:29-85 style grid
    for layers in (1, 2, 3, 4, 5, 8, 13, 28, 32, 40, 80):
        for ratio in (0.1, 0.5, 1.0, 1.7, 2.0, 3.5, 10.0, 28.7):
            t_comp = 40.0
            weight = int(ratio * t_comp * layers)
            s = rc.ModelSpec("m", max(weight, 1), 1, layers=layers, prefill_a_ms=0.0,
                             prefill_b_ms=t_comp * layers)
            for bw in (1.0, 3.0, 1e12):
                k = rc.required_prewarm_layers(s, bw)
                rows["required"].append([s.weight_bytes, 1, layers, 0.0, t_comp * layers, bw, 512, k])
                for m in sorted({0, 1, k - 1, k, layers // 2, layers}):
                    if m < 0:
                        continue
                    st = rc.catchup_stall_ms(s, m, bw)
                    rows["stall"].append([s.weight_bytes, 1, layers, 0.0, t_comp * layers, m, bw, 512, st])
    # Real shapes with the reference's default prefill coefficients
    shapes = [(16_060_522_496, 32), (15_231_233_024, 28), (14_483_464_192, 32),
              (7_642_159_104, 32), (141_107_412_992, 80), (7_340_032, 2)]
    for w, L in shapes:
        for par in (1, 2, 4, 8):
            for bw_gbs in (31.25, 55.0, 64.0, 128.0, 750.0, 900.0):
                bw = bw_gbs * GIB / 1000.0
                for a, b, tok in ((0.1, 5.0, 512), (0.0104, 1.0, 2048), (0.3, 11.4, 512)):
                    s = rc.ModelSpec("m", w, par, layers=L, prefill_a_ms=a, prefill_b_ms=b)
                    k = rc.required_prewarm_layers(s, bw, tok)
                    rows["required"].append([w, par, L, a, b, bw, tok, k])
                    for m in sorted({1, 4, k, L}):
                        rows["stall"].append([w, par, L, a, b, m, bw, tok,
                                              rc.catchup_stall_ms(s, m, bw, tok)])
            rows["pages"].append([w, par, PAGE, s.partition_bytes, s.partition_pages(PAGE), s.layer_bytes])
    # reservation_target: test_cluster.py:88-121 and Eq. 1 grid
    GB = 10**9
    rng = random.Random(11)
    for m, c, r, k in [(100 * GB, 32, 8, 20 * GB), (100 * GB, 32, 0, 0), (100 * GB, 32, 32, 40 * GB),
                       (100.0, 32, 8, 20.0)]:
        rows["reservation"].append([m, c, r, k, rc.reservation_target(m, c, r, k)])
    for _ in range(400):
        m = float(rng.randrange(1, 90_000) * PAGE)
        c = rng.randint(1, 256)
        r = rng.randint(0, c)
        k = rng.uniform(0, m)
        rows["reservation"].append([m, c, r, k, rc.reservation_target(m, c, r, k)])
    # pipelined_load: test_memswitch.py:38-114 inputs + random grid
    mu_cal = 0.0390625
    bw128 = 128 * GIB / 1000.0
    bwdy = float(2**25)
    cases = [(1024 * PAGE, bwdy, mu_cal, 64), (10 * GIB, bw128, mu_cal, 64), (32 * PAGE, bwdy, mu_cal, 64),
             (100 * PAGE + 12345, bw128, mu_cal, 64), (777 * PAGE, bw128, mu_cal, 16),
             (4096 * PAGE, bwdy, mu_cal, 64), (4096 * PAGE, bwdy, 0.0, 64),
             (16_060_522_496, bw128, mu_cal, 64), (16_060_522_496, bw128, mu_cal, 1)]
    for _ in range(300):
        pages = rng.randint(1, 4096)
        cases.append((pages * PAGE - rng.choice([0, 0, 1, 12345]), rng.uniform(0.5, 200.0) * PAGE,
                      rng.uniform(0.001, 0.5), rng.randint(1, 256)))
    for total, bw, mu, chunk in cases:
        p = rms.pipelined_load(total, bw, mu, chunk, PAGE)
        rows["pipeline"].append([total, bw, mu, chunk, PAGE, p.n_chunks, p.first_chunk_map_ms,
                                 p.finish_ms, p.critical_path_stall_ms])
    # background_kv_mapping: test_memswitch.py:142-171
    for pages, mu, rate in [(1000, 0.5, 1.0), (1000, 1.0, 1.0), (50, 2.0, 1.0)]:
        rows["kvmap"].append([pages, mu, rate, rms.background_kv_mapping(pages, mu, rate)])
    for _ in range(200):
        pages, mu, rate = rng.randint(0, 90_000), rng.uniform(0.001, 4.0), rng.uniform(0.05, 30.0)
        rows["kvmap"].append([pages, mu, rate, rms.background_kv_mapping(pages, mu, rate)])
    return rows


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    RC = Recorder.make_class()
    traces = []
    traces += gen_scenarios(RC)
    traces += gen_walks(RC, 300, 1234)
    traces += gen_engine(RC)
    traces = [t for t in traces if t["ops"]]
    n_ops = sum(len(t["ops"]) for t in traces)
    with gzip.open(OUT / "ledger_traces.json.gz", "wt") as f:
        json.dump(dict(source="prewarmsim 0.1.0 (/root/reference/pkg), oracle/gen_golden.py",
                       traces=traces), f, separators=(",", ":"))
    with open(OUT / "plan_math.json", "w") as f:
        json.dump(gen_math(), f, separators=(",", ":"))
    print(f"wrote {len(traces)} traces / {n_ops} ops and plan math to {OUT}")


if __name__ == "__main__":
    main()

"""BASELINE config 5: 8 universal workers, synthetic periodic multi-model
trace, TTFT p50/p99 and switch latency — the reference's modeled CPU path vs
the same engine driven by B200-measured latencies on this framework's Cluster.

Runs in the build container (needs /root/reference for the engine):

    python tools/config5_replay.py [--bench profiles/r1_bench_latest.json]

Writes profiles/r1_config5_replay.json.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")


def build_config5(days: int = 3, pages_per_gpu: int = 89_600):
    """The config-5 experiment: 8 universal workers (1 server x 8 GPUs), four
    models with reference-style modeled specs, a periodic 4-model trace
    (conftest.periodic_trace). Returns (engine module, cfg, requests, shapes)."""
    import prewarmsim.engine as engine
    from conftest import periodic_trace
    from prewarmsim.cluster import ModelSpec
    from prewarmsim.config import ClusterConfig, ExperimentConfig, LatencyConfig, PredictorConfig, SimConfig
    from prewarmsim.autoscaler import ScalePolicy
    from prewarmsim.trace import Request

    from paper_2512_09472_b200 import models as M

    shapes = {m.name: m for m in (M.LLAMA3_8B, M.QWEN25_7B, M.MISTRAL_7B, M.PHI3_MINI)}
    PAGE = 2 * 1024 * 1024
    # Reference-style modeled specs (table1_example.toml calibration style):
    # prefill a*tokens + b, decode c, default warm/cold start constants.
    specs = [ModelSpec(n, s.layout().total, 1, max_batch=16, layers=s.layers, prefill_a_ms=0.06 * s.layout().total / 16e9,
                       prefill_b_ms=5.0, decode_c_ms=20.0, kv_bytes_per_token=s.kv_geometry()[1])
             for n, s in shapes.items()]
    cfg = ExperimentConfig(
        seed=5, policy="warmserve",
        cluster=ClusterConfig(servers=1, gpus_per_server=8, page_size_bytes=PAGE, pages_per_gpu=pages_per_gpu,
                              h2d_gib_per_s=128.0),
        predictor=PredictorConfig(window_ms=60_000, seasonal_days=2),
        scaler=ScalePolicy(check_interval_ms=10_000.0, scale_down_utilization_threshold=0.5, sustain_windows=2),
        latency=LatencyConfig(warm_start_ms=500.0, cold_extra_ms=1500.0),
        sim=SimConfig(day_ms=600_000, drain_timeout_ms=120_000.0),
        models=specs)
    windows = {"llama3-8b": (0, 1, 4, 5), "qwen2.5-7b": (2, 3, 6), "mistral-7b": (5, 6, 7), "phi3-mini": (1, 8, 9)}
    parts = [periodic_trace(s.model_id, days, cfg.sim.day_ms, 60_000, windows[s.model_id], 6, s, slack_ms=400.0)
             for s in specs]
    merged = sorted((r for p in parts for r in p), key=lambda r: r.arrival)
    reqs = [Request(f"r{i:06d}", r.model_id, r.arrival, r.input_tokens, r.output_tokens) for i, r in enumerate(merged)]
    return engine, cfg, reqs, shapes


def main():
    from paper_2512_09472_b200.engine_adapter import Measured, run_measured

    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default=str(ROOT / "profiles" / "r1_bench_latest.json"))
    ap.add_argument("--config3", default=str(ROOT / "profiles" / "r1_config3_switch_burst_1000.json"))
    ap.add_argument("--days", type=int, default=3)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r1_config5_replay.json"))
    ap.add_argument("--artifacts", default=str(ROOT / "profiles" / "r1_config5_artifacts"),
                    help="reference-format requests.csv / decisions.jsonl (metrics.py:137-242) per arm")
    a = ap.parse_args()
    bench = json.loads(Path(a.bench).read_text())
    c3 = json.loads(Path(a.config3).read_text()) if Path(a.config3).exists() else None
    measured = Measured.from_bench(bench, c3)
    engine, cfg, reqs, shapes = build_config5(a.days)

    out = {"config": "BASELINE configs[4]: 8 universal workers, periodic 4-model trace",
           "requests": len(reqs), "measured_inputs": measured.__dict__, "policies": {}}
    for policy in ("warmserve", "sllm_gpu", "no_prewarm"):
        row = {}
        t0 = time.perf_counter()
        ref = engine.run(cfg, reqs, policy)
        row["reference_modeled"] = _summ(ref, time.perf_counter() - t0)
        t0 = time.perf_counter()
        ours = run_measured(engine, cfg, reqs, policy, measured, shapes)
        row["b200_measured"] = _summ(ours, time.perf_counter() - t0)
        if policy == "warmserve" and a.artifacts:
            # the reference's own artifact writer on both arms: byte-comparable formats
            row["artifacts"] = {
                "reference_modeled": [_rel(p) for p in
                                      ref.write_artifacts(Path(a.artifacts) / "reference_modeled")],
                "b200_measured": [_rel(p) for p in
                                  ours.write_artifacts(Path(a.artifacts) / "b200_measured")]}
        out["policies"][policy] = row
        print(policy, json.dumps(row), flush=True)
    Path(a.out).write_text(json.dumps(out, indent=1))
    print("wrote", a.out)


def _rel(p):
    p = Path(p).resolve()
    return str(p.relative_to(ROOT)) if p.is_relative_to(ROOT) else str(p)


def _summ(report, wall_s):
    s = report.overall_summary()
    ups = [x for x in report.audit if x["kind"] == "scale_up"]
    startup = sorted(x["startup_ms"] for x in ups)
    return {"ttft_ms": s["ttft_ms"], "hit_ratio": report.hit_ratio, "scale_ups": len(ups),
            "startup_ms_p50": startup[len(startup) // 2] if startup else None,
            "invariant_violations": len(report.invariant_violations), "sim_wall_s": round(wall_s, 3)}


if __name__ == "__main__":
    main()

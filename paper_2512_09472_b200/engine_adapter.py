"""Measured-latency engine adapter (BASELINE config 5).

Runs the reference's own event loop, placement and autoscaler
(``prewarmsim.engine`` — passed in, never imported by the product) on top of
this framework's ``Cluster`` with every latency term replaced by a number
measured on the B200 worker:

  reference term (engine.py)                    measured replacement
  LatencyModel.prefill_ms  a*tokens + b (97-108) warm prefill per token (bench value)
  LatencyModel.tpot_ms     c (110-113)           decode step (measured or HBM-bound)
  warm_start_ms            constant (557)        memory-switch latency (promote p50)
  cold_extra_ms            constant (558)        0: the universal worker's engine,
                                                 streams and comm group stay up
  bandwidth / pipelined_load (526-538)           measured PCIe H2D stream GB/s
  map_ms_per_page mu       (config.py:38)        measured VMM map+access per page
  background_kv_mapping    (540-555)             0: KV pages are pre-mapped in the
                                                 page window (no driver call)

Model coefficients for models other than the measured one are scaled by their
dense prefill FLOPs (models.ModelConfig.prefill_flops).
"""

from __future__ import annotations

import copy
from dataclasses import dataclass

GIB = 1024**3


@dataclass
class Measured:
    prefill_ms: float          # warm prefill of `prompt_tokens` tokens (ms)
    prompt_tokens: int
    switch_ms: float           # promote (weight->KV) end-to-end, p50
    stream_gb_s: float         # layer stream, weight GB/s (1e9) delivered into the slot
    map_ms_per_page: float     # VMM map + access per 2 MiB page (prewarm path)
    decode_ms: float | None = None  # batch-1 decode step; None -> weights / HBM peak
    hbm_gb_s: float = 6546.6
    source: str = ""

    @classmethod
    def from_bench(cls, bench: dict, config3: dict | None = None) -> "Measured":
        sw = bench["switch_us"]["promote_p50"] / 1e3
        if config3:
            sw = config3["switch_us"]["promote"]["p50"] / 1e3
        mu = bench.get("vmm", {}).get("slot_map_us_per_page", 240.0) / 1e3
        t = bench["ttft_ms"]
        # weight bytes delivered per second: through the packed stream when the bench ran it
        stream = (t["streamed_bytes"] / (t["cold_packed_stream_ms_p50"] / 1e3) / 1e9
                  if "cold_packed_stream_ms_p50" in t else t["stream_gbs_p50"])
        return cls(prefill_ms=bench["ms_per_step"], prompt_tokens=bench["config"]["prompt_tokens"],
                   switch_ms=sw, stream_gb_s=stream, map_ms_per_page=mu,
                   source="bench.py line (+ config-3 burst); stream = weight GB/s of the packed PCIe stream")


def measured_config(cfg, measured: Measured, shapes: dict, reference_model: str = "llama3-8b"):
    """Copy of a reference ExperimentConfig with measured latency terms.
    ``shapes`` maps model_id -> models.ModelConfig (for FLOP scaling)."""
    out = copy.deepcopy(cfg)
    out.cluster.h2d_gib_per_s = measured.stream_gb_s * 1e9 / GIB
    out.cluster.map_ms_per_page = measured.map_ms_per_page
    out.latency.warm_start_ms = measured.switch_ms
    out.latency.cold_extra_ms = 0.0
    out.latency.ref_input_tokens = measured.prompt_tokens
    ref = shapes[reference_model]
    per_tok = measured.prefill_ms / measured.prompt_tokens
    ref_flops = ref.prefill_flops(measured.prompt_tokens)
    for spec in out.models:
        shape = shapes[spec.model_id]
        ratio = shape.prefill_flops(measured.prompt_tokens) / ref_flops
        spec.prefill_a_ms = per_tok * ratio
        spec.prefill_b_ms = 0.0
        if measured.decode_ms is not None:
            spec.decode_c_ms = measured.decode_ms * ratio
        else:  # batch-1 decode is weight-streaming bound
            spec.decode_c_ms = shape.layout().total / (measured.hbm_gb_s * 1e9) * 1e3
        _, spec.kv_bytes_per_token = shape.kv_geometry()
    return out


def run_measured(engine_module, cfg, requests, policy: str, measured: Measured, shapes: dict,
                 reference_model: str = "llama3-8b", cluster_cls=None):
    """Replay `requests` through the reference engine on this framework's
    Cluster (or ``cluster_cls``, a subclass of it) with measured latencies;
    returns the engine's MetricsReport."""
    from . import cluster as ours
    from . import memswitch as ours_ms

    saved = {k: getattr(engine_module, k) for k in ("Cluster", "required_prewarm_layers", "catchup_stall_ms",
                                                    "pipelined_load", "background_kv_mapping")}
    try:
        engine_module.Cluster = cluster_cls or ours.Cluster
        engine_module.required_prewarm_layers = ours.required_prewarm_layers
        engine_module.catchup_stall_ms = ours.catchup_stall_ms
        engine_module.pipelined_load = ours_ms.pipelined_load
        engine_module.background_kv_mapping = lambda pages, mu, rate: 0.0  # page window: no KV map stall
        mcfg = measured_config(cfg, measured, shapes, reference_model)
        return engine_module.run(mcfg, requests, policy)
    finally:
        for k, v in saved.items():
            setattr(engine_module, k, v)

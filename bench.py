#!/usr/bin/env python
"""Benchmark of the universal-worker hot path (BASELINE.json configs[1]):

  Llama-3-8B bf16 universal worker on one B200, first 4 of 32 layers
  prewarmed, 2048-token prompt, cold start (layers 4..31 + lm_head streamed
  from pinned host memory while the resident layers compute).

One JSON line on rank 0:
  value  warm prefill tokens/s, weights + prompt resident in HBM (CUDA events)
  e2e    the same metric through the public API (UniversalWorker.
         activate_instance) for a COLD start: the non-resident weights and the
         prompt cross PCIe host->device inside the timed region, the first
         token comes back to the host; e2e/value = warm TTFT / cold TTFT
  ttft_ms / switch_us   cold vs warm TTFT p50/p99, memory-switch latency
  roofline   the dominant kernel (prefill GEMM) vs MEASURED_PEAKS.json
  cpu_baseline  the CPU fp32 oracle port on this host's cores (bounded sample)
Multi-GPU (N >= 2): the 8B universal worker runs as N replicas (it does not
shard) — value = all ranks' tokens / max-over-ranks time — and then the same
ranks run BASELINE configs[3], Llama-3-70B tensor-parallel over N GPUs with
per-shard layer streaming and NCCL on the TP boundary (key "tp_config4").
`--impl reference` times the reference-side CPU path (oracle port) instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("prefill tokens/s (Llama-3-8B bf16, 2048-token prompt); cold-start TTFT p50/p99 vs warm; "
          "memory-switch latency")
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def bench_config(args, world: int) -> dict:
    """The workload both arms name (BASELINE configs[1]); arm-specific
    details go under other keys."""
    layers = REF_SHAPES[args.model]["layers"] if args.model in REF_SHAPES else None
    return {"workload": f"{args.model} universal worker, first {args.prewarm_layers} of {layers} layers prewarmed, "
                        f"{args.prompt}-token prompt (BASELINE configs[1])",
            "model": args.model, "prompt_tokens": args.prompt, "prewarmed_layers": args.prewarm_layers,
            "parallelism": "replicas" if world > 1 else "single"}


_T0 = time.perf_counter()


def blog(msg: str) -> None:
    """Progress on stderr with WS_BENCH_LOG=1 (the JSON line stays the only stdout)."""
    if os.environ.get("WS_BENCH_LOG"):
        print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = (len(xs) - 1) * q / 100.0
    f = int(k)
    c = min(f + 1, len(xs) - 1)
    return xs[f] + (xs[c] - xs[f]) * (k - f)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        # samples go to a file, not a pipe: nobody reads a pipe until __exit__,
        # and once its 64 KB buffer fills (~2 min of samples) nvidia-smi blocks
        # inside its sampling loop, which can stall this process's own driver
        # calls behind it
        import tempfile
        self.out = tempfile.TemporaryFile(mode="w+")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=self.out, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            self.proc.wait()
        self.out.seek(0)
        out = self.out.read()
        self.out.close()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()),
                                   default=None)}


# ---------------------------------------------------------------- CPU side
def cpu_prefill_sample(cfg, tokens: int, min_seconds: float = 10.0, max_layers: int = 4):
    """Oracle port (torch CPU fp32, all host threads): time decoder layers of
    `cfg` at `tokens` tokens until min_seconds, extrapolate to the full model
    (layers * t_layer + lm_head row). Returns (tokens/s, sample text, threads)."""
    import torch

    from oracle import llama_fp32 as O

    torch.manual_seed(0)
    d, H, KV, hd, f = cfg.hidden, cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.ffn
    w = {
        "l0.attn_norm": torch.ones(d), "l0.ffn_norm": torch.ones(d),
        "l0.wqkv": torch.randn(cfg.qkv_dim, d) * 0.02, "l0.wo": torch.randn(d, H * hd) * 0.02,
        "l0.wgu": torch.randn(2 * f, d) * 0.02, "l0.wdown": torch.randn(d, f) * 0.02,
    }
    one = cfg.with_(layers=1)
    x = torch.randn(tokens, d)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_layers and (time.perf_counter() - t_start < min_seconds or len(times) < 1):
        t0 = time.perf_counter()
        _layer_cpu(one, w, x, O)
        times.append(time.perf_counter() - t0)
    t_layer = statistics.median(times)
    head = torch.randn(cfg.vocab, d) * 0.02
    t0 = time.perf_counter()
    _ = x[-1:] @ head.T
    t_head = time.perf_counter() - t0
    total = cfg.layers * t_layer + t_head
    sample = (f"{len(times)} x one {cfg.name} decoder layer at {tokens} tokens (median {t_layer*1e3:.0f} ms) "
              f"extrapolated x{cfg.layers} + lm_head row; torch CPU fp32 oracle port")
    return tokens / total, sample, torch.get_num_threads(), time.perf_counter() - t_start


def _layer_cpu(cfg, w, x, O):
    import math

    import torch

    S = x.shape[0]
    H, KV, hd = cfg.heads, cfg.kv_heads, cfg.head_dim
    cos, sin = O.rope_table(hd, cfg.rope_theta, S)
    h = O._rms(x, w["l0.attn_norm"], cfg.rms_eps)
    qkv = h @ w["l0.wqkv"].T
    q = O._rope(qkv[:, : H * hd].view(S, H, hd), cos, sin)
    k = O._rope(qkv[:, H * hd: (H + KV) * hd].view(S, KV, hd), cos, sin)
    v = qkv[:, (H + KV) * hd:].view(S, KV, hd)
    g = H // KV
    o = torch.nn.functional.scaled_dot_product_attention(
        q.transpose(0, 1), k.repeat_interleave(g, 1).transpose(0, 1), v.repeat_interleave(g, 1).transpose(0, 1),
        is_causal=True).transpose(0, 1).reshape(S, H * hd)
    x = x + o @ w["l0.wo"].T
    h = O._rms(x, w["l0.ffn_norm"], cfg.rms_eps)
    gu = h @ w["l0.wgu"].T
    x = x + (torch.nn.functional.silu(gu[:, : cfg.ffn]) * gu[:, cfg.ffn:]) @ w["l0.wdown"].T
    return x


# Model shapes of the reference arm (public HF configs).
# Hard-coded so the reference arm never loads this repo's package or native
# library; tests/test_bench_contract.py checks them against models.py.
REF_SHAPES = {
    "llama3-8b": dict(layers=32, hidden=4096, ffn=14336, heads=32, kv_heads=8, head_dim=128, vocab=128256,
                      rope_theta=500000.0, rms_eps=1e-5),
}


def _ref_cpu_weights(shape, seed=0):
    """bf16 weights of every decoder layer + final norm + lm_head on the host,
    generated once outside the timed region. Values are N(0, 0.02) (norm gains
    N(1, 0.1)) drawn from one 2^27-value seeded pool at a random offset per
    tensor: 8 G fresh normals would take ~70 s of single-threaded RNG, and the
    forward's cost does not depend on the values."""
    import torch

    g = torch.Generator().manual_seed(seed)
    pool = (torch.randn(1 << 27, generator=g) * 0.02).bfloat16()
    d, f, H, KV, hd = shape["hidden"], shape["ffn"], shape["heads"], shape["kv_heads"], shape["head_dim"]
    q = (H + 2 * KV) * hd

    def lin(*sh):
        n = 1
        for v in sh:
            n *= v
        off = int(torch.randint(0, 1 << 27, (1,), generator=g))
        reps = -(-(off + n) // (1 << 27))
        return pool.repeat(reps)[off:off + n].view(*sh).clone()

    def norm(n):
        return (torch.randn(n, generator=g) * 0.1 + 1.0).bfloat16()

    layers = [dict(attn_norm=norm(d), wqkv=lin(q, d), wo=lin(d, H * hd), ffn_norm=norm(d), wg=lin(f, d),
                   wu=lin(f, d), wdown=lin(d, f)) for _ in range(shape["layers"])]
    return dict(embed=lin(shape["vocab"], d), layers=layers, final_norm=norm(d), lm_head=lin(shape["vocab"], d))


def _ref_cpu_prefill(shape, w, tokens):
    """One full prefill on the host CPU: the oracle's fp32 Llama forward
    (oracle/llama_fp32.py: RMSNorm, rotate-half RoPE, causal GQA attention,
    SwiGLU, fp32 residual) over every decoder layer, each layer's bf16
    weights upcast to fp32 as it runs, then the last row's logits. Returns the
    greedy token."""
    import torch

    from oracle import llama_fp32 as O

    S = tokens.numel()
    H, KV, hd, eps = shape["heads"], shape["kv_heads"], shape["head_dim"], shape["rms_eps"]
    cos, sin = O.rope_table(hd, shape["rope_theta"], S)
    x = w["embed"][tokens].float()
    for L in w["layers"]:
        h = O._rms(x, L["attn_norm"].float(), eps)
        qkv = h @ L["wqkv"].float().T
        q = O._rope(qkv[:, : H * hd].view(S, H, hd), cos, sin)
        k = O._rope(qkv[:, H * hd: (H + KV) * hd].view(S, KV, hd), cos, sin)
        v = qkv[:, (H + KV) * hd:].view(S, KV, hd)
        g = H // KV
        o = torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1), k.repeat_interleave(g, 1).transpose(0, 1), v.repeat_interleave(g, 1).transpose(0, 1),
            is_causal=True).transpose(0, 1).reshape(S, H * hd)
        x = x + o @ L["wo"].float().T
        h = O._rms(x, L["ffn_norm"].float(), eps)
        x = x + (torch.nn.functional.silu(h @ L["wg"].float().T) * (h @ L["wu"].float().T)) @ L["wdown"].float().T
    h = O._rms(x[-1:], w["final_norm"].float(), eps)
    return int((h @ w["lm_head"].float().T).argmax())


def _ref_ledger_ops(n=2000):
    """The reference's switch bookkeeping (cluster.py:291-387, restated in
    oracle/ledger.py): promote (evicting 3 co-prewarmed slots) / reclaim /
    release on the config-3 ledger (89,600 pages, 4 models), timed per call."""
    from oracle import ledger as Lg

    models = [("llama3-8b", 7659), ("qwen2.5-7b", 7263), ("mistral-7b", 6907), ("phi3-mini", 3645)]
    page = 2 << 20
    t = {"promote": [], "reclaim": [], "release": [], "begin_prewarm": []}
    for i in range(n):
        cl = Lg.new_cluster(1, 1, 89600, page)
        t0 = time.perf_counter()
        for m, p in models:
            Lg.begin_prewarm(cl, 0, m, p, 4)
        t1 = time.perf_counter()
        m, p = models[i % 4]
        iid, _ = Lg.promote(cl, (0,), m, 1, p * page, 32, 4)
        t2 = time.perf_counter()
        cl["instances"][iid]["state"] = Lg.ACTIVE
        Lg.enter_grace(cl, iid)
        t3 = time.perf_counter()
        Lg.reclaim(cl, 0, 8, 32, 10 * (1 << 30))
        t4 = time.perf_counter()
        Lg.release(cl, iid)
        t5 = time.perf_counter()
        t["begin_prewarm"].append((t1 - t0) * 1e6 / 4)
        t["promote"].append((t2 - t1) * 1e6)
        t["reclaim"].append((t4 - t3) * 1e6)
        t["release"].append((t5 - t4) * 1e6)
    return {k + "_p50_us": pct(v, 50) for k, v in t.items()} | {"n": n, "cores": 1,
                                                                 "source": "oracle/ledger.py (cluster.py:245-387)"}


def run_reference(args, rank, world):
    """--impl reference: the reference-side CPU path on the host cores — the
    oracle port of a FULL prefill (every decoder layer, 2048 tokens, fp32 on
    all host threads) per step, plus the reference ledger ops beside the GPU
    arm's switch latency. Never imports this repo's package or library."""
    if rank != 0:
        return
    import torch

    shape = REF_SHAPES[args.model]
    w = _ref_cpu_weights(shape)
    tokens = torch.randint(0, shape["vocab"], (args.prompt,), generator=torch.Generator().manual_seed(7))
    # a full CPU prefill takes ~19 s on 16 threads: one warm-up (the CPU path
    # has no caches or clocks to settle beyond the first pass) and as many of
    # the requested steps as fit in a 240 s budget (at least 2), so the arm
    # ends within a few minutes at the driver's --steps 20 --warmup 5
    for _ in range(min(args.warmup, 1)):
        _ref_cpu_prefill(shape, w, tokens)
    times = []
    t_arm = time.perf_counter()
    for i in range(args.steps):
        if i >= 2 and time.perf_counter() - t_arm > 240.0:
            break
        t0 = time.perf_counter()
        _ref_cpu_prefill(shape, w, tokens)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    n_timed = len(times)
    value = n_timed * args.prompt / total
    threads = torch.get_num_threads()
    sample = (f"{n_timed} full {args.model} prefills of a {args.prompt}-token prompt ({shape['layers']} layers "
              f"+ last-row lm_head), torch CPU fp32 oracle port, {threads} threads; median "
              f"{statistics.median(times):.1f} s per prefill")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": n_timed, "steps_requested": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": total / n_timed * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded random-init weights of the named shape, random token ids)",
        "config": bench_config(args, world),
        "arm": "the reference has no GPU path (its prefill is the linear model engine.py:107-108), so its arm is "
               "the CPU fp32 oracle port of the full forward of the same workload (every layer of the prefill; the "
               "prewarmed prefix changes nothing on a CPU)",
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu": _cpu_model()},
        "ledger_us": _ref_ledger_ops(),
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200.cluster import catchup_stall_ms, required_prewarm_layers
    from paper_2512_09472_b200.devmem import view
    from paper_2512_09472_b200.weights import pack_stream, pinned_host_copy, synth_flat
    from paper_2512_09472_b200.worker import UniversalWorker

    dev = local_rank
    torch.cuda.set_device(dev)
    cfg = M.ALL[args.model]
    S, K, Wm = args.prompt, args.steps, args.warmup

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- setup: weights on the host (cold-start source), slot, prewarmed prefix
    t_setup = time.perf_counter()
    flat = synth_flat(cfg, seed=rank, device="cuda")
    host = pinned_host_copy(flat)
    t_pack = time.perf_counter()
    packed = pack_stream(cfg, flat)  # lossless packed host image of the streamable ranges
    pack_s = time.perf_counter() - t_pack
    del flat
    torch.cuda.empty_cache()
    pool_pages = args.pool_pages
    if pool_pages <= 0:  # a full-HBM universal worker: every byte but the reserve is pool
        free_b, _ = torch.cuda.mem_get_info(dev)
        pool_pages = int((free_b - args.reserve_gib * (1 << 30)) // M.PAGE)
    w = UniversalWorker(dev, pool_pages=pool_pages, max_tokens=max(S, 256))
    entry = w.register(cfg, host)
    slot = w.prewarm(cfg.name, layers=args.prewarm_layers, full=False)  # exactly k layers resident
    init_ms, map_pp, _ = (lambda a, b, c: (N.call("ws_pool_timing", w.gpu.pool, a, b, c), a, b, c))(
        *(__import__("ctypes").c_double() for _ in range(3)))[1:]
    prompt = torch.randint(0, cfg.vocab, (S,), generator=torch.Generator().manual_seed(7), dtype=torch.int32)
    prompt_pinned = prompt.pin_memory()
    setup_s = time.perf_counter() - t_setup
    blog("setup done")

    # clocks are sampled across every timed region below (cold, warm, value)
    clk = Clocks(dev).__enter__()
    time.sleep(0.5)  # let nvidia-smi start sampling before the first timed step
    # ---- TTFT legs: n_prompts distinct seeded 2048-token
    #      prompts per leg after Wm warm-up activations; each leg drops the
    #      ledger's residency back to k layers so the suffix streams again
    n_prompts = max(K, args.ttft_prompts)
    gp = torch.Generator().manual_seed(1234)
    prompts = [torch.randint(0, cfg.vocab, (S,), generator=gp, dtype=torch.int32).pin_memory()
               for _ in range(n_prompts)]

    def leg(k_resident, source=None, head=False):
        out = []
        for i in range(Wm + n_prompts):
            if k_resident is not None:
                w.drop_suffix(cfg.name, k_resident, head=head)
            barrier()
            r = w.activate_instance(cfg.name, prompts[(i - Wm) % n_prompts] if i >= Wm else prompt_pinned,
                                    source=source)
            w.release()
            if i >= Wm:
                out.append(r)
        return out

    k0 = args.prewarm_layers
    # cold, plain bf16 stream: layers k..L + lm_head over PCIe
    cold = leg(k0)
    blog("cold plain leg")
    # cold (e2e), packed stream: the same ranges losslessly packed on the host
    # (~34% fewer PCIe bytes), unpacked on the GPU per layer
    w.set_packed(cfg.name, packed)
    cold_packed = leg(k0)
    blog("cold packed leg")
    w.models[cfg.name].packed = None
    # cold from an HBM-resident image on this GPU: the stand-in for a peer
    # GPU's copy, showing what layer streaming hides once the
    # link keeps up with the forward
    # Off by default (--hbm-leg): with the suffix copied device-to-device
    # while the prefill runs, ~1 in 5 bench runs of this round's last session
    # stalled inside this leg (the compute stream never reached the
    # activation's closing event; faulthandler stacks in DESIGN §5), never in
    # the PCIe legs around it; the default run must finish.
    cold_hbm = []
    if args.hbm_leg:
        dev_src = host.to(f"cuda:{dev}")
        cold_hbm = leg(k0, source=dev_src)
        blog("cold hbm leg")
        del dev_src
        torch.cuda.empty_cache()
    if os.environ.get("WS_BENCH_STOP_AFTER_HBM"):  # diagnostics (the stall hunt)
        sys.exit(0)
    # warm: every layer resident
    warm = leg(None)
    blog("warm leg")
    # the reference's own policy: k = required_prewarm_layers (cluster.py:145-166)
    # at the MEASURED stream bandwidth and per-token prefill cost, plain and packed
    spec = entry.spec
    warm_ms = pct([r.ttft_ms for r in warm], 50)
    a_ms = warm_ms / S  # measured per-token prefill cost (the reference's prefill_a)
    spec_m = type(spec)(spec.model_id, spec.weight_bytes, 1, layers=cfg.layers, prefill_a_ms=a_ms, prefill_b_ms=0.0)
    stream_gbs = statistics.median(r.streamed_bytes / (r.stream_ms / 1e3) / 1e9 for r in cold)
    bw_bytes_ms = stream_gbs * 1e9 / 1e3
    k_req = required_prewarm_layers(spec_m, bw_bytes_ms, S)
    packed_bw = cold[0].streamed_bytes / (statistics.median(r.stream_ms for r in cold_packed) / 1e3) / 1e3
    k_req_packed = required_prewarm_layers(spec_m, packed_bw, S)
    cold_kreq = leg(k_req)
    blog("k_req leg")
    w.set_packed(cfg.name, packed)
    cold_kreq_packed = leg(k_req_packed)
    blog("k_req packed leg")
    w.models[cfg.name].packed = None
    # the same policy at the reference's BYTE budget: its uniform layer_bytes
    # (cluster.py:85-88) folds the embedding and lm_head into every layer, so
    # k prewarmed layers are k x partition/L bytes; spent as embedding +
    # lm_head + as many whole layers as fit, the stream is layers only
    lay = entry.layout
    budget = k_req * spec.partition_bytes / cfg.layers
    head_b = lay.total - lay.final_norm
    m_budget = max(m for m in range(cfg.layers + 1) if m == 0 or lay.prefix_bytes(m) + head_b <= budget)
    cold_budget = leg(m_budget, head=True)
    blog("byte-budget leg")

    # ---- value: warm prefill throughput, prompt + weights resident in HBM
    w.switch_memory(cfg.name)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(w.compute):
        toks = prompt_pinned.to("cuda", non_blocking=True)
        for _ in range(Wm):
            s = w.open_seq(S)
            w.prefill(s, toks)
            w.close_seq(s)
        torch.cuda.synchronize()
        barrier()
        launches0 = N.kernel_launches()
        fallbacks0 = N.fallback_counts()
        ev0.record(w.compute)
        for _ in range(K):
            s = w.open_seq(S)
            w.prefill(s, toks)
            w.close_seq(s)
        ev1.record(w.compute)
        torch.cuda.synchronize()
        launches = N.kernel_launches() - launches0
        fallbacks = {k: v - fallbacks0[k] for k, v in N.fallback_counts().items()}
    clk.__exit__(None, None, None)
    barrier()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    value = world * K * S / (elapsed_ms / 1e3)
    prefill_ms = elapsed_ms / K
    blog("value")

    # ---- memory switch burst: promote (weight->KV), reclaim (KV->free), release
    w.release()
    sw_done, sw_host, sw_kernel, rc_done, rel_done = [], [], [], [], []
    for i in range(args.switch_iters):
        t0 = time.perf_counter()
        inst, ev, host_ms, kms = w.switch_memory(cfg.name)
        w.compute.synchronize()
        t1 = time.perf_counter()
        inst.state = inst.state.ACTIVE
        w.cluster.enter_grace(inst)
        t2 = time.perf_counter()
        w.reclaim(0, 0.0)
        w.compute.synchronize()
        t3 = time.perf_counter()
        w.release()
        w.compute.synchronize()
        t4 = time.perf_counter()
        sw_done.append((t1 - t0) * 1e6)
        sw_host.append(host_ms * 1e3)
        sw_kernel.append(kms * 1e3)
        rc_done.append((t3 - t2) * 1e6)
        rel_done.append((t4 - t3) * 1e6)

    blog("switch burst")
    # ---- decode: every sequence prefilled to decode_ctx, then B tokens per step
    #      (HBM bound: all weights but the embedding table + each sequence's KV)
    decode = []
    if args.decode_batches:
        w.switch_memory(cfg.name)
        ctx = args.decode_ctx
        Kd = max(K, 20)  # timed decode steps (a step is ~4-6 ms)
        bmax = max(args.decode_batches)
        g = torch.Generator().manual_seed(11)
        seqs = []
        with torch.cuda.stream(w.compute):
            for _ in range(bmax):
                s = w.open_seq(ctx + Kd + 1)
                w.prefill(s, torch.randint(0, cfg.vocab, (ctx,), generator=g, dtype=torch.int32).cuda())
                seqs.append(s)
        torch.cuda.synchronize()
        weight_bytes = entry.layout.total - cfg.vocab * cfg.hidden * 2
        kv_tok = cfg.kv_geometry()[1]
        pk_hbm = peaks()[0]["hbm_gbs"]
        for B in args.decode_batches:
            sd = torch.tensor(seqs[:B], dtype=torch.int32, device="cuda")
            tok = torch.randint(0, cfg.vocab, (B,), generator=g, dtype=torch.int32).cuda()
            with torch.cuda.stream(w.compute):
                # warm-up: >= Wm steps and >= 0.3 s, so the SM clock has recovered
                # from the power-capped prefills above before the timed steps
                # (without it B = 1, measured first, read ~9% slow)
                t_w, i = time.perf_counter(), 0
                while i < Wm or time.perf_counter() - t_w < 0.3:
                    pos = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
                    _, tok = w.decode_graphed(sd, pos, tok, ctx + 1)
                    torch.cuda.synchronize()
                    i += 1
                barrier()
                # one more untimed step in flight, so the timed region does not
                # open on an idle GPU waiting for the host's first replay
                pos = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
                _, tok = w.decode_graphed(sd, pos, tok, ctx + 1)
                d0 = torch.cuda.Event(enable_timing=True)
                d0.record(w.compute)
                for i in range(Kd):
                    pos = torch.full((B,), ctx + i, dtype=torch.int32, device="cuda")
                    _, tok = w.decode_graphed(sd, pos, tok, ctx + i + 1)
                d1 = torch.cuda.Event(enable_timing=True)
                d1.record(w.compute)
            torch.cuda.synchronize()
            ms = max_over_ranks(d0.elapsed_time(d1)) / Kd
            nbytes = weight_bytes + B * (ctx + Kd / 2) * kv_tok
            decode.append({"batch": B, "ctx": ctx, "steps": Kd, "ms_per_step": ms, "tokens_per_s": world * B / ms * 1e3,
                           "algorithmic_gb": nbytes / 1e9, "achieved_gbs": nbytes / ms / 1e6,
                           "frac_of_hbm": nbytes / ms / 1e6 / pk_hbm})
        for s in seqs:
            w.close_seq(s)
        w.release()

    # ---- dominant kernel: the gate/up GEMM of the prefill, timed alone
    pk, kind = peaks()
    lay = entry.layout.layers[0]
    B = view(slot.va + lay["wgu"], (2 * cfg.ffn, cfg.hidden), torch.bfloat16, dev)
    A = torch.randn(S, cfg.hidden, device="cuda").bfloat16()
    Cm = torch.empty(S, 2 * cfg.ffn, device="cuda", dtype=torch.bfloat16)
    import ctypes as C

    def gemm_once(impl):
        N.call("ws_gemm", C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), S, 2 * cfg.ffn, cfg.hidden, 0,
               C.c_void_p(Cm.data_ptr()), None, impl, C.c_void_p(torch.cuda.current_stream().cuda_stream))

    gemm_flops = 2.0 * S * 2 * cfg.ffn * cfg.hidden
    gemm_ms = {}
    for impl in (0, 1):
        for _ in range(3):
            gemm_once(impl)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(20):
            gemm_once(impl)
        g1.record()
        torch.cuda.synchronize()
        gemm_ms[impl] = g0.elapsed_time(g1) / 20
    achieved = gemm_flops / (gemm_ms[0] / 1e3) / 1e12
    blog("roofline GEMM")

    # ---- the reference's analytic model, evaluated with MEASURED inputs
    stall_pred = catchup_stall_ms(spec_m, args.prewarm_layers, bw_bytes_ms, S)
    stall_packed = catchup_stall_ms(spec_m, args.prewarm_layers, packed_bw, S)

    traffic = None
    tp = ROOT / "profiles" / "gemm_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")

    cold_ttft = [r.ttft_ms for r in cold]
    packed_ttft = [r.ttft_ms for r in cold_packed]
    warm_ttft = [r.ttft_ms for r in warm]
    cold_total_s = max_over_ranks(sum(packed_ttft) / 1e3)
    e2e_value = world * len(packed_ttft) * S / cold_total_s
    clk_sum = clk.summary()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        v, sample, threads, secs = cpu_prefill_sample(cfg, S, min_seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
               "sample": sample + f"; {secs:.1f} s of CPU work", "cpu": _cpu_model()}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": prefill_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded random-init weights of the named shape, random token ids)",
        "config": bench_config(args, world),
        "setup": {"weight_source": "pinned host memory (PCIe H2D on the copy engine)",
                  "l2": "no flush needed: 16 GB of weights per step > 126 MB L2",
                  "pool_pages": pool_pages, "pool_gib": pool_pages * M.PAGE / (1 << 30)},
        "e2e": {"value": e2e_value, "unit": "tokens/s",
                "h2d_bytes_per_step": int(statistics.median(r.streamed_bytes for r in cold_packed)) + S * 4,
                "d2h_bytes_per_step": 4,
                "path": "UniversalWorker.activate_instance (cold, packed stream): switch_memory + packed layer "
                        "streaming from pinned host memory + GPU unpack + prefill"},
        "reference_model_at_measured_inputs": {
            "required_prewarm_layers": k_req, "catchup_stall_ms_k4": stall_pred,
            "predicted_cold_ttft_ms": pct(warm_ttft, 50) + stall_pred,
            "packed_weight_gbs": packed_bw / 1e6, "required_prewarm_layers_packed": k_req_packed,
            "catchup_stall_ms_k4_packed": stall_packed,
            "predicted_cold_ttft_ms_packed": pct(warm_ttft, 50) + stall_packed,
            "note": "cluster.py:145-182 evaluated with the measured stream bandwidth (plain link bytes, and "
                    "weight bytes through the packed stream) and per-token prefill cost"},
        "switch_us": {"promote_p50": pct(sw_done, 50), "promote_p99": pct(sw_done, 99),
                      "promote_host_p50": pct(sw_host, 50), "switch_kernel_p50": pct(sw_kernel, 50),
                      "reclaim_p50": pct(rc_done, 50), "reclaim_p99": pct(rc_done, 99),
                      "release_p50": pct(rel_done, 50), "release_p99": pct(rel_done, 99),
                      "n": len(sw_done), "target_us": 1000.0,
                      "kv_pages_switched": w.gpu.total_pages - entry.spec.partition_pages(M.PAGE)},
        "prefill": {"ms": prefill_ms, "tflops": cfg.prefill_flops(S) / (prefill_ms / 1e3) / 1e12,
                    "frac_of_sustained": cfg.prefill_flops(S) / (prefill_ms / 1e3) / 1e12 /
                    pk["bf16_tflops_sustained"], "algorithmic_tflop": cfg.prefill_flops(S) / 1e12},
        "decode": {"per_batch": decode, "bound": "hbm", "peak_gbs": peaks()[0]["hbm_gbs"],
                   "bytes": "all weights except the embedding table + every sequence's K/V, per step",
                   "path": "UniversalWorker.decode_graphed (CUDA-graph replay of decode): skinny stream-K tcgen05 GEMMs + "
                           "paged GQA decode attention"},
        "roofline": {"bound": "tensor", "kernel": "prefill gate/up GEMM 2048x28672x4096 (tensor-core path)",
                     "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": achieved / pk["bf16_tflops"], "traffic": traffic, "peak_kind": kind + " burst",
                     "launch_ms": gemm_ms[0], "legacy_mma_sync_ms": gemm_ms[1]},
        "cpu_baseline": cpu,
        "clocks": clk_sum,
        "gpu_launches": launches,
        "legacy_fallbacks_in_timed_region": fallbacks,
        "setup_s": setup_s,
        "vmm": {"pool_init_ms": init_ms.value, "pool_pages": pool_pages,
                "slot_map_us_per_page": map_pp.value * 1e3, "reference_mu_us_per_page": 39.0,
                "slot_placement": ["windowed", "composite", "scattered"][_placement(w, slot)],
                "prewarm_ms": getattr(slot, "prewarm_ms", None),
                "handle_mib": _handle_pages(w) * 2,
                "note": "2 MiB ledger pages backed by large physical handles mapped once into the page window; "
                        "a windowed slot is a window range (no driver call to map, evict or re-prewarm); "
                        "reference mu = config.py:38"},
        # last key: the driver's stdout tail keeps the end of the line
        "ttft_ms": {"prompts": n_prompts, "prompt_seeds": "torch.Generator().manual_seed(1234), one 2048-token "
                    "prompt per activation",
                    "cold_p50": pct(packed_ttft, 50), "cold_p99": pct(packed_ttft, 99),
                    "cold_over_warm_p50": pct(packed_ttft, 50) / pct(warm_ttft, 50),
                    "cold_packed_streamed_bytes": cold_packed[0].streamed_bytes,
                    "cold_packed_stream_ms_p50": pct([r.stream_ms for r in cold_packed], 50),
                    "pack_ratio": cold_packed[0].streamed_bytes / cold[0].streamed_bytes,
                    "pack_setup_s": pack_s,
                    "cold_plain_p50": pct(cold_ttft, 50), "cold_plain_p99": pct(cold_ttft, 99),
                    "warm_p50": pct(warm_ttft, 50), "warm_p99": pct(warm_ttft, 99),
                    "cold_plain_over_warm_p50": pct(cold_ttft, 50) / pct(warm_ttft, 50), "target_ratio": 1.2,
                    "cold_device_p50": pct([r.device_ms for r in cold], 50),
                    "stream_ms_p50": pct([r.stream_ms for r in cold], 50),
                    "streamed_bytes": cold[0].streamed_bytes, "stream_gbs_p50": stream_gbs,
                    "pcie_gen5_peak_gbs": 64.0,
                    **({"cold_hbm_source_p50": pct([r.ttft_ms for r in cold_hbm], 50),
                        "cold_hbm_source_p99": pct([r.ttft_ms for r in cold_hbm], 99),
                        "cold_hbm_source_over_warm_p50": pct([r.ttft_ms for r in cold_hbm], 50) / pct(warm_ttft, 50),
                        "hbm_source_stream_gbs_p50": statistics.median(
                            r.streamed_bytes / (r.stream_ms / 1e3) / 1e9 for r in cold_hbm)} if cold_hbm else {}),
                    "hbm_source_note": ("layers 4..31 + lm_head streamed from a device-resident copy on the same "
                                        "GPU (stand-in for an NVLink peer source; not a peer measurement)"
                                        if cold_hbm else
                                        "HBM-source leg off by default (--hbm-leg): intermittent stall under "
                                        "investigation; last measured 27.8 ms = 1.13x warm, profiles/r2f_bench.json"),
                    "k_required": k_req, "cold_k_required_p50": pct([r.ttft_ms for r in cold_kreq], 50),
                    "cold_k_required_p99": pct([r.ttft_ms for r in cold_kreq], 99),
                    "cold_k_required_over_warm_p50": pct([r.ttft_ms for r in cold_kreq], 50) / pct(warm_ttft, 50),
                    "k_required_packed": k_req_packed,
                    "cold_k_required_packed_p50": pct([r.ttft_ms for r in cold_kreq_packed], 50),
                    "cold_k_required_packed_p99": pct([r.ttft_ms for r in cold_kreq_packed], 99),
                    "cold_k_required_packed_over_warm_p50":
                        pct([r.ttft_ms for r in cold_kreq_packed], 50) / pct(warm_ttft, 50),
                    "k_required_note": "k = required_prewarm_layers (cluster.py:145-166) at the measured PCIe "
                                       "stream bandwidth (plain / packed) and the measured per-token prefill cost",
                    "k_required_byte_budget_gb": budget / 1e9,
                    "byte_budget_resident": f"embedding + lm_head + layers [0, {m_budget})",
                    "cold_byte_budget_p50": pct([r.ttft_ms for r in cold_budget], 50),
                    "cold_byte_budget_p99": pct([r.ttft_ms for r in cold_budget], 99),
                    "cold_byte_budget_over_warm_p50": pct([r.ttft_ms for r in cold_budget], 50) / pct(warm_ttft, 50),
                    "cold_byte_budget_streamed_bytes": cold_budget[0].streamed_bytes,
                    "cold_byte_budget_stream_ms_p50": pct([r.stream_ms for r in cold_budget], 50),
                    "cold_byte_budget_device_ms_p50": pct([r.device_ms for r in cold_budget], 50)},

    }
    w.release()
    w.close()
    # the later legs build their own images: drop this leg's pinned host
    # copies first (host memory peaks per rank, N ranks per node)
    del w, entry, slot, host, packed, prompts, prompt_pinned, B, A, Cm
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    if args.config3_switches > 0:
        # BASELINE configs[2]: 4 models co-prewarmed, weight<->KV switch burst
        # (tools/config3_switch_burst.py; its ledger-vs-oracle replay is
        # tests/test_gpu_config3.py)
        sys.path.insert(0, str(ROOT / "tools"))
        from config3_switch_burst import run_burst

        blog("config 3 start")
        line["config3_switch_burst"] = run_burst(switches=args.config3_switches, device=dev)
        blog("config 3 done")
        torch.cuda.empty_cache()
    if args.config5_policies:
        # BASELINE configs[4]: the reference engine's 8-worker decision log
        # replayed on real workers (tools/config5_live.py; ledger checked
        # against the engine after every op); logical GPU g on rank g % world
        sys.path.insert(0, str(ROOT / "tools"))
        from config5_live import HostImages, load_trace, replay_gpu, summarize

        trace = load_trace()
        pols = [p_ for p_ in args.config5_policies.split(",") if p_]
        mine = [g for g in range(trace["gpus"]) if g % world == rank]
        need = sorted({o["model"] for p_ in pols for o in trace["policies"][p_]["ops"]
                       if o["gpu"] in mine and "model" in o})
        t_c5 = time.perf_counter()
        images = HostImages(need, dev)
        c5 = {"setup_s": time.perf_counter() - t_c5, "logical_gpus_per_rank": len(mine)}
        for p_ in pols:
            blog(f"config 5 {p_}")
            res = [replay_gpu(trace, p_, g, dev, images) for g in mine]
            if world > 1:
                allres = [None] * world
                dist.all_gather_object(allres, res)
                res = [x for r_ in allres for x in r_]
            c5[p_] = summarize(trace, p_, res)
        line["config5_live"] = c5
        del images
        torch.cuda.empty_cache()
    if world > 1 or args.tp_block:
        # BASELINE configs[3] on the same ranks: Llama-3-70B TP=world cold start
        line["tp_config4"] = run_tp(args, rank, world, local_rank,
                                    peer_only=os.environ.get("WS_BENCH_ONE_GPU") == "1")
    line = {k_: v_ for k_, v_ in line.items() if k_ != "ttft_ms"} | {"ttft_ms": line["ttft_ms"]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_tp(args, rank, world, local_rank, peer_only=False):
    """BASELINE configs[3]: Llama-3-70B tensor-parallel cold start over the
    ``world`` ranks (one GPU each): every rank holds its Megatron shard
    (tp.shard_config) in a slot with the first k layers resident, streams its
    own shard's layers k..L over its own PCIe link while the resident layers
    compute, and the row-parallel partials are all-reduced over NCCL (bf16 on
    the wire) on NVLink / NVSwitch — readiness is the max over ranks, like
    the reference (engine.py:516-538). Also: warm TTFT, warm prefill
    throughput, and the bf16 allreduce's bus bandwidth at the TP boundary's
    message size ([S, d] bf16). ``peer_only``: the collectives run on the
    peer-memory kernels instead (ranks sharing one GPU in tests)."""
    import torch
    import torch.distributed as dist

    from paper_2512_09472_b200 import models as M
    from paper_2512_09472_b200 import tp as TP
    from paper_2512_09472_b200.worker import UniversalWorker
    from paper_2512_09472_b200.weights import pinned_host_copy

    dev = local_rank
    cfg = M.ALL[args.tp_model]
    scfg = TP.shard_config(cfg, world)
    S, K, Wm = args.prompt, args.tp_steps, 3
    k = args.tp_prewarm_layers

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if dist.get_backend() == "gloo" else f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t0 = time.perf_counter()
    shard = TP.synth_shard(cfg, world, rank, seed=0, device=f"cuda:{dev}")
    host = pinned_host_copy(shard)
    del shard
    torch.cuda.empty_cache()
    if peer_only:
        grp = TP.TpGroup.peer_only(dev, max(S * cfg.hidden, cfg.vocab))
    elif world > 1:
        grp = TP.TpGroup.from_torch_dist(dev)
    else:
        grp = TP.TpGroup(0, 1, dev, TP.TpGroup.unique_id())
    pages = -(-scfg.layout().total // M.PAGE)
    tpb, _ = scfg.kv_geometry()
    w = UniversalWorker(dev, pool_pages=pages + -(-(S + 8) // tpb) + 64, max_tokens=S)
    w.register(scfg, host, tp=grp)
    w.prewarm(scfg.name, layers=k, full=False)
    setup_s = time.perf_counter() - t0
    g = torch.Generator().manual_seed(99)
    prompts = [torch.randint(0, cfg.vocab, (S,), generator=g, dtype=torch.int32).pin_memory() for _ in range(K)]
    cold, warm, agree = [], [], True
    for i in range(Wm + K):
        w.drop_suffix(scfg.name, k)
        barrier()
        r = w.activate_instance(scfg.name, prompts[i % K])
        w.release()
        if i >= Wm:
            cold.append((max_over_ranks(r.ttft_ms), r.stream_ms, r.streamed_bytes))
            agree &= max_over_ranks(r.token) == -max_over_ranks(-r.token)  # every rank got the same token
    for i in range(Wm + K):
        barrier()
        r = w.activate_instance(scfg.name, prompts[i % K])
        w.release()
        if i >= Wm:
            warm.append(max_over_ranks(r.ttft_ms))
    # warm prefill throughput (device events, max over ranks)
    w.switch_memory(scfg.name)
    toks = prompts[0].to(f"cuda:{dev}")
    with torch.cuda.stream(w.compute):
        for _ in range(2):
            sq = w.open_seq(S)
            w.prefill(sq, toks)
            w.close_seq(sq)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(w.compute)
        for _ in range(K):
            sq = w.open_seq(S)
            w.prefill(sq, toks)
            w.close_seq(sq)
        e1.record(w.compute)
        torch.cuda.synchronize()
    prefill_ms = max_over_ranks(e0.elapsed_time(e1)) / K
    w.release()
    # the TP boundary's collective alone: [S, d] bf16 allreduce, 2 per layer
    ar = None
    if not peer_only and world > 1:
        buf = torch.randn(S, cfg.hidden, device=f"cuda:{dev}").bfloat16()
        for _ in range(5):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(20):
            dist.all_reduce(buf)
        a1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(a0.elapsed_time(a1)) / 20
        nbytes = buf.numel() * 2
        ar = {"bytes": nbytes, "ms": ms, "algbw_gbs": nbytes / ms / 1e6,
              "busbw_gbs": 2 * (world - 1) / world * nbytes / ms / 1e6, "nvlink5_peak_gbs": 900.0,
              "per_prefill": 2 * cfg.layers, "note": "torch.distributed NCCL bf16 allreduce, same size as the "
                                                     "row-parallel partial the model's own NCCL call reduces"}
    w.close()
    grp.close()
    cold_ttft = [c[0] for c in cold]
    return {
        "model": cfg.name, "tp": world, "prewarmed_layers": k, "prompt_tokens": S, "steps": K,
        "collectives": "peer-memory kernels (IPC)" if peer_only else "NCCL (bf16 row-parallel partials)",
        "shard_gb": scfg.layout().total / 1e9,
        "cold_ttft_p50_ms": pct(cold_ttft, 50), "cold_ttft_p99_ms": pct(cold_ttft, 99),
        "warm_ttft_p50_ms": pct(warm, 50), "cold_over_warm_p50": pct(cold_ttft, 50) / pct(warm, 50),
        "stream_ms_p50_rank0": pct([c[1] for c in cold], 50),
        "streamed_gb_per_rank": cold[0][2] / 1e9,
        "prefill_ms": prefill_ms, "prefill_tokens_per_s": S / prefill_ms * 1e3,
        "prefill_tflops_per_gpu": cfg.prefill_flops(S) / world / (prefill_ms / 1e3) / 1e12,
        "ranks_agree_on_tokens": agree, "allreduce": ar, "setup_s": setup_s,
    }


def _placement(w, slot):
    import ctypes as C

    from paper_2512_09472_b200 import _native as N

    kind, nh = C.c_int32(), C.c_int64()
    N.call("ws_slot_placement", w.gpu.pool, slot.slot_id, C.byref(kind), C.byref(nh))
    return kind.value


def _handle_pages(w):
    import ctypes as C

    from paper_2512_09472_b200 import _native as N

    v = C.c_int64()
    N.call("ws_pool_handle_pages", w.gpu.pool, C.byref(v))
    return v.value


def _cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return f"x{os.cpu_count()}"


def main():
    # a stuck run leaves every thread's Python stack on stderr (WS_BENCH_WATCHDOG
    # seconds, default 1200; the whole default run takes ~4-5 min) instead of
    # an opaque timeout
    import faulthandler
    faulthandler.enable()
    wd = float(os.environ.get("WS_BENCH_WATCHDOG", "1200"))
    if wd > 0:
        faulthandler.dump_traceback_later(wd, exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--prompt", type=int, default=2048)
    ap.add_argument("--prewarm-layers", type=int, default=4)
    ap.add_argument("--pool-pages", type=int, default=0, help="0: all free HBM but --reserve-gib")
    ap.add_argument("--reserve-gib", type=float, default=24.0,
                    help="HBM left outside the pool: the 16 GB HBM-source stand-in, workspace, graphs")
    ap.add_argument("--switch-iters", type=int, default=200)
    ap.add_argument("--hbm-leg", action="store_true",
                    help="also time cold starts from an HBM-resident copy (the peer-source stand-in)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ttft-prompts", type=int, default=100)
    ap.add_argument("--tp-model", default="llama3-70b", help="model of the TP block (N >= 2 or --tp-block)")
    ap.add_argument("--tp-prewarm-layers", type=int, default=10)
    ap.add_argument("--tp-steps", type=int, default=5)
    ap.add_argument("--tp-block", action="store_true", help="run the TP block at N = 1 too (TP = 1)")
    ap.add_argument("--only-tp", action="store_true", help="test hook: run only the TP block")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--config5-policies", default="warmserve,no_prewarm",
                    help="BASELINE configs[4] live replay policies ('' to skip)")
    ap.add_argument("--config3-switches", type=int, default=1000,
                    help="BASELINE configs[2] switch burst length (0: skip)")
    ap.add_argument("--decode-ctx", type=int, default=1024)
    ap.add_argument("--decode-batches", type=lambda v: [int(x) for x in v.split(",") if x], default=[1, 16, 64])
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("WS_BENCH_ONE_GPU") == "1":
            # test hook: every rank on cuda:0 over gloo, to exercise the
            # multi-rank path (barriers, max-over-ranks) on a one-GPU box
            local_rank = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.only_tp:
        res = run_tp(args, rank, world, local_rank, peer_only=os.environ.get("WS_BENCH_ONE_GPU") == "1")
        if rank == 0:
            print(json.dumps({"tp_config4": res}), flush=True)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

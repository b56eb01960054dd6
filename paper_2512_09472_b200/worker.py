"""UniversalWorker — the north_star worker API on one B200:

    prewarm(model, layers)      prewarmed-weight pool with layer-granular residency
    switch_memory(model)        weight<->KV switch (VMM pages + switch kernel)
    activate_instance(model, …) layer-streamed cold-start prefill -> first token
    prefill(...) / decode(...)  on the paged KV pool

It composes the reference-protocol ``Cluster`` (ledger, role machine — the
reference engine can drive the same object) with the native model forward
and the layer streamer. Host-side bookkeeping follows the reference:
slot.layers_loaded / weight_bytes_loaded / required_prewarm_layers
(cluster.py:97-107, engine.py:658-686); activation timing decomposes like the
reference's startup breakdown (engine.py:557-597) but every term is measured.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import torch

from . import _native as N
from .cluster import Cluster, InstanceState, ModelSpec, PrewarmSlot, Role, required_prewarm_layers
from .devmem import view
from .models import PAGE, ModelConfig, model_spec


def _nvtx(fn):
    """NVTX range per worker op (prewarm / switch_memory / activate_instance /
    prefill / decode / reclaim / release), named ws.<op>: the op boundaries
    show up on an nsys / ncu timeline next to the kernels they issue."""
    import functools

    name = "ws." + fn.__name__

    @functools.wraps(fn)
    def wrapped(*a, **k):
        torch.cuda.nvtx.range_push(name)
        try:
            return fn(*a, **k)
        finally:
            torch.cuda.nvtx.range_pop()

    return wrapped


@dataclass
class ModelEntry:
    cfg: ModelConfig
    spec: ModelSpec
    layout: object
    host: torch.Tensor | None  # pinned bf16 image: cold-start source
    handle: C.c_void_p
    peer: torch.Tensor | None = None  # optional peer-device image (NVLink source)
    packed: object | None = None      # weights.PackedImage: the packed cold-start stream
    tp: object | None = None          # tp.TpGroup of a TP shard (None: single GPU)


@dataclass
class _Loader:
    """Background prewarm of one slot: a streamer whose ranges are the
    embedding, layers 0..L-1 and the final norm + lm_head (or only the
    first k + 1 of them when the prewarm stops at k)."""
    streamer: C.c_void_p
    n_ranges: int = 0   # ranges still tracked (0: settled / idle)
    full: bool = True
    k: int = 0


@dataclass
class ActivationResult:
    model: str
    token: int
    ttft_ms: float                 # host clock: call -> first token on host
    device_ms: float               # CUDA events: switch start -> token ready
    switch_ms: float               # host clock of the memory switch (ledger + kernel launch)
    switch_kernel_ms: float
    streamed_layers: int
    streamed_bytes: int            # bytes over the link (packed bytes on the packed stream)
    stream_ms: float               # copy stream: start -> last layer landed (unpacked)
    evicted: list = field(default_factory=list)
    seq: int = -1


class UniversalWorker:
    def __init__(self, device: int = 0, pool_pages: int = 12288, page_size: int = PAGE,
                 max_seqs: int = 64, max_tokens: int = 4096, bandwidth_gbs: float = 55.0):
        torch.cuda.set_device(device)
        self.device = device
        self.dev = torch.device("cuda", device)
        bw = bandwidth_gbs * 1e9 / 1e3  # bytes/ms, the reference's unit
        self.cluster = Cluster(1, 1, pool_pages, page_size, bw, devices={0: device})
        self.cluster.map_on_prewarm = False
        self.gpu = self.cluster.gpu(0)
        self.compute = torch.cuda.Stream(self.dev)
        self.copy = torch.cuda.Stream(self.dev)
        self.gpu.stream = self.compute.cuda_stream
        self.page_size = page_size
        self.max_tokens = max_tokens
        N.call("ws_pool_seq_config", self.gpu.pool, max_seqs, pool_pages)
        self.models: dict[str, ModelEntry] = {}
        self.instance = None
        self.active_model: str | None = None
        st = C.c_void_p()
        N.call("ws_streamer_create", 512, C.byref(st))
        self.streamer = st
        self._ws = None
        self._ws_bytes = 0
        self.logits = None
        self.next_tok = torch.zeros(256, dtype=torch.int32, device=self.dev)
        self.open_seqs: set[int] = set()
        self._graphs: dict = {}  # (model, batch, ctx bucket) -> (CUDAGraph, static seqs, pos, tokens)
        self.unpack = torch.cuda.Stream(self.dev)  # packed stream: rebuilds bf16 ranges in the slot
        self._staging = None
        self._loaders: dict[int, _Loader] = {}  # slot id -> background prewarm streamer

    # ------------------------------------------------------------ models
    def register(self, cfg: ModelConfig, host_weights: torch.Tensor | None, max_batch: int = 32,
                 tp=None) -> ModelEntry:
        """Register a model (or, with ``tp`` = a ``tp.TpGroup``, this rank's
        shard: ``cfg`` is then ``tp.shard_config(full, size)`` and the forward
        all-reduces on the TP boundary over NCCL). The per-GPU ledger holds the
        rank's shard as its slot; the cluster-level TP group (one instance over
        ``parallelism`` GPUs of one server) is the reference Cluster's job."""
        h = C.c_void_p()
        N.call("ws_model_create", C.byref(cfg.c()), self.device, C.byref(h))
        if tp is not None:
            N.call("ws_model_set_comm", h, tp.handle)
        spec = model_spec(cfg, max_batch=max_batch)
        e = ModelEntry(cfg, spec, cfg.layout(), host_weights, h, tp=tp)
        self.models[cfg.name] = e
        need = C.c_int64()
        N.call("ws_model_workspace_bytes", h, self.max_tokens, C.byref(need))
        if need.value > self._ws_bytes:
            self._ws = torch.empty(need.value, dtype=torch.uint8, device=self.dev)
            self._ws_bytes = need.value
        v = max(m.cfg.vocab for m in self.models.values())
        if self.logits is None or self.logits.numel() < 256 * v:
            self.logits = torch.empty(256 * v, dtype=torch.float32, device=self.dev)
        self._graphs.clear()  # captured decode steps hold the old workspace / logits pointers
        return e

    def set_packed(self, name: str, packed) -> None:
        """Attach a weights.PackedImage: cold activations of ``name`` then
        stream the packed ranges (fewer PCIe bytes) instead of the bf16 image."""
        self.models[name].packed = packed
        need = 2 * (-(-packed.max_range_bytes // 256) * 256)
        if self._staging is None or self._staging.numel() < need:
            self._staging = torch.empty(need, dtype=torch.uint8, device=self.dev)

    def set_gemm_impl(self, impl: int) -> None:
        for e in self.models.values():
            N.call("ws_model_set_gemm", e.handle, impl)

    def set_tp_fp32(self, name: str, on: bool) -> None:
        """TP row-parallel partials in fp32 over NCCL (default: bf16 on the wire)."""
        N.call("ws_model_set_tp_dtype", self.models[name].handle, int(bool(on)))

    def set_prune_last(self, name: str, on: bool) -> None:
        """Per-model opt-in: the last decoder layer runs attention, O and the
        FFN for the last prompt row only (every row's QKV + KV append still
        runs). A TP group must set the same value on every rank: the last
        layer's row-parallel collectives change size with it."""
        N.call("ws_model_set_prune_last", self.models[name].handle, int(bool(on)))

    def slot(self, name: str) -> PrewarmSlot | None:
        return self.gpu.slots.get(name)

    def weights_ptr(self, name: str) -> int:
        return self.slot(name).va

    def slot_view(self, name: str) -> torch.Tensor:
        e = self.models[name]
        return view(self.slot(name).va, (e.layout.total // 2,), torch.bfloat16, self.device)

    # ------------------------------------------------------------ prewarm
    @_nvtx
    def prewarm(self, name: str, layers: int | None = None, source: torch.Tensor | None = None,
                full: bool = True, wait: str | None = "ready", head: bool = False) -> PrewarmSlot:
        """prewarm(model, layers): take a slot (cluster.py:245-274) and start
        loading the model into it on the copy engine (engine.py:885-919).

        ``layers`` is the slot's required prefix k (``None``: the reference's
        stall-free k, required_prewarm_layers at the worker's bandwidth). With
        ``full=True`` (the reference's prewarm) the whole partition streams in
        the background, layer by layer — "ready" once k layers have landed,
        "full" at L (engine.py:658-686) — and the slot's ``layers_loaded`` /
        ``weight_bytes_loaded`` follow the per-layer copy events
        (``residency()``); ``full=False`` stops after k layers (a worker
        prewarmed to exactly k, BASELINE configs[1]); ``head=True`` with it
        also loads the final norm + lm_head (the reference's uniform
        layer_bytes folds the embedding and head into every layer,
        cluster.py:85-88 — with the head resident, a k-layer prefix holds about
        the reference's k x layer_bytes). ``wait``: "ready" (return once k
        layers are resident), "full", or None (return at once).

        One copy range per unit: the embedding, each decoder layer, then the
        final norm + lm_head; a windowed slot needs no driver call at all, a
        composite one maps its handles before the copies are queued."""
        e = self.models[name]
        if layers is None:
            layers = required_prewarm_layers(e.spec, self.cluster.bandwidth)
        L = e.cfg.layers
        layers = max(0, min(layers, L))
        pages = e.spec.partition_pages(self.page_size)
        slot = self.cluster.begin_prewarm(self.gpu, e.spec, pages, max(layers, 1))
        t0 = time.perf_counter()
        N.call("ws_slot_map_chunk", self.gpu.pool, slot.slot_id, 0, pages)
        map_ms = (time.perf_counter() - t0) * 1e3
        src = source if source is not None else e.host
        lay = e.layout
        units = [(0, 0, lay.layers[0]["begin"])] + [(x["begin"], x["begin"], x["end"] - x["begin"]) for x in lay.layers]
        units.append((lay.final_norm, lay.final_norm, lay.total - lay.final_norm))
        n = len(units) if full else layers + 1
        if not full and head:
            units = units[:layers + 1] + units[-1:]
            n += 1
        slot.layers_loaded = 0
        slot.weight_bytes_loaded = 0.0
        slot.load_start = time.perf_counter() * 1e3
        slot.load_finish = None
        slot.map_ms = map_ms
        if src is None:  # ledger/layout only (no weight image registered): nothing to copy
            slot.layers_loaded = layers if not full else L
            slot.weight_bytes_loaded = float(lay.prefix_bytes(slot.layers_loaded) if not full else lay.total)
            slot.prewarm_ms = map_ms
            return slot
        ld = self._loader_for(slot)
        flat = (C.c_int64 * (3 * n))(*[v for u in units[:n] for v in u])
        self.copy.wait_stream(self.compute)  # the slot's pages may have held KV a moment ago
        N.call("ws_streamer_start", ld.streamer, C.c_void_p(slot.va), C.c_void_p(src.data_ptr()), flat, n,
               C.c_void_p(self.copy.cuda_stream))
        ld.n_ranges, ld.full, ld.k = n, full, layers
        slot.head_resident = full or head
        if wait == "ready":  # range k = embedding + layers [0, k); k = L: everything
            N.call("ws_streamer_sync", ld.streamer, layers if layers < L else n - 1)
        elif wait == "full":
            N.call("ws_streamer_sync", ld.streamer, n - 1)
        self.residency(name)
        slot.prewarm_ms = (time.perf_counter() - t0) * 1e3
        return slot

    def _loader_for(self, slot) -> "_Loader":
        ld = self._loaders.get(slot.slot_id)
        if ld is None:
            st = C.c_void_p()
            N.call("ws_streamer_create", 512, C.byref(st))
            ld = self._loaders[slot.slot_id] = _Loader(st)
        return ld

    def residency(self, name: str) -> int:
        """Refresh the slot's layer residency from the copy events of its
        background prewarm (never blocks) and return ``layers_loaded`` — the
        measured counterpart of the reference's linear _slot_layers_at
        (engine.py:426-432): a layer counts once its bytes have landed."""
        slot = self.slot(name)
        if slot is None:
            return 0
        ld = self._loaders.get(slot.slot_id)
        if ld is None or ld.n_ranges == 0:
            return slot.layers_loaded
        d = C.c_int32()
        N.call("ws_streamer_progress", ld.streamer, C.byref(d))
        e = self.models[name]
        L = e.cfg.layers
        got = max(0, min(d.value - 1, L if ld.full else ld.k))
        slot.layers_loaded = max(slot.layers_loaded, got)
        head = e.layout.total - e.layout.final_norm if (not ld.full and slot.head_resident
                                                        and d.value == ld.n_ranges) else 0
        slot.weight_bytes_loaded = float(e.layout.prefix_bytes(slot.layers_loaded) + head) if d.value else 0.0
        if d.value == ld.n_ranges:  # every range landed: settle (engine.py:634-640)
            if ld.full:
                slot.layers_loaded = L
                slot.weight_bytes_loaded = float(e.layout.total)
            slot.load_finish = time.perf_counter() * 1e3
            ld.n_ranges = 0
        return slot.layers_loaded

    def _fence_loader(self, name: str) -> None:
        """A forward that does not ride the slot's background prewarm layer by
        layer waits (on the device) for all of it."""
        slot = self.slot(name)
        ld = self._loaders.get(slot.slot_id) if slot else None
        if ld is not None and ld.n_ranges:
            N.call("ws_streamer_wait", ld.streamer, ld.n_ranges - 1, C.c_void_p(self.compute.cuda_stream))
            self.residency(name)

    def wait_resident(self, name: str, layers: int | None = None) -> int:
        """Block until ``layers`` (default: everything the prewarm loads) are resident."""
        slot = self.slot(name)
        ld = self._loaders.get(slot.slot_id) if slot else None
        if ld is not None and ld.n_ranges:
            N.call("ws_streamer_sync", ld.streamer, ld.n_ranges - 1 if layers is None else min(layers, ld.n_ranges - 1))
        return self.residency(name)

    @_nvtx
    def evict(self, name: str):
        """evict_slot (cluster.py:276-289) on this worker: copies still landing
        in the slot are fenced on the compute stream first (its pages may
        become another slot or KV next), then the pages return to the free
        list and the VA is unmapped in the background."""
        slot = self.slot(name)
        if slot is None:
            return None
        ld = self._loaders.get(slot.slot_id)
        if ld is not None and ld.n_ranges:
            N.call("ws_streamer_wait", ld.streamer, ld.n_ranges - 1, C.c_void_p(self.compute.cuda_stream))
            ld.n_ranges = 0
        return self.cluster.evict_slot(self.gpu, name)

    def drop_suffix(self, name: str, layers: int, head: bool = False) -> None:
        """Forget residency of layers >= ``layers`` (and of the final norm +
        lm_head unless ``head``): bytes stay, the ledger says they are gone,
        so the next activation streams them again."""
        self.wait_resident(name)
        s = self.slot(name)
        e = self.models[name]
        s.layers_loaded = layers
        s.head_resident = head
        s.weight_bytes_loaded = float(e.layout.prefix_bytes(layers)
                                      + (e.layout.total - e.layout.final_norm if head else 0))

    # ------------------------------------------------------------ switch
    @_nvtx
    def switch_memory(self, name: str):
        """Weight->KV memory switch (promote_to_dedicated, cluster.py:291-342):
        evict other slots (async VMM unmap), every free page becomes KV via the
        switch kernel, no driver call on this path. Returns (inst, evicted,
        host_ms, kernel_ms)."""
        e = self.models[name]
        # In-flight prewarm copies into slots this promote evicts must land
        # before those pages become KV; the promoted slot's own background
        # load keeps streaming (activate_instance waits on it layer by layer).
        for other, s_ in self.gpu.slots.items():
            ld = self._loaders.get(s_.slot_id)
            if other != name and ld is not None and ld.n_ranges:
                N.call("ws_streamer_wait", ld.streamer, ld.n_ranges - 1, C.c_void_p(self.compute.cuda_stream))
                ld.n_ranges = 0
        t0 = time.perf_counter()
        inst, evicted = self.cluster.promote_to_dedicated((0,), e.spec, self.slot(name).required_prewarm_layers
                                                          if self.slot(name) else 1)
        host_ms = (time.perf_counter() - t0) * 1e3
        kms, ent = C.c_double(), C.c_int64()
        N.call("ws_pool_last_switch", self.gpu.pool, C.byref(kms), C.byref(ent))
        self.instance = inst
        self.active_model = name
        return inst, evicted, host_ms, kms.value

    def kv_used_bytes(self) -> int:
        """Device truth for the reference's _kv_used_bytes (engine.py:391-404):
        the bytes of the KV pages that hold live blocks of open sequences (the
        reference counts tokens x kv_bytes_per_token; a page is the block, so
        this is the token count rounded up per sequence to whole blocks —
        exactly the pages a shrink must keep)."""
        return self.gpu.counts().kv_pages_allocated * self.page_size

    @_nvtx
    def reclaim(self, inflight: int, kv_used_bytes: float | None = None) -> int:
        """KV->weights switch on a draining worker (cluster.py:351-365).
        ``kv_used_bytes=None`` takes the pool's live blocks (kv_used_bytes())."""
        if self.gpu.role == Role.DEDICATED:
            self.cluster.enter_grace(self.instance)
        used = self.kv_used_bytes() if kv_used_bytes is None else kv_used_bytes
        return self.cluster.reclaim_on_completion(self.gpu, inflight, self.instance.max_batch, used)

    @_nvtx
    def release(self) -> None:
        """End of grace (cluster.py:367-387): KV pages back to free, slots kept."""
        for s in list(self.open_seqs):
            self.close_seq(s)
        if self.instance is None:
            return
        if self.instance.state != InstanceState.GRACE:
            if self.instance.state == InstanceState.STARTING:
                self.instance.state = InstanceState.ACTIVE
            self.cluster.enter_grace(self.instance)
        self.cluster.release_instance(self.instance)
        self.instance = None
        self.active_model = None

    # ------------------------------------------------------------ sequences
    def open_seq(self, n_tokens: int) -> int:
        s = C.c_int32()
        N.call("ws_seq_open", self.gpu.pool, C.byref(s))
        self.open_seqs.add(s.value)
        self.reserve(s.value, n_tokens)
        return s.value

    def reserve(self, seq: int, n_tokens: int) -> None:
        tpb, _ = self.models[self.active_model].cfg.kv_geometry(self.page_size)
        N.call("ws_seq_reserve", self.gpu.pool, seq, -(-n_tokens // tpb), self.compute.cuda_stream)

    def close_seq(self, seq: int) -> None:
        N.call("ws_seq_close", self.gpu.pool, seq)
        self.open_seqs.discard(seq)

    # ------------------------------------------------------------ compute
    @_nvtx
    def prefill(self, seq: int, tokens_dev: torch.Tensor, pos0: int = 0, stream_from: int | None = None,
                streamer=None):
        """Prefill on the paged pool; returns (logits view [vocab], next-token device scalar).
        ``stream_from``: layer l >= stream_from waits for range l - stream_from
        of ``streamer`` (default: the worker's activation streamer)."""
        e = self.models[self.active_model]
        rows = tokens_dev.numel()
        if rows > self.max_tokens:  # the workspace is sized for max_tokens rows
            raise ValueError(f"prefill of {rows} tokens exceeds this worker's max_tokens={self.max_tokens}")
        st = (streamer or self.streamer) if stream_from is not None else None
        if st is None:
            self._fence_loader(e.cfg.name)
        caller = torch.cuda.current_stream(self.dev)
        if caller != self.compute:
            self.compute.wait_stream(caller)  # inputs produced on the caller's stream
        N.call("ws_model_prefill", e.handle, self.gpu.pool, C.c_void_p(self.slot(e.cfg.name).va), seq,
               C.c_void_p(tokens_dev.data_ptr()), rows, pos0, st, stream_from or 0,
               C.c_void_p(self._ws.data_ptr()), C.c_void_p(self.logits.data_ptr()),
               C.c_void_p(self.next_tok.data_ptr()), C.c_void_p(self.compute.cuda_stream))
        if caller != self.compute:
            caller.wait_stream(self.compute)  # outputs visible to the caller's stream
        return self.logits[: e.cfg.vocab], self.next_tok[:1]

    @_nvtx
    def decode(self, seqs_dev: torch.Tensor, pos_dev: torch.Tensor, tokens_dev: torch.Tensor, max_ctx: int):
        e = self.models[self.active_model]
        n = seqs_dev.numel()
        if n > self.max_tokens:
            raise ValueError(f"decode batch {n} exceeds this worker's max_tokens={self.max_tokens}")
        if not torch.cuda.is_current_stream_capturing():  # decode_graphed fences before capturing
            self._fence_loader(e.cfg.name)
        caller = torch.cuda.current_stream(self.dev)
        if caller != self.compute:
            self.compute.wait_stream(caller)
        N.call("ws_model_decode", e.handle, self.gpu.pool, C.c_void_p(self.slot(e.cfg.name).va),
               C.c_void_p(seqs_dev.data_ptr()), C.c_void_p(pos_dev.data_ptr()),
               C.c_void_p(tokens_dev.data_ptr()), n, max_ctx, C.c_void_p(self._ws.data_ptr()),
               C.c_void_p(self.logits.data_ptr()), C.c_void_p(self.next_tok.data_ptr()),
               C.c_void_p(self.compute.cuda_stream))
        if caller != self.compute:
            caller.wait_stream(self.compute)
        return self.logits[: n * e.cfg.vocab].view(n, e.cfg.vocab), self.next_tok[:n]

    @_nvtx
    def decode_graphed(self, seqs_dev: torch.Tensor, pos_dev: torch.Tensor, tokens_dev: torch.Tensor,
                       max_ctx: int, ctx_bucket: int = 256):
        """decode() replayed from a CUDA graph: the step's 8-11 kernels per layer
        (PDL edges included) go out as one launch, so a small batch is not
        bound by host launch issue. One graph per (model, batch, context
        bucket): the attention grid is sized for the bucket and every CTA
        clips to its sequence's length, so results equal decode() with
        max_ctx = the bucket. Inputs are copied into the graph's static
        buffers on the compute stream."""
        tp = self.models[self.active_model].tp
        if tp is not None and getattr(tp, "peer", None) is not None:
            # The peer allreduce advances its epoch and picks its double-buffered
            # slot on the host at launch time; a graph would freeze both and a
            # replay could read peers' slots before they are written.
            raise RuntimeError("decode_graphed: a TP model on the peer-memory allreduce cannot be graph-captured "
                               "(host-side epochs); use decode()")
        n = seqs_dev.numel()
        cap = -(-max_ctx // ctx_bucket) * ctx_bucket
        key = (self.active_model, n, cap)
        ent = self._graphs.get(key)
        caller = torch.cuda.current_stream(self.dev)
        if caller != self.compute:
            self.compute.wait_stream(caller)
        if ent is None:
            st = [torch.empty_like(seqs_dev), torch.empty_like(pos_dev), torch.empty_like(tokens_dev)]
            with torch.cuda.stream(self.compute):
                for d, s in zip(st, (seqs_dev, pos_dev, tokens_dev)):
                    d.copy_(s)
                self.decode(*st, cap)  # first use allocates the split-K scratch outside the capture
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.compute):
                    self.decode(*st, cap)
            ent = self._graphs[key] = (g, *st)
        g, s_seqs, s_pos, s_tok = ent
        with torch.cuda.stream(self.compute):
            s_seqs.copy_(seqs_dev, non_blocking=True)
            s_pos.copy_(pos_dev, non_blocking=True)
            s_tok.copy_(tokens_dev, non_blocking=True)
            g.replay()
        if caller != self.compute:
            caller.wait_stream(self.compute)
        vocab = self.models[self.active_model].cfg.vocab
        return self.logits[: n * vocab].view(n, vocab), self.next_tok[:n]

    # ------------------------------------------------------------ activation
    @_nvtx
    def activate_instance(self, name: str, prompt_host: torch.Tensor, source: torch.Tensor | None = None,
                          keep_seq: bool = False) -> ActivationResult:
        """Cold (or warm) start: switch memory, stream the non-resident layers
        on the copy engine, prefill the prompt with per-layer waits, return
        the first token on the host. prompt_host: pinned int32 tokens."""
        e = self.models[name]
        if source is not None and hasattr(source, "tensor"):  # a peer_source.PeerSource
            source = source.tensor
        if not 1 <= prompt_host.numel() <= self.max_tokens:  # checked before any state changes
            raise ValueError(f"prompt of {prompt_host.numel()} tokens: need 1..max_tokens={self.max_tokens}")
        L = e.cfg.layers
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record(self.compute)
        self.residency(name)
        inst, evicted, sw_ms, sw_kernel_ms = self.switch_memory(name)
        slot = self.slot(name)
        k = slot.layers_loaded
        stream_from = None
        streamer = None
        streamed = 0
        ld = self._loaders.get(slot.slot_id)
        if ld is not None and ld.n_ranges and ld.full:
            # The slot's background prewarm is still landing: prefill rides it,
            # layer l waiting for that prewarm's range l + 1 (range 0 is the
            # embedding) — no second copy of anything.
            N.call("ws_streamer_wait", ld.streamer, 0, C.c_void_p(self.compute.cuda_stream))
            streamer, stream_from = ld.streamer, -1
            streamed = int(e.layout.total - e.layout.prefix_bytes(k))
            k = L
        elif ld is not None and ld.n_ranges:
            # a prefix-only prewarm still landing: wait for its last range, stream the rest
            N.call("ws_streamer_wait", ld.streamer, ld.n_ranges - 1, C.c_void_p(self.compute.cuda_stream))
            k = ld.k
            ld.n_ranges = 0
        # The embedding kernel reads the pinned prompt straight from host
        # memory (mapped under UVA; the same PCIe bytes, no copy engine): a
        # prompt H2D copy queued on a copy engine behind the weight stream (or
        # behind a background prewarm still landing) held the whole prefill
        # until the stream drained — measured device time 34.9 vs 56.3 ms at
        # k = 30, bimodal with the engine the two streams happened to share.
        seq = self.open_seq(prompt_host.numel() + 1)
        if prompt_host.is_pinned():
            toks = prompt_host
        else:
            with torch.cuda.stream(self.compute):
                toks = prompt_host.to(self.dev, non_blocking=True)
        if k < L and source is None and e.packed is not None:
            rows = e.packed.rows(k)
            if slot.head_resident:
                rows = rows[:-1]  # final norm + lm_head already resident
            flat = (C.c_int64 * (6 * len(rows)))(*[v for r in rows for v in r])
            self.copy.wait_stream(self.compute)  # copy after the switch (pages owned)
            self.unpack.wait_stream(self.compute)
            N.call("ws_streamer_start_packed", self.streamer, C.c_void_p(slot.va),
                   C.c_void_p(e.packed.blob.data_ptr()), flat, len(rows), C.c_void_p(self._staging.data_ptr()),
                   self._staging.numel(), C.c_void_p(self.copy.cuda_stream), C.c_void_p(self.unpack.cuda_stream))
            stream_from = k
            streamed = sum(r[5] for r in rows)
            n_ranges = len(rows)
        elif k < L:
            src = source if source is not None else e.host
            ranges = e.layout.stream_ranges(k)
            if slot.head_resident:
                ranges = ranges[:-1]
            flat = (C.c_int64 * (3 * len(ranges)))(*[v for r in ranges for v in r])
            self.copy.wait_stream(self.compute)  # copy after the switch (pages owned)
            N.call("ws_streamer_start", self.streamer, C.c_void_p(slot.va), C.c_void_p(src.data_ptr()),
                   flat, len(ranges), C.c_void_p(self.copy.cuda_stream))
            stream_from = k
            streamed = sum(r[2] for r in ranges)
            n_ranges = len(ranges)
        _, nt = self.prefill(seq, toks, 0, stream_from, streamer)
        with torch.cuda.stream(self.compute):
            out = torch.empty(1, dtype=torch.int32, pin_memory=True)
            out.copy_(nt, non_blocking=True)
        ev1.record(self.compute)
        ev1.synchronize()
        ttft = (time.perf_counter() - t0) * 1e3
        stream_ms = 0.0
        if ld is not None and ld.n_ranges:
            ld.n_ranges = 0  # every range landed before the prefill finished
        if stream_from is not None and streamer is None:
            times = (C.c_float * n_ranges)()
            N.call("ws_streamer_times", self.streamer, times, n_ranges)
            stream_ms = times[n_ranges - 1]
        slot.layers_loaded = L
        slot.head_resident = True
        slot.weight_bytes_loaded = float(e.layout.total)
        inst.state = InstanceState.ACTIVE
        if not keep_seq:
            self.close_seq(seq)
        return ActivationResult(name, int(out.item()), ttft, ev0.elapsed_time(ev1), sw_ms, sw_kernel_ms,
                                L - k, streamed, stream_ms, evicted, seq if keep_seq else -1)

    def close(self) -> None:
        torch.cuda.synchronize(self.dev)
        for e in self.models.values():
            if e.handle:
                N.fns["ws_model_destroy"](e.handle)
                e.handle = None
        if self.streamer:
            N.fns["ws_streamer_destroy"](self.streamer)
            self.streamer = None
        for ld in self._loaders.values():
            N.fns["ws_streamer_destroy"](ld.streamer)
        self._loaders.clear()
        if self.gpu.pool:  # the pool's HBM goes back now, not at garbage collection
            N.fns["ws_pool_destroy"](self.gpu.pool)
            self.gpu.pool = None
        self._ws = self.logits = self._staging = None

/*
 * warmserve.h — C-ABI of the B200-native universal-GPU-worker data path.
 *
 * The reference (prewarmsim, /root/reference/pkg) is a pure-Python simulator
 * with no FFI; its drop-in seam is the Python `Cluster` object protocol plus
 * the memswitch / planning functions. Each entry point below
 * cites the reference interface it replaces. The Python package
 * `paper_2512_09472_b200` binds these with ctypes and re-exposes the
 * reference's Cluster protocol on top (INTEGRATION.md shows the binding).
 *
 * Conventions: plain pointers and sizes only; every function returns a
 * WS_* status (0 = ok) and writes results through out-pointers;
 * ws_last_error() returns the thread's last error text. Device pointers are
 * CUDA device addresses; `stream` arguments are cudaStream_t passed as void*.
 * Single writer: all pool/ledger calls for one pool come from one host thread
 * (cluster.py:200-201); only the internal unmap worker runs concurrently.
 */
#ifndef WARMSERVE_H_
#define WARMSERVE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to ClusterError / ValueError by the mirror) ---- */
#define WS_OK 0
#define WS_ERR_INVALID 1          /* ValueError in the reference               */
#define WS_ERR_INSUFFICIENT 2     /* "insufficient pages" cluster.py:259-263    */
#define WS_ERR_DUPLICATE 3        /* "already holds a slot" cluster.py:255-258  */
#define WS_ERR_NO_SLOT 4          /* unknown slot id                            */
#define WS_ERR_STATE 5            /* op illegal in the pool's current state     */
#define WS_ERR_CUDA 6             /* CUDA runtime / driver failure              */
#define WS_ERR_NO_DEVICE 7        /* device op on a ledger-only pool            */
#define WS_ERR_KV_BUSY 8          /* KV shrink would drop live blocks           */
#define WS_ERR_FRAGMENTED 9       /* device pool: no slot placement exists at   *
                                   * the physical handle granularity            */

const char* ws_last_error(void);
int ws_version(int* major, int* minor);
/* Kernel launches issued by this library since load (evidence for gpu_launches). */
int ws_kernel_launches(int64_t* out);
/* Launches that fell back to a legacy kernel because the shape is outside the
 * tcgen05 tilings, by kind: [0] GEMM on mma.sync, [1] GEMM on the CUDA-core
 * GEMV, [2] prefill attention on mma.sync. Explicit A/B selections
 * (ws_model_set_gemm) are not fallbacks and are not counted. */
int ws_fallback_counts(int64_t* out, int32_t n);

/* ======================================================================
 * Planning math — bit-exact float64 restatements of the reference's
 * analytic model, used by the worker to size prewarm prefixes and by the
 * engine adapter. All verified against golden vectors of the reference.
 * ==================================================================== */

/* cluster.py:145-166 required_prewarm_layers(spec, bandwidth, ref_input_tokens) */
int ws_required_prewarm_layers(int64_t weight_bytes, int32_t parallelism, int32_t layers,
                               double prefill_a_ms, double prefill_b_ms, double bandwidth,
                               int32_t ref_input_tokens, int32_t* k_out);

/* cluster.py:169-182 catchup_stall_ms(spec, layers_loaded, bandwidth, ref_input_tokens) */
int ws_catchup_stall_ms(int64_t weight_bytes, int32_t parallelism, int32_t layers,
                        double prefill_a_ms, double prefill_b_ms, int32_t layers_loaded,
                        double bandwidth, int32_t ref_input_tokens, double* stall_out);

/* cluster.py:185-197 reservation_target(M, C, R, K) = max(M*R/C, K + M/C) */
int ws_reservation_target(double kv_capacity_bytes, int32_t max_batch, int32_t inflight,
                          double kv_used_bytes, double* target_out);

/* cluster.py:79-83 ModelSpec.partition_bytes / partition_pages */
int ws_partition_pages(int64_t weight_bytes, int32_t parallelism, int64_t page_size,
                       int64_t* partition_bytes_out, int64_t* partition_pages_out);

typedef struct ws_transfer_plan {
  int64_t total_bytes;
  double bandwidth;          /* bytes / ms */
  int64_t chunk_pages;
  int64_t page_size;
  int64_t n_chunks;
  double first_chunk_map_ms;
  double finish_ms;
  double critical_path_stall_ms;
} ws_transfer_plan;

/* memswitch.py:59-98 pipelined_load + kernels.py:68-77 pipeline_finish */
int ws_pipelined_load(int64_t total_bytes, double bandwidth, double map_ms_per_page,
                      int64_t chunk_pages, int64_t page_size, ws_transfer_plan* out);

/* memswitch.py:101-117 background_kv_mapping */
int ws_background_kv_mapping(int64_t pages, double map_ms_per_page, double consumption_rate,
                             double* stall_out);

/* ======================================================================
 * Page pool — one per GPU worker. Replaces the page ledger of
 * GpuWorker (cluster.py:110-129) and the physical effects of the Cluster
 * operations that touch it. device < 0 gives a ledger-only pool (host
 * bookkeeping, identical page identities, no CUDA calls).
 *
 * Device pools back the ledger's pages with physical handles of
 * `handle_pages` pages each (cuMemCreate; default 64 x 2 MiB = 128 MiB — the
 * driver's cost is per handle, so a full-HBM pool builds in about a second),
 * all mapped once, in page order, into one "page window" VA at init (page p
 * at window + p*page_size). KV blocks address pages through the window, so
 * converting pages between weight slots and the KV cache never calls the
 * driver (PAPER.md:420-453 slots, engine.py:615-632 async unmap).
 *
 * Page identity rules (documented, deterministic; the reference pins only
 * counts): a new slot takes (1) for a keyed slot, the run of pages it held
 * last time if that run is free; else (2) the lowest contiguous run of free
 * pages — a WINDOWED slot whose VA is window + first*page_size, created and
 * evicted with zero driver calls; else (3) a COMPOSITE placement: the longest
 * free suffix of one handle, then whole free handles (lowest first), then
 * the shortest sufficient free prefix of one more handle, each handle mapped
 * whole into a private VA reservation (unmapped asynchronously on evict);
 * else a device pool fails with WS_ERR_FRAGMENTED and a ledger-only pool
 * takes the lowest free pages. Promotion turns every free page into KV; a
 * KV shrink returns the highest-id KV pages, migrating any live KV block that
 * sits on one of them to the lowest-id unallocated KV page that stays.
 * ==================================================================== */
typedef struct ws_pool ws_pool;

typedef struct ws_pool_counts {
  int64_t total_pages;
  int64_t free_pages;        /* cluster.py:127-129 */
  int64_t slot_pages;        /* cluster.py:123-125 */
  int64_t kv_pages_mapped;   /* cluster.py:118     */
  int64_t kv_pages_used;     /* cluster.py:119     */
  int64_t kv_capacity_pages; /* cluster.py:120     */
  int64_t kv_pages_allocated;/* pages holding live KV blocks of open sequences */
  int64_t n_slots;
  int64_t pending_unmaps;
} ws_pool_counts;

int ws_pool_create(int32_t device, int64_t total_pages, int64_t page_size, ws_pool** out);
/* Same with an explicit physical handle size in pages (ws_pool_create: 64). */
int ws_pool_create_ex(int32_t device, int64_t total_pages, int64_t page_size, int64_t handle_pages,
                      ws_pool** out);
int ws_pool_handle_pages(ws_pool* pool, int64_t* handle_pages_out);
int ws_pool_destroy(ws_pool* pool);
int ws_pool_counts_get(ws_pool* pool, ws_pool_counts* out);
/* Host copy of the page-ownership map: -1 free, -2 KV, >=0 owning slot id. */
int ws_pool_owner_map(ws_pool* pool, int32_t* out, int64_t n);
/* Device copy of the same map (device pools only), for parity checks. */
int ws_pool_device_owner_map(ws_pool* pool, int32_t* host_out, int64_t n);
/* Base of the page window (page p lives at base + p*page_size). */
int ws_pool_window(ws_pool* pool, void** base_out);
/* Measured driver cost (ms) of the pool init, of slot mapping per slot page
 * placed on the device so far (windowed slots count as 0 — the memswitch.py
 * μ this hardware achieves), and of the last async unmap per page. */
int ws_pool_timing(ws_pool* pool, double* init_ms, double* map_ms_per_slot_page,
                   double* last_unmap_ms_per_page);
/* Wait for the background unmap worker to drain. */
int ws_pool_sync_unmaps(ws_pool* pool);

/* begin_prewarm (cluster.py:245-274): reserve a slot VA, take `pages` pages.
 * map_now=1 maps all of them before returning (device pools); map_now=0 lets
 * the caller drive ws_slot_map_chunk() from the pipelined loader. */
int ws_slot_create(ws_pool* pool, int64_t slot_id, int64_t pages, int32_t map_now, void** va_out);
/* Same, with a per-model key (nonzero): the model's next slot takes back the
 * page run its last windowed slot held if that run is free (rule 1 above). */
int ws_slot_create_keyed(ws_pool* pool, int64_t slot_id, int64_t pages, int32_t map_now, uint64_t key,
                         void** va_out);
/* Slot pages mapped by the driver (composite) vs addressed through the page
 * window with no driver call (windowed), since create. */
int ws_pool_map_stats(ws_pool* pool, int64_t* remapped_pages, int64_t* reused_pages);
/* Map pages [first, first+count) of the slot into its VA (memswitch.py:78-88
 * per-chunk map step). */
int ws_slot_map_chunk(ws_pool* pool, int64_t slot_id, int64_t first, int64_t count);
/* evict_slot (cluster.py:276-289): pages return to the free list now, the
 * slot VA is unmapped asynchronously after `fence_stream` drains (may be NULL). */
int ws_slot_evict(ws_pool* pool, int64_t slot_id, void* fence_stream);
int ws_slot_info(ws_pool* pool, int64_t slot_id, int64_t* pages_out, int64_t* mapped_out, void** va_out);
int ws_slot_pages(ws_pool* pool, int64_t slot_id, int32_t* ids_out, int64_t cap, int64_t* n_out);
/* ---- peer-HBM weight source ----
 * Export the physical handles covering a WINDOWED slot as POSIX fds (the
 * pool's handles are created exportable when the system supports it): fds[i]
 * and sizes[i] (bytes) for each handle, offset_out = the slot's byte offset in
 * the first one. The fds belong to the caller (send them to the peer process,
 * e.g. SCM_RIGHTS, then close). */
int ws_pool_export_slot(ws_pool* pool, int64_t slot_id, int32_t* fds, int64_t* sizes, int64_t cap,
                        int64_t* n_out, int64_t* offset_out);
/* Import exported handles into this process and map them, read-only, for
 * `device`: a device pointer to the peer's memory (over NVLink when the
 * exporter is another GPU). The layer streamer copies from it
 * (ws_streamer_start src_base). The caller still owns / closes the fds. */
typedef struct ws_peer_map ws_peer_map;
int ws_peer_map_import(int32_t device, const int32_t* fds, const int64_t* sizes, int64_t n, void** va_out,
                       ws_peer_map** out);
int ws_peer_map_release(ws_peer_map* map);
int ws_device_can_access_peer(int32_t device, int32_t peer_device, int32_t* out);

/* Placement of a slot: kind 0 windowed, 1 composite, 2 scattered (ledger-only
 * pools); handles_out = physical handles a composite slot maps. */
int ws_slot_placement(ws_pool* pool, int64_t slot_id, int32_t* kind_out, int64_t* handles_out);

/* promote_to_dedicated KV step (cluster.py:332-338): every free page becomes
 * KV; capacity = mapped = the resulting KV page count. */
int ws_kv_map_all(ws_pool* pool, void* stream, int64_t* kv_pages_out);
/* reclaim_on_completion (cluster.py:351-365) page math + the shrink. */
int ws_kv_reclaim(ws_pool* pool, int32_t inflight, int32_t max_batch, double kv_used_bytes,
                  void* stream, int64_t* freed_bytes_out);
/* Set kv_pages_mapped to an explicit count (grow from free / shrink). */
int ws_kv_resize(ws_pool* pool, int64_t kv_pages, void* stream);
/* release_instance KV step (cluster.py:377-381): all KV pages to free. */
int ws_kv_release(ws_pool* pool, void* stream);

/* ---- sequences on the paged KV pool (block = one page) ---- */
/* Device block-table matrix [max_seqs, max_blocks] of int32 page ids. */
int ws_pool_seq_config(ws_pool* pool, int32_t max_seqs, int32_t max_blocks);
int ws_seq_open(ws_pool* pool, int32_t* seq_out);
/* Ensure blocks for `n_blocks` total blocks; allocates lowest-id free KV pages. */
int ws_seq_reserve(ws_pool* pool, int32_t seq, int32_t n_blocks, void* stream);
int ws_seq_close(ws_pool* pool, int32_t seq);
int ws_seq_blocks(ws_pool* pool, int32_t seq, int32_t* ids_out, int32_t cap, int32_t* n_out);
int ws_pool_block_tables(ws_pool* pool, int32_t** dev_out, int32_t* max_blocks_out);

/* Time (ms, CUDA events on `stream`) of the last switch kernel launch. */
int ws_pool_last_switch(ws_pool* pool, double* kernel_ms_out, int64_t* entries_out);

/* ======================================================================
 * Layer streaming — the copy side of activate_instance(): copy byte ranges
 * (layers k..L of a prewarmed slot) from pinned host memory or a peer
 * device into the slot on a copy stream, one CUDA event per range; the
 * compute stream waits per layer (engine.py:526-538 "cold" branch and
 * cluster.py:169-182 catch-up semantics made physical).
 * ==================================================================== */
typedef struct ws_streamer ws_streamer;
int ws_streamer_create(int32_t max_ranges, ws_streamer** out);
int ws_streamer_destroy(ws_streamer* s);
/* Enqueue copies of ranges[i] = {dst_offset, src_offset, bytes} (int64 x3). */
int ws_streamer_start(ws_streamer* s, void* dst_base, const void* src_base, const int64_t* ranges,
                      int32_t n_ranges, void* copy_stream);
/* Packed stream (same per-range events): ranges stored losslessly packed on
 * the host (bf16 = sign|mantissa byte + exponent as a canonical Huffman
 * code, or as a 4-bit code relative to a per-range base + escape list;
 * layouts in kernels/unpack.cu). desc[i] = {dst_offset, packed_offset,
 * n_values, e_base (-1 = Huffman), n_escapes, packed_bytes}
 * (int64 x6). The copy engine moves each packed range into one of two
 * halves of `staging` (device, 256-byte aligned) on copy_stream; a kernel on
 * unpack_stream rebuilds the exact bf16 bytes at dst_base + dst_offset.
 * Replaces the same cold-start copy as ws_streamer_start (engine.py:526-538)
 * with ~34% (Huffman) / ~25% (4-bit) fewer PCIe bytes. */
int ws_streamer_start_packed(ws_streamer* s, void* dst_base, const void* packed_base, const int64_t* desc,
                             int32_t n_ranges, void* staging, int64_t staging_bytes, void* copy_stream,
                             void* unpack_stream);
/* Make `stream` wait until range i has landed (no-op if i >= started). */
int ws_streamer_wait(ws_streamer* s, int32_t i, void* stream);
/* Host-side residency: number of leading ranges already landed (event
 * query, never blocks) — the per-layer "layers_loaded" progress of a
 * background prewarm (engine.py:426-432, 658-686). */
int ws_streamer_progress(ws_streamer* s, int32_t* done_out);
/* Block the host until range i has landed (the "ready" / "full" stages). */
int ws_streamer_sync(ws_streamer* s, int32_t i);
/* ms from start to each range's completion (after sync). */
int ws_streamer_times(ws_streamer* s, float* ms_out, int32_t n);

/* ======================================================================
 * Model forward on the paged pool — the compute half of
 * activate_instance() and the prefill/decode the reference models with
 * LatencyModel (engine.py:97-116, a18) and _kv_used_bytes (engine.py:391-404).
 * Llama-family decoder (RMSNorm, RoPE rotate_half, GQA, SwiGLU), bf16
 * weights, fp32 residual stream, sm_100a kernels.
 * ==================================================================== */
typedef struct ws_model_config {
  int32_t layers, hidden, ffn, heads, kv_heads, head_dim, vocab;
  float rope_theta, rms_eps;
  int32_t qkv_bias;       /* Qwen2.5-style q/k/v biases */
  int32_t max_positions;  /* RoPE table length */
  int32_t lm_head_rows;   /* vocab-parallel lm_head shard rows (0 = vocab) */
} ws_model_config;

/* ---- tensor parallelism (config 4): NCCL communicator, created once at
 * prewarm time. With a communicator set on a model, the
 * row-parallel O and down projections write fp32 partials that are
 * all-reduced (sum) before the residual add, and the vocab-parallel lm_head
 * shards are all-gathered into full logits. ---- */
typedef struct ws_comm ws_comm;
int ws_nccl_unique_id(uint8_t* out, int32_t n);  /* n >= 128 */
int ws_comm_create(const uint8_t* unique_id, int32_t rank, int32_t nranks, int32_t device, ws_comm** out);
int ws_comm_destroy(ws_comm* comm);

/* Allreduce (fp32 sum) over peer memory: every rank exports one buffer
 * (cudaIpcMemHandle_t, 64 bytes) and maps every peer's; a call copies the
 * local partial into the rank's own buffer and one kernel signals the peers,
 * waits for theirs, and sums all ranks' partials in rank order (bit-identical
 * on every rank). Replaces ncclAllReduce for the row-parallel O / down
 * partials (TP, config 4; reference: the NCCL-free cost model of
 * PAPER.md:686-689 / SURVEY §8e). Every rank must issue the same sequence of
 * calls. */
typedef struct ws_peer ws_peer;
int ws_peer_buffer_bytes(int64_t max_count, int64_t* out);
int ws_peer_buffer_alloc(int64_t max_count, void** ptr, uint8_t* handle, int32_t handle_bytes);
int ws_peer_buffer_free(void* ptr);
int ws_peer_buffer_open(const uint8_t* handle, void** ptr);
int ws_peer_buffer_close(void* ptr);
int ws_peer_create(int32_t rank, int32_t world, void* const* bufs, int64_t max_count, ws_peer** out);
int ws_peer_destroy(ws_peer* p);
int ws_peer_allreduce_f32(ws_peer* p, float* buf, int64_t count, void* stream);
/* Fused form for a row-parallel projection: the GEMM writes its fp32 partial
 * straight into the rank's next exported slot (ws_peer_next_slot), then
 * ws_peer_reduce_add_f32 does x += sum over ranks in one kernel — no staging
 * copy and no separate residual-add launch. */
int ws_peer_next_slot(ws_peer* p, float** slot);
int ws_peer_reduce_add_f32(ws_peer* p, float* x, int64_t count, void* stream);
/* Row-parallel projection fused with its allreduce (replaces the
 * reference's TP sync term engine.py:110-113): x[M, N] += sum over ranks of
 * A_r[M, K] W_r[N, K]^T. For prefill-sized shapes (M >= 256, N % 256 == 0,
 * K % 64 == 0) the CTA-pair tcgen05 GEMM stores its bf16 partial into the
 * exported slot and publishes every 128 x 256 block with a system-scope flag;
 * a reduce kernel running beside it (programmatic dependent launch) has the
 * block's owner rank sum the W partials in rank order as soon as they are all
 * published, and every rank add the owner's reduced block into x — the link
 * traffic (2(W-1)/W of the bf16 partial per rank) overlaps the GEMM tile by
 * tile. Other shapes: fp32 partial into the slot + ws_peer_reduce_add_f32.
 * Results are bit-identical on all ranks. Every rank must make the same calls. */
int ws_peer_gemm_reduce_add(ws_peer* p, const void* A, const void* W, int32_t M, int32_t N, int32_t K, float* x,
                            void* stream);
/* recv[r * count + i] = rank r's send[i] (the vocab-parallel lm_head shards). */
int ws_peer_allgather_f32(ws_peer* p, const float* send, float* recv, int64_t count, void* stream);
/* A TP communicator with no NCCL behind it: every collective on `peer`
 * (calls above max_count floats fail). */
int ws_comm_create_peer(int32_t rank, int32_t nranks, int32_t device, ws_peer* peer, int64_t max_count,
                        ws_comm** out);
/* Route a TP communicator's allreduces of <= max_count floats through `peer`
 * (NULL restores ncclAllReduce); the lm_head allgather stays on NCCL. */
int ws_comm_set_peer(ws_comm* comm, ws_peer* peer, int64_t max_count);

/* Weight layout of one (TP-partition of a) model inside its slot: byte
 * offsets, every tensor 256-byte aligned. offsets_out receives
 * [embed, final_norm, lm_head, total] then per layer
 * [begin, attn_norm, wqkv, bqkv(-1 if none), wo, ffn_norm, wgu, wdown, end]
 * (4 + 9*layers int64). Layer l occupies [begin, end) contiguously, in
 * order, so layers k..L-1 + final_norm + lm_head form one suffix range. */
int ws_model_layout(const ws_model_config* cfg, int64_t* offsets_out, int64_t n);
/* Tokens per KV block (one pool page) and KV bytes per token (engine.py a19). */
int ws_model_kv_geometry(const ws_model_config* cfg, int64_t page_size, int32_t* tokens_per_block,
                         int64_t* kv_bytes_per_token);

typedef struct ws_model ws_model;
int ws_model_create(const ws_model_config* cfg, int32_t device, ws_model** out);
int ws_model_destroy(ws_model* m);
int ws_model_workspace_bytes(const ws_model* m, int32_t max_tokens, int64_t* bytes_out);
/* Kernel selection bits (A/B tests): 0 = tcgen05 GEMMs + tcgen05 attention (default);
 * bit 0 = legacy mma.sync GEMMs, bit 1 = legacy mma.sync attention (3 = all legacy). */
int ws_model_set_gemm(ws_model* m, int32_t impl);
/* Opt-in (default off): the last decoder layer of a prefill runs attention, O
 * and the FFN for the last row only (every row's QKV + KV append still runs);
 * same first token and KV cache. Every rank of a TP group must agree. */
int ws_model_set_prune_last(ws_model* m, int32_t on);
/* TP row-parallel partials over NCCL: 0 = bf16 on the wire (default; the
 * sum is added to the fp32 residual), 1 = fp32. The peer-memory allreduce
 * always moves fp32. Every rank of a group must agree. */
int ws_model_set_tp_dtype(ws_model* m, int32_t fp32);

/* Prefill `rows` new tokens of sequence `seq` (positions pos0..pos0+rows-1;
 * blocks must be reserved). `weights` is the slot VA. If `streamer` is set,
 * layer l >= first_streamed waits for range (l - first_streamed) and the
 * final norm + lm_head wait for range (layers - first_streamed): the
 * layer-streamed cold start. Writes last-row logits (fp32 [vocab]) and the
 * greedy next token. */
int ws_model_prefill(ws_model* m, ws_pool* pool, const void* weights, int32_t seq,
                     const int32_t* tokens_dev, int32_t rows, int32_t pos0, ws_streamer* streamer,
                     int32_t first_streamed, void* workspace, float* logits_dev,
                     int32_t* next_token_dev, void* stream);

/* One decode step for n sequences: seqs/pos/tokens are device int32[n];
 * max_ctx >= max(pos)+1 bounds the split-K grid. logits fp32 [n, vocab]. */
int ws_model_decode(ws_model* m, ws_pool* pool, const void* weights, const int32_t* seqs_dev,
                    const int32_t* pos_dev, const int32_t* tokens_dev, int32_t n, int32_t max_ctx,
                    void* workspace, float* logits_dev, int32_t* next_tokens_dev, void* stream);

/* Attach a TP communicator (NULL detaches). The model config must be the
 * rank's shard (heads/TP, kv_heads/TP, ffn/TP, lm_head_rows = vocab/TP). */
int ws_model_set_comm(ws_model* m, ws_comm* comm);

/* Standalone GEMM entry for tests/bench: C = A[M,K] * B[N,K]^T, epilogue
 * 0 bf16, 1 bf16+bias, 2 fp32 accumulate, 3 fp32 store, 4 SwiGLU (B = Wgu with
 * 128-row interleaved gate/up blocks, C = bf16 [M, N/2]; tcgen05 paths only).
 * impl: 0 dispatch (skinny tcgen05 for M <= 128, tcgen05 tiles above), 1 legacy
 * mma.sync, 2 legacy GEMV, 3 force the tiled tcgen05 kernel, 4 force the skinny
 * split-K tcgen05 kernel. */
int ws_gemm(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epilogue,
            void* C, const void* bias, int32_t impl, void* stream);

/* Standalone prefill-attention entry for tests/bench: causal GQA attention of
 * `rows` queries (positions pos0..pos0+rows-1) of sequence `seq` over its
 * paged K/V of `layer` in the pool ([0, pos0+rows) must already be appended).
 * qkv: bf16 [rows, (heads + 2 kv_heads) head_dim] (q columns used); out: bf16
 * [rows, heads head_dim]. Geometry from the model's config. impl: 0 the
 * tcgen05 kernels (dispatch as in prefill), 1 the legacy mma.sync kernel. */
int ws_attn_prefill(ws_model* m, ws_pool* pool, int32_t layer, int32_t seq, const void* qkv, int32_t rows,
                    int32_t pos0, void* out, int32_t impl, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* WARMSERVE_H_ */

// Llama-family forward on the paged pool: the compute half of
// activate_instance() and the prefill/decode entry points.
//
// Weights live in the slot VA (contiguous per layer, layout below); KV lives
// in pool pages addressed through the block tables; activations live in a
// caller-provided workspace. The layer loop is host C++ issuing one stream of
// kernels; for a layer-streamed cold start each layer first waits on the copy
// event of its weights (ws_streamer_wait), so compute of resident layers
// overlaps the copy of the rest (cluster.py:145-182).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "kernels/ops.cuh"
#include "tp.h"

namespace ws {
int pool_kv_view(ws_pool* p, char** window, int64_t* page_size, int32_t** block_tables,
                 int32_t* max_blocks, int64_t* n_pages);
}

namespace {

constexpr int64_t kAlign = 256;
int64_t align_up(int64_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  int64_t embed, final_norm, lm_head, total;
  struct L {
    int64_t begin, attn_norm, wqkv, bqkv, wo, ffn_norm, wgu, wdown, end;
  };
  std::vector<L> layers;
};

int qkv_dim(const ws_model_config& c) { return (c.heads + 2 * c.kv_heads) * c.head_dim; }

bool valid_cfg(const ws_model_config& c) {
  return c.layers > 0 && c.hidden > 0 && c.ffn > 0 && c.heads > 0 && c.kv_heads > 0 &&
         c.heads % c.kv_heads == 0 && (c.head_dim == 64 || c.head_dim == 96 || c.head_dim == 128) &&
         c.vocab > 0 && c.hidden % 32 == 0 && c.ffn % 128 == 0 && c.max_positions > 0 &&
         c.heads / c.kv_heads <= 8 && c.hidden <= 8192;  // rmsnorm keeps a row in registers
}

Layout make_layout(const ws_model_config& c) {
  Layout L;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = off;
    off = align_up(off + bytes);
    return at;
  };
  const int64_t d = c.hidden, q = qkv_dim(c), o = (int64_t)c.heads * c.head_dim;
  L.embed = take((int64_t)c.vocab * d * 2);
  for (int l = 0; l < c.layers; ++l) {
    Layout::L x;
    x.begin = off;
    x.attn_norm = take(d * 2);
    x.wqkv = take(q * d * 2);
    x.bqkv = c.qkv_bias ? take(q * 2) : -1;
    x.wo = take(d * o * 2);
    x.ffn_norm = take(d * 2);
    x.wgu = take(2 * (int64_t)c.ffn * d * 2);
    x.wdown = take(d * c.ffn * 2);
    x.end = off;
    L.layers.push_back(x);
  }
  L.final_norm = take(d * 2);
  L.lm_head = take((int64_t)(c.lm_head_rows > 0 ? c.lm_head_rows : c.vocab) * d * 2);
  L.total = off;
  return L;
}

struct Workspace {
  int64_t x, h, qkv, attn, gu, act, hl, seqs, scratch, partial, shard_logits, gathered, norm_ss, norm_scale, total;
};

int head_rows(const ws_model_config& c) { return c.lm_head_rows > 0 ? c.lm_head_rows : c.vocab; }

int decode_cap(int max_tokens) { return max_tokens < 256 ? max_tokens : 256; }

Workspace make_ws(const ws_model_config& c, int T) {
  Workspace w;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = off;
    off = align_up(off + bytes);
    return at;
  };
  const int64_t d = c.hidden;
  w.x = take((int64_t)T * d * 4);
  w.h = take((int64_t)T * d * 2);
  w.qkv = take((int64_t)T * qkv_dim(c) * 2);
  w.attn = take((int64_t)T * c.heads * c.head_dim * 2);
  w.gu = take((int64_t)T * 2 * c.ffn * 2);
  w.act = take((int64_t)T * c.ffn * 2);
  w.hl = take((int64_t)T * d * 2);
  w.seqs = take(4 * 4);
  w.scratch = take((int64_t)ws::decode_scratch_floats(decode_cap(T), c.heads, c.kv_heads,
                                                      c.head_dim) * 4);
  // TP only: fp32 row-parallel partials and the local lm_head shard logits
  const bool tp = head_rows(c) != c.vocab;
  w.partial = take(tp ? (int64_t)T * d * 4 : 0);
  w.shard_logits = take(tp ? (int64_t)decode_cap(T) * head_rows(c) * 4 : 0);
  w.gathered = take(tp ? (int64_t)decode_cap(T) * c.vocab * 4 : 0);
  // decode RMSNorm folded into the skinny GEMMs (<= 128 rows): per-(row,
  // 32-column group) sums of squares and the per-row scales
  const int64_t fold_rows = T < 128 ? T : 128;
  w.norm_ss = take(fold_rows * (d / 32) * 4);
  w.norm_scale = take(fold_rows * 4);
  w.total = off;
  return w;
}

}  // namespace

struct ws_model {
  ws_model_config cfg;
  Layout layout;
  int device = 0;
  float2* rope = nullptr;  // [max_positions, head_dim/2] (cos, sin)
  void* argmax_scratch = nullptr;  // split-row argmax: per-row partial keys + arrival counters (zeroed)
  int gemm_impl = 0;
  bool prune_last = false;  // ws_model_set_prune_last
  bool tp_fp32 = false;     // ws_model_set_tp_dtype: row-parallel partials in fp32 (default bf16)
  ws_comm* comm = nullptr;  // TP group (config 4); null = single GPU
};

namespace {

void gemm(const ws_model* m, const ws::bf16* A, const ws::bf16* B, int M, int N, int K, ws::Epi e,
          void* C, const ws::bf16* bias, cudaStream_t st) {
  if ((m->gemm_impl & 1) && M >= 16)
    ws::launch_gemm_mma(A, B, M, N, K, e, C, bias, st);
  else if (m->gemm_impl & 1)
    ws::launch_gemv(A, B, M, N, K, e, C, bias, st);  // legacy path end to end
  else
    ws::launch_gemm(A, B, M, N, K, e, C, bias, st);
}

// QKV projection + RoPE + paged KV append. One tcgen05 launch with the fused
// epilogue when the shape allows it, else GEMM then the rope_kv kernel.
bool qkv_rope(const ws_model* m, const ws::bf16* h, const ws::bf16* w, const ws::bf16* b, int rows,
              const ws::KvGeom& kv, int layer, int seq0, int pos0, const int32_t* seqs, const int32_t* pos,
              ws::bf16* qkv, cudaStream_t st, const ws::TcEpilogue* norm = nullptr) {
  using namespace ws;
  const ws_model_config& c = m->cfg;
  const int q = (c.heads + 2 * c.kv_heads) * c.head_dim;
  if (!(m->gemm_impl & 1)) {
    TcEpilogue e = norm ? *norm : TcEpilogue{};
    e.mode = Epi::kRopeKV;
    e.C = qkv;
    e.bias = b;
    e.rope = m->rope;
    e.kv = kv;
    e.layer = layer;
    e.heads = c.heads;
    e.seq0 = seq0;
    e.pos0 = pos0;
    e.seq_arr = seqs;
    e.pos_arr = pos;
    // a few decode rows: skinny split-K GEMM with RoPE/KV-append in its fix-up
    // (one launch less; for more rows the plain fix-up + rope kernel is faster)
    static const bool fuse = !(getenv("WS_FUSE_ROPE") && getenv("WS_FUSE_ROPE")[0] == '0');
    // decode (seqs given) up to 32 rows: B = 9..32 -0.5% per step with the
    // cluster reduce doing the RoPE; a prefill of 16 / 32 rows is 0.5% slower so
    static const int fuse_env = getenv("WS_FUSE_ROPE_ROWS") ? atoi(getenv("WS_FUSE_ROPE_ROWS")) : 0;
    const int fuse_rows = fuse_env ? fuse_env : (seqs ? 32 : 8);
    if (fuse && rows <= fuse_rows && launch_gemm_skinny(h, w, rows, q, c.hidden, e, st)) return true;
    if (norm) {  // folded RMSNorm: the skinny GEMM applies the row scales, then RoPE / KV append
      e.mode = b ? Epi::kBiasBf16 : Epi::kStoreBf16;
      e.C = qkv;
      if (!launch_gemm_skinny(h, w, rows, q, c.hidden, e, st)) return false;  // no unscaled fallback
      launch_rope_kv(qkv, m->rope, kv, layer, rows, c.heads, seqs, pos, seq0, pos0, st);
      return true;
    }
    if (rows >= 16 && !(rows <= 128 && gemm_skinny_enabled()) && launch_gemm_tc_epi(h, w, rows, q, c.hidden, e, st))
      return true;
  }
  if (norm) return false;
  gemm(m, h, w, rows, q, c.hidden, b ? Epi::kBiasBf16 : Epi::kStoreBf16, qkv, b, st);
  launch_rope_kv(qkv, m->rope, kv, layer, rows, c.heads, seqs, pos, seq0, pos0, st);
  return true;
}

// gate/up projection + SwiGLU (fused epilogue on the tcgen05 path).
bool gate_up_swiglu(const ws_model* m, const ws::bf16* h, const ws::bf16* w, int rows, ws::bf16* gu,
                    ws::bf16* act, cudaStream_t st, const ws::TcEpilogue* norm = nullptr) {
  using namespace ws;
  const ws_model_config& c = m->cfg;
  if (!(m->gemm_impl & 1)) {
    TcEpilogue e = norm ? *norm : TcEpilogue{};
    e.mode = Epi::kSwiGLU;
    e.C = act;
    if (rows <= 128 && launch_gemm_skinny(h, w, rows, 2 * c.ffn, c.hidden, e, st)) return true;  // decode
    if (norm) return false;  // folded RMSNorm: no unscaled fallback
    if (rows >= 16 && launch_gemm_tc_epi(h, w, rows, 2 * c.ffn, c.hidden, e, st)) return true;
  }
  if (norm) return false;
  gemm(m, h, w, rows, 2 * c.ffn, c.hidden, Epi::kStoreBf16, gu, nullptr, st);
  launch_silu_mul(gu, act, rows, c.ffn, st);
  return true;
}

// Row-parallel projection + residual add: x += A.B^T, summed over the TP group
// (NCCL allreduce of the bf16 partial on the TP boundary; fp32
// partials with ws_model_set_tp_dtype(m, 1) and on the peer-memory kernels).
int row_parallel(const ws_model* m, const ws::bf16* A, const ws::bf16* B, int M, int N, int K, float* x,
                 float* partial, cudaStream_t st) {
  using namespace ws;
  if (!m->comm) {
    gemm(m, A, B, M, N, K, Epi::kAddF32, x, nullptr, st);
    return WS_OK;
  }
  if (ws_peer* peer = comm_peer(m->comm, (int64_t)M * N)) {
    // peer memory: the GEMM writes its partial straight into this rank's
    // exported slot; prefill shapes reduce it block by block beside the GEMM
    // (ws_peer_gemm_reduce_add), decode shapes with one reduce-add kernel
    if (!(m->gemm_impl & 1)) return ws_peer_gemm_reduce_add(peer, A, B, M, N, K, x, st);
    float* slot = nullptr;
    if (int e = ws_peer_next_slot(peer, &slot)) return e;
    gemm(m, A, B, M, N, K, Epi::kStoreF32, slot, nullptr, st);
    return ws_peer_reduce_add_f32(peer, x, (int64_t)M * N, st);
  }
  if (!m->tp_fp32 && comm_has_nccl(m->comm)) {
    // bf16 partials on the wire ([S, d] bf16 per allreduce), summed
    // into the fp32 residual after the collective
    bf16* pb = reinterpret_cast<bf16*>(partial);
    gemm(m, A, B, M, N, K, Epi::kStoreBf16, pb, nullptr, st);
    if (int e = comm_allreduce_bf16(m->comm, pb, (int64_t)M * N, st)) return e;
    launch_add_bf16_f32(x, pb, (int64_t)M * N, st);
    return WS_OK;
  }
  gemm(m, A, B, M, N, K, Epi::kStoreF32, partial, nullptr, st);
  if (int e = comm_allreduce_f32(m->comm, partial, (int64_t)M * N, st)) return e;
  launch_add_f32(x, partial, (int64_t)M * N, st);
  return WS_OK;
}

// Row-parallel projection + residual add, then RMSNorm of the updated rows into `out`.
int row_parallel_norm(const ws_model* m, const ws::bf16* A, const ws::bf16* B, int M, int N, int K, float* x,
                      float* partial, const ws::bf16* norm_w, ws::bf16* out, cudaStream_t st) {
  if (int e = row_parallel(m, A, B, M, N, K, x, partial, st)) return e;
  ws::launch_rmsnorm(x, norm_w, out, M, N, m->cfg.rms_eps, st);
  return WS_OK;
}

// lm_head for `rows` normalized rows -> fp32 logits [rows, vocab] + argmax.
// TP: each rank holds vocab/TP rows; shards are all-gathered and reordered.
int lm_head(const ws_model* m, const ws::bf16* hl, const ws::bf16* W, int rows, float* logits,
            float* shard, float* gathered, int32_t* next, cudaStream_t st) {
  using namespace ws;
  const ws_model_config& c = m->cfg;
  const int Vs = head_rows(c);
  if (!m->comm) {
    gemm(m, hl, W, rows, c.vocab, c.hidden, Epi::kStoreF32, logits, nullptr, st);
  } else {
    gemm(m, hl, W, rows, Vs, c.hidden, Epi::kStoreF32, shard, nullptr, st);
    if (int e = comm_allgather_f32(m->comm, shard, gathered, (int64_t)rows * Vs, st)) return e;
    launch_gather_vocab(gathered, logits, comm_size(m->comm), rows, Vs, st);
  }
  launch_argmax(logits, rows, c.vocab, next, m->argmax_scratch, st);
  return WS_OK;
}

int kv_geom(ws_model* m, ws_pool* pool, ws::KvGeom* g) {
  int32_t* bt;
  if (int e = ws::pool_kv_view(pool, &g->window, &g->page_size, &bt, &g->max_blocks, &g->n_pages)) return e;
  g->block_tables = bt;
  int64_t kvb = 0;
  if (int e = ws_model_kv_geometry(&m->cfg, g->page_size, &g->tpb, &kvb)) return e;
  g->layers = m->cfg.layers;
  g->kv_heads = m->cfg.kv_heads;
  g->head_dim = m->cfg.head_dim;
  return WS_OK;
}

template <typename T>
const T* W(const void* base, int64_t off) {
  return reinterpret_cast<const T*>(static_cast<const char*>(base) + off);
}

}  // namespace

extern "C" {

int ws_model_layout(const ws_model_config* cfg, int64_t* out, int64_t n) {
  if (!cfg || !valid_cfg(*cfg)) WS_FAIL(WS_ERR_INVALID, "invalid model config");
  if (n < 4 + 9 * (int64_t)cfg->layers) WS_FAIL(WS_ERR_INVALID, "layout buffer too small");
  Layout L = make_layout(*cfg);
  out[0] = L.embed;
  out[1] = L.final_norm;
  out[2] = L.lm_head;
  out[3] = L.total;
  for (int l = 0; l < cfg->layers; ++l) {
    const auto& x = L.layers[l];
    int64_t* o = out + 4 + 9 * l;
    o[0] = x.begin; o[1] = x.attn_norm; o[2] = x.wqkv; o[3] = x.bqkv; o[4] = x.wo;
    o[5] = x.ffn_norm; o[6] = x.wgu; o[7] = x.wdown; o[8] = x.end;
  }
  return WS_OK;
}

int ws_model_kv_geometry(const ws_model_config* cfg, int64_t page_size, int32_t* tpb,
                         int64_t* kv_bytes_per_token) {
  if (!cfg || !valid_cfg(*cfg)) WS_FAIL(WS_ERR_INVALID, "invalid model config");
  const int64_t per_tok = (int64_t)cfg->layers * 2 * cfg->kv_heads * cfg->head_dim * 2;
  if (kv_bytes_per_token) *kv_bytes_per_token = per_tok;
  if (tpb) {
    if (page_size < per_tok) WS_FAIL(WS_ERR_INVALID, "a page cannot hold one token of KV");
    *tpb = (int32_t)(page_size / per_tok);
  }
  return WS_OK;
}

int ws_model_create(const ws_model_config* cfg, int32_t device, ws_model** out) {
  if (!cfg || !valid_cfg(*cfg)) WS_FAIL(WS_ERR_INVALID, "invalid model config");
  ws_model* m = new ws_model();
  m->cfg = *cfg;
  m->layout = make_layout(*cfg);
  m->device = device;
  const int half = cfg->head_dim / 2;
  std::vector<float2> tab((size_t)cfg->max_positions * half);
  for (int i = 0; i < half; ++i) {
    const double inv = std::pow((double)cfg->rope_theta, -2.0 * i / (double)cfg->head_dim);
    for (int p = 0; p < cfg->max_positions; ++p) {
      const double a = (double)p * inv;
      tab[(size_t)p * half + i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  }
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaMalloc(&m->rope, tab.size() * sizeof(float2)) != cudaSuccess ||
      cudaMemcpy(m->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cudaMalloc(&m->argmax_scratch, ws::argmax_scratch_bytes()) != cudaSuccess ||
      cudaMemset(m->argmax_scratch, 0, ws::argmax_scratch_bytes()) != cudaSuccess) {
    if (m->rope) cudaFree(m->rope);
    delete m;
    WS_FAIL(WS_ERR_CUDA, "RoPE table upload failed");
  }
  *out = m;
  return WS_OK;
}

int ws_model_destroy(ws_model* m) {
  if (!m) return WS_OK;
  if (m->rope) cudaFree(m->rope);
  if (m->argmax_scratch) cudaFree(m->argmax_scratch);
  delete m;
  return WS_OK;
}

int ws_model_workspace_bytes(const ws_model* m, int32_t max_tokens, int64_t* bytes) {
  if (!m || max_tokens < 1) WS_FAIL(WS_ERR_INVALID, "bad workspace request");
  *bytes = make_ws(m->cfg, max_tokens).total;
  return WS_OK;
}

int ws_model_set_comm(ws_model* m, ws_comm* comm) {
  if (!m) WS_FAIL(WS_ERR_INVALID, "null model");
  if (comm && head_rows(m->cfg) * ws::comm_size(comm) != m->cfg.vocab)
    WS_FAIL(WS_ERR_INVALID, "lm_head_rows x TP size must equal vocab");
  m->comm = comm;
  return WS_OK;
}

int ws_model_set_gemm(ws_model* m, int32_t impl) {
  if (!m || impl < 0 || impl > 3) WS_FAIL(WS_ERR_INVALID, "impl must be in 0..3");
  m->gemm_impl = impl;
  return WS_OK;
}

int ws_model_set_tp_dtype(ws_model* m, int32_t fp32) {
  if (!m) WS_FAIL(WS_ERR_INVALID, "null model");
  m->tp_fp32 = fp32 != 0;
  return WS_OK;
}

int ws_model_set_prune_last(ws_model* m, int32_t on) {
  if (!m) WS_FAIL(WS_ERR_INVALID, "null model");
  m->prune_last = on != 0;
  return WS_OK;
}

int ws_model_prefill(ws_model* m, ws_pool* pool, const void* wts, int32_t seq,
                     const int32_t* tokens, int32_t rows, int32_t pos0, ws_streamer* streamer,
                     int32_t first_streamed, void* workspace, float* logits, int32_t* next_token,
                     void* stream) {
  using namespace ws;
  if (!m || !wts || !workspace || rows < 1) WS_FAIL(WS_ERR_INVALID, "bad prefill arguments");
  const ws_model_config& c = m->cfg;
  if (pos0 + rows > c.max_positions) WS_FAIL(WS_ERR_INVALID, "positions exceed the RoPE table");
  KvGeom kv;
  if (int e = kv_geom(m, pool, &kv)) return e;
  if ((pos0 + rows + kv.tpb - 1) / kv.tpb > kv.max_blocks) WS_FAIL(WS_ERR_INVALID, "sequence too long");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Workspace w = make_ws(c, rows);
  char* wsb = static_cast<char*>(workspace);
  float* x = reinterpret_cast<float*>(wsb + w.x);
  bf16* h = reinterpret_cast<bf16*>(wsb + w.h);
  bf16* qkv = reinterpret_cast<bf16*>(wsb + w.qkv);
  bf16* attn = reinterpret_cast<bf16*>(wsb + w.attn);
  bf16* gu = reinterpret_cast<bf16*>(wsb + w.gu);
  bf16* act = reinterpret_cast<bf16*>(wsb + w.act);
  bf16* hl = reinterpret_cast<bf16*>(wsb + w.hl);
  float* partial = reinterpret_cast<float*>(wsb + w.partial);
  float* shard = reinterpret_cast<float*>(wsb + w.shard_logits);
  float* gathered = reinterpret_cast<float*>(wsb + w.gathered);
  const int d = c.hidden, q = qkv_dim(c), o = c.heads * c.head_dim;
  const float scale = 1.0f / std::sqrt((float)c.head_dim);
  const Layout& L = m->layout;

  launch_embed(tokens, W<bf16>(wts, L.embed), x, rows, d, st);
  for (int l = 0; l < c.layers; ++l) {
    if (streamer && l >= first_streamed)
      if (int e = ws_streamer_wait(streamer, l - first_streamed, stream)) return e;
    const auto& Ly = L.layers[l];
    launch_rmsnorm(x, W<bf16>(wts, Ly.attn_norm), h, rows, d, c.rms_eps, st);
    qkv_rope(m, h, W<bf16>(wts, Ly.wqkv), c.qkv_bias ? W<bf16>(wts, Ly.bqkv) : nullptr, rows, kv, l, seq,
             pos0, nullptr, nullptr, qkv, st);
    // Per-model opt-in (ws_model_set_prune_last): in the last layer every
    // row's K/V is in the cache after qkv_rope and only the last row feeds the
    // final norm + lm_head, so attention, O and the FFN may run for that row
    // alone. Off by default: the measured prefill then does every row's full
    // work, like the reference's per-token cost model and the CPU oracle. A TP
    // group sets it on every rank (the row-parallel collectives change size).
    const int r0 = m->prune_last && l + 1 == c.layers ? rows - 1 : 0, n = rows - r0;
    const bf16* q_rows = qkv + (int64_t)r0 * q;
    float* x_rows = x + (int64_t)r0 * d;
    if ((m->gemm_impl & 2) || attn_prefill_prefers_mma(kv, n, c.heads)) {
      launch_attn_prefill(q_rows, attn, kv, l, seq, n, pos0 + r0, c.heads, scale, st);
    } else if (!launch_attn_prefill_tc(q_rows, attn, kv, l, seq, n, pos0 + r0, c.heads, scale, st)) {
      count_fallback(kFallbackAttnMma, "prefill attention shape outside attn_tc (head_dim / GQA) runs mma.sync");
      launch_attn_prefill(q_rows, attn, kv, l, seq, n, pos0 + r0, c.heads, scale, st);
    }
    if (int e = row_parallel(m, attn, W<bf16>(wts, Ly.wo), n, d, o, x_rows, partial, st)) return e;
    launch_rmsnorm(x_rows, W<bf16>(wts, Ly.ffn_norm), h, n, d, c.rms_eps, st);
    gate_up_swiglu(m, h, W<bf16>(wts, Ly.wgu), n, gu, act, st);
    if (int e = row_parallel(m, act, W<bf16>(wts, Ly.wdown), n, d, c.ffn, x_rows, partial, st)) return e;
  }
  if (streamer && c.layers >= first_streamed)
    if (int e = ws_streamer_wait(streamer, c.layers - first_streamed, stream)) return e;
  launch_rmsnorm(x + (int64_t)(rows - 1) * d, W<bf16>(wts, L.final_norm), hl, 1, d, c.rms_eps, st);
  if (int e = lm_head(m, hl, W<bf16>(wts, L.lm_head), 1, logits, shard, gathered, next_token, st)) return e;
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

int ws_model_decode(ws_model* m, ws_pool* pool, const void* wts, const int32_t* seqs,
                    const int32_t* pos, const int32_t* tokens, int32_t n, int32_t max_ctx,
                    void* workspace, float* logits, int32_t* next_tokens, void* stream) {
  using namespace ws;
  if (!m || !wts || !workspace || n < 1) WS_FAIL(WS_ERR_INVALID, "bad decode arguments");
  const ws_model_config& c = m->cfg;
  if (n > 256) WS_FAIL(WS_ERR_INVALID, "decode batch above 256");
  if (max_ctx > c.max_positions) WS_FAIL(WS_ERR_INVALID, "context exceeds the RoPE table");
  KvGeom kv;
  if (int e = kv_geom(m, pool, &kv)) return e;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Workspace w = make_ws(c, n);
  char* wsb = static_cast<char*>(workspace);
  float* x = reinterpret_cast<float*>(wsb + w.x);
  bf16* h = reinterpret_cast<bf16*>(wsb + w.h);
  bf16* qkv = reinterpret_cast<bf16*>(wsb + w.qkv);
  bf16* attn = reinterpret_cast<bf16*>(wsb + w.attn);
  bf16* gu = reinterpret_cast<bf16*>(wsb + w.gu);
  bf16* act = reinterpret_cast<bf16*>(wsb + w.act);
  bf16* hl = reinterpret_cast<bf16*>(wsb + w.hl);
  float* scratch = reinterpret_cast<float*>(wsb + w.scratch);
  float* partial = reinterpret_cast<float*>(wsb + w.partial);
  float* shard = reinterpret_cast<float*>(wsb + w.shard_logits);
  float* gathered = reinterpret_cast<float*>(wsb + w.gathered);
  const int d = c.hidden, q = qkv_dim(c), o = c.heads * c.head_dim;
  const float scale = 1.0f / std::sqrt((float)c.head_dim);
  const Layout& L = m->layout;

  // Fold the per-layer RMSNorms into the skinny GEMMs: each residual GEMM
  // (O, down) also writes bf16(x * g) and row sums of squares, the next
  // projection (gate/up, next layer's QKV) scales its rows by rsqrt(mean +
  // eps) — two launches fewer per layer. Graph-replayed 8B steps, ctx 1024:
  // B = 1 / 4 / 16 3.96 / 4.12 / 4.31 -> 3.79 / 4.05 / 4.23 ms; no gain at
  // B = 32 and 0.6% slower at B = 64 (the load-add-store residual and the
  // wider fix-up epilogues cost what the launches saved), so up to 16 rows at first. Off for TP (the
  // residual is summed across ranks first), the legacy GEMMs, shapes outside
  // the skinny kernel, and WS_FOLD_NORM=0 (A/B).
  static const bool fold_env = !(getenv("WS_FOLD_NORM") && getenv("WS_FOLD_NORM")[0] == '0');
  // since the cluster reduce serves 17-32 rows too, up to 32 (B = 17 / 32
  // 4.08 / 4.38 -> 4.03 / 4.31 ms; B = 48 / 64 still 1.2% / 0.2% slower)
  static const int fold_rows = getenv("WS_FOLD_ROWS") ? atoi(getenv("WS_FOLD_ROWS")) : 32;
  const bool fold = fold_env && n <= fold_rows && !m->comm && !(m->gemm_impl & 1) &&
                    gemm_skinny_supported(n, d, o, Epi::kAddF32) &&
                    gemm_skinny_supported(n, d, c.ffn, Epi::kAddF32) &&
                    gemm_skinny_supported(n, q, d, Epi::kStoreBf16) &&
                    gemm_skinny_supported(n, 2 * c.ffn, d, Epi::kSwiGLU);
  TcEpilogue np, nc;  // producer / consumer halves of a folded norm
  if (fold) {
    np.mode = Epi::kAddF32;
    np.C = x;
    np.norm_role = 1;
    np.norm_out = h;
    np.row_ss = reinterpret_cast<float*>(wsb + w.norm_ss);
    nc.norm_role = 2;
    nc.norm_d = d;
    nc.norm_eps = c.rms_eps;
    nc.row_ss = np.row_ss;
    nc.row_scale = reinterpret_cast<float*>(wsb + w.norm_scale);
  }
  // L2 prefetch hints (WS_L2PF bit mask, A/B): a latency-bound kernel pulls a
  // later kernel's weights into L2 — 1: attention -> the O weights, 2: QKV ->
  // the O weights, 4: O -> a prefix of every gate/up row, 8: gate/up -> a
  // prefix of every quarter-row of down, 16: down -> the next QKV's half-rows.
  static const int pf_mask = getenv("WS_L2PF") ? atoi(getenv("WS_L2PF")) : 0;
  static const int pf_frac = getenv("WS_L2PF_FRAC") ? atoi(getenv("WS_L2PF_FRAC")) : 50;
  static const int pf_at = getenv("WS_L2PF_AT") ? atoi(getenv("WS_L2PF_AT")) : 0;
  static const int pf_rows = getenv("WS_L2PF_ROWS") ? atoi(getenv("WS_L2PF_ROWS")) : 16;
  const int pfm = fold && n <= pf_rows ? pf_mask : 0;
  auto pf_whole = [](const void* p, int64_t bytes) {
    L2Pf f;
    f.p = static_cast<const char*>(p);
    f.pitch = 1 << 16;
    f.seg_bytes = 1 << 16;
    f.rows = (int)((bytes + f.pitch - 1) / f.pitch);
    f.limit = bytes;
    return f;
  };
  auto pf_prefix = [&](const void* p, int rows, int K, int nseg) {  // prefix of each of nseg slices of every row
    L2Pf f;
    f.p = static_cast<const char*>(p);
    f.pitch = (int64_t)K * 2;
    f.rows = rows;
    f.nseg = nseg;
    f.seg_stride = f.pitch / nseg;
    f.seg_bytes = (int)(f.seg_stride * pf_frac / 100) & ~15;
    f.limit = f.pitch * rows;
    return f;
  };
  launch_embed(tokens, W<bf16>(wts, L.embed), x, n, d, st);
  launch_rmsnorm(x, W<bf16>(wts, L.layers[0].attn_norm), h, n, d, c.rms_eps, st);
  nc.l2pf_at = np.l2pf_at = pf_at;
  for (int l = 0; l < c.layers; ++l) {
    const auto& Ly = L.layers[l];
    const bool last = l + 1 == c.layers;
    nc.l2pf = (pfm & 2) ? pf_whole(W<bf16>(wts, Ly.wo), (int64_t)d * o * 2) : L2Pf{};
    if (!qkv_rope(m, h, W<bf16>(wts, Ly.wqkv), c.qkv_bias ? W<bf16>(wts, Ly.bqkv) : nullptr, n, kv, l, 0, 0, seqs,
                  pos, qkv, st, fold && l > 0 ? &nc : nullptr))
      WS_FAIL(WS_ERR_CUDA, "folded-norm QKV GEMM declined");
    launch_attn_decode(qkv, attn, kv, l, seqs, pos, n, c.heads, max_ctx, scale, scratch, st,
                       (pfm & 1) ? pf_whole(W<bf16>(wts, Ly.wo), (int64_t)d * o * 2) : L2Pf{});
    if (fold) {
      np.norm_g = W<bf16>(wts, Ly.ffn_norm);
      np.l2pf = (pfm & 4) ? pf_prefix(W<bf16>(wts, Ly.wgu), 2 * c.ffn, d, 1) : L2Pf{};
      if (!launch_gemm_skinny(attn, W<bf16>(wts, Ly.wo), n, d, o, np, st)) WS_FAIL(WS_ERR_CUDA, "folded O GEMM");
      nc.l2pf = (pfm & 8) ? pf_prefix(W<bf16>(wts, Ly.wdown), d, c.ffn, 4) : L2Pf{};
      if (!gate_up_swiglu(m, h, W<bf16>(wts, Ly.wgu), n, gu, act, st, &nc))
        WS_FAIL(WS_ERR_CUDA, "folded-norm gate/up GEMM declined");
      if (!last) {
        np.norm_g = W<bf16>(wts, L.layers[l + 1].attn_norm);
        np.l2pf = (pfm & 16) ? pf_prefix(W<bf16>(wts, L.layers[l + 1].wqkv), q, d, 2) : L2Pf{};
        if (!launch_gemm_skinny(act, W<bf16>(wts, Ly.wdown), n, d, c.ffn, np, st))
          WS_FAIL(WS_ERR_CUDA, "folded down GEMM");
        continue;
      }
      np.l2pf = L2Pf{};
      nc.l2pf = L2Pf{};
      // last layer: plain residual + the final norm kernel for the lm_head rows
      if (int e = row_parallel_norm(m, act, W<bf16>(wts, Ly.wdown), n, d, c.ffn, x, partial,
                                    W<bf16>(wts, L.final_norm), hl, st))
        return e;
      continue;
    }
    if (int e = row_parallel_norm(m, attn, W<bf16>(wts, Ly.wo), n, d, o, x, partial, W<bf16>(wts, Ly.ffn_norm), h,
                                  st))
      return e;
    gate_up_swiglu(m, h, W<bf16>(wts, Ly.wgu), n, gu, act, st);
    // the residual after the FFN feeds the next layer's attn_norm (or the final norm)
    if (int e = row_parallel_norm(m, act, W<bf16>(wts, Ly.wdown), n, d, c.ffn, x, partial,
                                  W<bf16>(wts, last ? L.final_norm : L.layers[l + 1].attn_norm), last ? hl : h, st))
      return e;
  }
  if (int e = lm_head(m, hl, W<bf16>(wts, L.lm_head), n, logits, shard, gathered, next_tokens, st)) return e;
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

int ws_attn_prefill(ws_model* m, ws_pool* pool, int32_t layer, int32_t seq, const void* qkv, int32_t rows,
                    int32_t pos0, void* out, int32_t impl, void* stream) {
  using namespace ws;
  if (!m || !pool || !qkv || !out || rows < 1 || pos0 < 0 || layer < 0 || layer >= m->cfg.layers)
    WS_FAIL(WS_ERR_INVALID, "bad attention arguments");
  KvGeom kv;
  if (int e = kv_geom(m, pool, &kv)) return e;
  if ((pos0 + rows + kv.tpb - 1) / kv.tpb > kv.max_blocks) WS_FAIL(WS_ERR_INVALID, "sequence too long");
  const ws_model_config& c = m->cfg;
  const float scale = 1.0f / std::sqrt((float)c.head_dim);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bf16* q = static_cast<const bf16*>(qkv);
  bf16* o = static_cast<bf16*>(out);
  if (impl == 1 || !launch_attn_prefill_tc(q, o, kv, layer, seq, rows, pos0, c.heads, scale, st))
    launch_attn_prefill(q, o, kv, layer, seq, rows, pos0, c.heads, scale, st);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

int ws_gemm(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epi, void* C,
            const void* bias, int32_t impl, void* stream) {
  using namespace ws;
  if (M < 1 || N < 1 || K < 32 || K % 32 || epi < 0 || epi > 4) WS_FAIL(WS_ERR_INVALID, "bad GEMM shape");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bf16* a = static_cast<const bf16*>(A);
  const bf16* b = static_cast<const bf16*>(B);
  const bf16* bi = static_cast<const bf16*>(bias);
  if (epi == (int)Epi::kSwiGLU) {
    TcEpilogue e;
    e.mode = Epi::kSwiGLU;
    e.C = C;
    const bool ok = impl == 4   ? launch_gemm_skinny(a, b, M, N, K, e, st)
                    : impl == 3 ? launch_gemm_tc_epi(a, b, M, N, K, e, st)
                                : (M <= 128 && launch_gemm_skinny(a, b, M, N, K, e, st)) ||
                                      launch_gemm_tc_epi(a, b, M, N, K, e, st);
    if (!ok) WS_FAIL(WS_ERR_INVALID, "SwiGLU GEMM %dx%dx%d unsupported", M, N, K);
  } else if (impl == 1 && M >= 16) {
    launch_gemm_mma(a, b, M, N, K, (Epi)epi, C, bi, st);
  } else if (impl == 2) {
    launch_gemv(a, b, M, N, K, (Epi)epi, C, bi, st);
  } else if (impl == 3) {
    if (!launch_gemm_tc(a, b, M, N, K, (Epi)epi, C, bi, st))
      WS_FAIL(WS_ERR_INVALID, "shape %dx%dx%d outside the tcgen05 tiling", M, N, K);
  } else if (impl == 4) {
    TcEpilogue e;
    e.mode = (Epi)epi;
    e.C = C;
    e.bias = bi;
    if (!launch_gemm_skinny(a, b, M, N, K, e, st))
      WS_FAIL(WS_ERR_INVALID, "shape %dx%dx%d outside the skinny tcgen05 envelope", M, N, K);
  } else {
    launch_gemm(a, b, M, N, K, (Epi)epi, C, bi, st);
  }
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

}  // extern "C"

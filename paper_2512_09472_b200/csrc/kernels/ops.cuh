// Launchers of the model kernels. All activations are row-major with the
// feature dimension contiguous; weights are [out, in] row-major (K-major for
// both GEMM operands). The residual stream is fp32; everything a GEMM reads is
// bf16.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace ws {

using bf16 = __nv_bfloat16;

// L2 prefetch hint for a decode kernel: the weights of a LATER kernel of the
// step, pulled into L2 while this one is latency-bound and leaves HBM
// bandwidth idle (weights are immutable, so the prefetch may run before the
// PDL wait). Items = rows x nseg byte ranges [p + r*pitch + s*seg_stride,
// + seg_bytes) clipped at `limit` bytes from p, spread round-robin over the
// launch's CTAs (cp.async.bulk.prefetch.L2, one issuing thread per CTA).
struct L2Pf {
  const char* p = nullptr;
  int64_t pitch = 0, seg_stride = 0, limit = 0;
  int rows = 0, nseg = 1, seg_bytes = 0;
};

// Paged KV cache geometry: block = one pool page holding `tpb` tokens of every
// layer; inside a page: [layer][k|v][kv_head][tpb][head_dim] bf16.
struct KvGeom {
  char* window;          // page window base (page p at window + p*page_size)
  int64_t page_size;
  const int32_t* block_tables;  // [max_seqs, max_blocks]
  int32_t max_blocks;
  int32_t tpb;           // tokens per block
  int32_t layers, kv_heads, head_dim;
  int64_t n_pages;       // pages in the window (TMA descriptor extent)

  __host__ __device__ int64_t head_stride() const { return (int64_t)tpb * head_dim; }
  // element offset of (layer, kind, head, slot 0) inside a page
  __host__ __device__ int64_t plane(int layer, int kind, int head) const {
    return (((int64_t)layer * 2 + kind) * kv_heads + head) * head_stride();
  }
};

void launch_embed(const int32_t* tokens, const bf16* table, float* x, int n_tokens, int d,
                  cudaStream_t st);
void launch_rmsnorm(const float* x, const bf16* w, bf16* out, int rows, int d, float eps,
                    cudaStream_t st);
void launch_silu_mul(const bf16* gu, bf16* act, int rows, int ffn, cudaStream_t st);

// q,k rotated in place inside qkv ([rows, (H+2KV)*hd]); k,v appended to the
// paged cache at positions pos[r] of sequence seq[r] (both device arrays), or
// pos0 + r / seq0 when the arrays are null (single-sequence prefill).
void launch_rope_kv(bf16* qkv, const float2* rope_table, const KvGeom& kv, int layer, int rows,
                    int heads, const int32_t* seq, const int32_t* pos, int seq0, int pos0,
                    cudaStream_t st);

// Causal GQA attention of one sequence's `rows` new queries (positions
// pos0..pos0+rows-1) over its paged KV [0, pos0+rows). out: [rows, H*hd].
void launch_attn_prefill(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq,
                         int rows, int pos0, int heads, float scale, cudaStream_t st);

// tcgen05/TMEM flash-attention version (attn_tc.cu), head_dim 64 or 128;
// returns false (nothing launched) for other head dims.
bool launch_attn_prefill_tc(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                            int pos0, int heads, float scale, cudaStream_t st);
// Whether launch_attn_prefill_tc runs the paired-head kernel for this shape
// (even GQA group, TMA-addressable blocks), and whether a prompt of `rows`
// queries is better served by launch_attn_prefill: a short prompt gives the
// tcgen05 kernels a few long serial tile chains on a few dozen SMs.
bool attn_prefill_tc_paired(const KvGeom& kv, int heads);
bool attn_prefill_prefers_mma(const KvGeom& kv, int rows, int heads);

// One query token per sequence: seqs[i] at position pos[i] (context pos+1,
// its own K/V already appended). scratch: decode_scratch_floats() floats.
void launch_attn_decode(const bf16* qkv, bf16* out, const KvGeom& kv, int layer,
                        const int32_t* seqs, const int32_t* pos, int n_seqs, int heads,
                        int max_ctx, float scale, float* scratch, cudaStream_t st,
                        const L2Pf& pf = L2Pf{});
int decode_scratch_floats(int n_seqs, int heads, int kv_heads, int head_dim);

// C[M,N] = A[M,K] * B[N,K]^T with epilogue:
//   kSwiGLU  (tcgen05 only): B = interleaved gate/up rows (128-row blocks);
//            C = bf16 [M, N/2] = silu(gate) * up
//   kRopeKV  (tcgen05 only): B = Wqkv; optional bias; q/k heads rotated (RoPE),
//            q written to C ([M, N] bf16), k/v appended to the paged cache
enum class Epi { kStoreBf16 = 0, kBiasBf16 = 1, kAddF32 = 2, kStoreF32 = 3, kSwiGLU = 4, kRopeKV = 5 };

struct TcEpilogue {
  Epi mode = Epi::kStoreBf16;
  void* C = nullptr;
  const bf16* bias = nullptr;
  // kRopeKV
  const float2* rope = nullptr;
  KvGeom kv{};
  int layer = 0, heads = 0, seq0 = 0, pos0 = 0;
  const int32_t* seq_arr = nullptr;
  const int32_t* pos_arr = nullptr;
  // Decode RMSNorm folded across a residual GEMM and the next projection
  // (skinny path only). norm_role 1 (kAddF32 producer): besides x += A.W^T,
  // write norm_out = bf16(x_new * norm_g) and per-(row, 32-column group)
  // sums of squares row_ss[M][norm_d / 32]. norm_role 2 (consumer): A is
  // norm_out, and every output row is scaled by rsqrt(sum(row_ss) / norm_d +
  // norm_eps) before bias / RoPE / SwiGLU — exact by linearity; row_scale[M]
  // carries the scales from the GEMM to its fix-up kernels.
  int norm_role = 0, norm_d = 0;
  float norm_eps = 0.f;
  const bf16* norm_g = nullptr;
  bf16* norm_out = nullptr;
  float* row_ss = nullptr;
  float* row_scale = nullptr;
  // Tile publication (CTA-pair tcgen05 kernel, kStoreBf16 / kStoreF32 only):
  // once the TMA stores of a CTA's 128 rows x 256 columns of tile t have
  // landed, tile_flags[2 t + rank in pair] = tile_epoch with a system-scope
  // release, so a consumer on this or a peer GPU can take the block while the
  // GEMM still runs (peer.cu's fused row-parallel allreduce).
  uint32_t* tile_flags = nullptr;
  uint32_t tile_epoch = 0;
  // kRopeKV on the CTA-pair kernel: set by the launcher when the rotated K/V
  // rows can leave as TMA boxes of 16 tokens into the page window (prefill of
  // one sequence, block-aligned pos0, 16-token runs per block)
  int kv_tma = 0;
  // skinny decode GEMMs: L2 prefetch of a later kernel's weights (see L2Pf),
  // issued at the start (l2pf_at 0) or after the producer's last load (1)
  L2Pf l2pf{};
  int l2pf_at = 0;
};
bool gemm_tc_epilogue_supported(const TcEpilogue& e, int N, int head_dim);
bool launch_gemm_tc_epi(const bf16* A, const bf16* B, int M, int N, int K, const TcEpilogue& e,
                        cudaStream_t st);
// Dispatch: M >= 16 -> tensor-core GEMM, else the skinny GEMV.
void launch_gemm(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                 const bf16* bias, cudaStream_t st);
// Legacy mma.sync GEMM (baseline + parity reference for the tcgen05 kernel).
void launch_gemm_mma(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                     const bf16* bias, cudaStream_t st);
// tcgen05/TMEM/TMA GEMM (gemm_tc.cu): needs M >= 16, N % 256 == 0, K % 64 == 0;
// returns false (nothing launched) otherwise.
bool gemm_tc_supported(int M, int N, int K);
// The CTA-pair kernel serves this M (M >= 256 unless WS_GEMM_PAIR=0); only it
// honours TcEpilogue::tile_flags.
bool gemm_tc_pair_enabled(int M);
bool launch_gemm_tc(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                    const bf16* bias, cudaStream_t st);
// Decode-shaped tcgen05 GEMM (gemm_skinny.cu): M <= 128, N % 128 == 0
// (% 256 for kSwiGLU), K % 64 == 0, any epilogue but kRopeKV; swap-AB split-K,
// HBM bound. Returns false (nothing launched) outside that envelope or when
// disabled with WS_SKINNY=0.
bool gemm_skinny_enabled();
// launch_gemm_skinny's shape envelope (kRopeKV aside, which may also decline
// when the weight has more units than the grid has CTAs)
bool gemm_skinny_supported(int M, int N, int K, Epi mode);
bool launch_gemm_skinny(const bf16* A, const bf16* W, int M, int N, int K, const TcEpilogue& e, cudaStream_t st);
// Legacy CUDA-core GEMV for M <= 16 (fallback when the skinny kernel does not apply).
void launch_gemv(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                 const bf16* bias, cudaStream_t st);
// TP boundary helpers: x += p (fp32, count elements); reorder all-gathered
// vocab shards [tp][rows][vs] into logits [rows][tp*vs].
void launch_add_f32(float* x, const float* p, int64_t count, cudaStream_t st);
void launch_add_bf16_f32(float* x, const bf16* p, int64_t count, cudaStream_t st);
void launch_gather_vocab(const float* gathered, float* logits, int tp, int rows, int vs, cudaStream_t st);
// Packed bf16 weight ranges (unpack.cu): section offsets of a packed range
// of n values with n_esc escapes, and the two-pass rebuild into dst.
void packed_sections(int64_t n, int64_t n_esc, int64_t* codes_off, int64_t* idx_off, int64_t* exp_off,
                     int64_t* total);
void launch_unpack_bf16(void* dst, const void* packed, int64_t n, int e_base, int64_t n_esc, cudaStream_t st);
void huff_sections(int64_t n, int64_t* lut_off, int64_t* offs_off, int64_t* words_off);
void launch_unpack_huff(void* dst, const void* packed, int64_t n, cudaStream_t st);
// Argmax of M rows of fp32 logits. scratch: argmax_scratch_bytes() of
// device memory, ZEROED once at allocation (per-row arrival counters that the
// kernel resets itself); null runs one CTA per row. M <= kArgmaxMaxRows.
constexpr int kArgmaxMaxRows = 256, kArgmaxMaxSplit = 32;
constexpr int64_t argmax_scratch_bytes() { return (int64_t)kArgmaxMaxRows * kArgmaxMaxSplit * 8 + kArgmaxMaxRows * 4; }
void launch_argmax(const float* logits, int M, int V, int32_t* out, void* scratch, cudaStream_t st);

}  // namespace ws

// Paged attention over the pool's page window (block = one 2 MiB page).
//
// Prefill: FlashAttention-2 style causal GQA — one CTA per (64-query tile,
// q head), 4 warps x 16 query rows, K/V tiles of 64 keys gathered page by page
// with cp.async (double-buffered), S = QK^T and O += PV on mma.sync, online
// softmax in fp32 registers (exp2 with the log2e-folded scale).
// Decode: split-K over the context, one CTA per (split, kv head, sequence)
// serving all q heads of the GQA group, then a combine kernel.
#include "../common.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {
namespace {

using namespace dev;

constexpr int kQTile = 64, kKTile = 64, kWarps = 4;

template <int HD>
struct PrefillSmem {
  static constexpr int kStride = HD + 8;  // padded rows: conflict-free ldmatrix
  static constexpr int kQ = kQTile * kStride;
  static constexpr int kKV = kKTile * kStride;
  static constexpr int kBytes = (kQ + 4 * kKV) * 2;  // Q + double-buffered K,V
};

template <int HD>
__global__ void __launch_bounds__(kWarps * 32) attn_prefill_kernel(const bf16* __restrict__ qkv,
                                                                   bf16* __restrict__ out, KvGeom kv,
                                                                   int layer, int seq, int rows,
                                                                   int pos0, int heads,
                                                                   float scale_log2) {
  pdl_trigger();
  pdl_wait();
  using S = PrefillSmem<HD>;
  constexpr int ST = S::kStride;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + S::kQ;        // [2][kKTile][ST]
  bf16* sV = sK + 2 * S::kKV;   // [2][kKTile][ST]

  const int n_qt = (rows + kQTile - 1) / kQTile;
  const int qt = n_qt - 1 - blockIdx.x;  // heaviest (latest) query tiles first
  const int h = blockIdx.y;
  const int kvh = h / (heads / kv.kv_heads);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q_row0 = qt * kQTile;
  const int ldq = (heads + 2 * kv.kv_heads) * HD;
  const int n_keys = pos0 + min(rows, q_row0 + kQTile);  // keys visible to this tile
  const int n_kt = (n_keys + kKTile - 1) / kKTile;
  const int32_t* bt = kv.block_tables + (int64_t)seq * kv.max_blocks;
  const int64_t k_plane = kv.plane(layer, 0, kvh), v_plane = kv.plane(layer, 1, kvh);

  // Q tile -> smem
  for (int i = tid; i < kQTile * CH; i += kWarps * 32) {
    const int r = i / CH, c = i % CH;
    const int gr = q_row0 + r;
    const bf16* src = qkv + (int64_t)(gr < rows ? gr : 0) * ldq + h * HD + c * 8;
    cp_async16(sQ + r * ST + c * 8, src, gr < rows);
  }
  auto load_kv = [&](int buf, int kt) {
    for (int i = tid; i < kKTile * CH; i += kWarps * 32) {
      const int r = i / CH, c = i % CH;
      const int key = kt * kKTile + r;
      const bool ok = key < n_keys;
      const int kk = ok ? key : 0;
      const int32_t page = bt[kk / kv.tpb];
      const bf16* base = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) +
                         (int64_t)(kk % kv.tpb) * HD + c * 8;
      cp_async16(sK + buf * S::kKV + r * ST + c * 8, base + k_plane, ok);
      cp_async16(sV + buf * S::kKV + r * ST + c * 8, base + v_plane, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[j][e] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];
  const int my_row0 = q_row0 + warp * 16 + (lane >> 2);  // rows my_row0 and my_row0 + 8
  const int qpos0 = pos0 + my_row0, qpos1 = qpos0 + 8;

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) load_kv((kt + 1) & 1, kt + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3],
                    sQ + (warp * 16 + (lane & 15)) * ST + kk * 16 + (lane >> 4) * 8);
    }
    const bf16* tK = sK + (kt & 1) * S::kKV;
    const bf16* tV = sV + (kt & 1) * S::kKV;
    // S = Q K^T for 16 rows x 64 keys
    float s[kKTile / 8][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < kKTile / 16; ++j) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3,
                    tK + (j * 16 + (lane & 7) + ((lane >> 4) << 3)) * ST + kk * 16 +
                        ((lane >> 3) & 1) * 8);
        uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
        mma_bf16_16816(s[2 * j], qf[kk], bl);
        mma_bf16_16816(s[2 * j + 1], qf[kk], bh);
      }
    }
    // causal + bounds mask, online softmax (base 2)
    const int key_base = kt * kKTile + (lane & 3) * 2;
    float mx[2] = {m_run[0], m_run[1]};
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = key_base + j * 8 + (e & 1);
        const int qp = (e >> 1) ? qpos1 : qpos0;
        float v = s[j][e] * scale_log2;
        if (key > qp || key >= n_keys) v = -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], lsum[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float base = mx[r] == -INFINITY ? 0.f : mx[r];
      corr[r] = exp2f(m_run[r] - base);
      m_run[r] = mx[r];
      mx[r] = base;
    }
    uint32_t pf[kKTile / 16][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j) {
      const float p0 = exp2f(s[j][0] - mx[0]), p1 = exp2f(s[j][1] - mx[0]);
      const float p2 = exp2f(s[j][2] - mx[1]), p3 = exp2f(s[j][3] - mx[1]);
      lsum[0] += p0 + p1;
      lsum[1] += p2 + p3;
      pf[j / 2][(j & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[j / 2][(j & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * corr[r] + lsum[r];
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
    // O += P V ; P as A fragments: a0/a1 from n8 tile 2t (rows lo/hi), a2/a3 from tile 2t+1
#pragma unroll
    for (int t = 0; t < kKTile / 16; ++t) {
      uint32_t a[4] = {pf[t][0], pf[t][1], pf[t][2], pf[t][3]};
#pragma unroll
      for (int d = 0; d < HD / 16; ++d) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(b0, b1, b2, b3,
                          tV + (t * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * ST + d * 16 +
                              (lane >> 4) * 8);
        uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
        mma_bf16_16816(o[2 * d], a, bl);
        mma_bf16_16816(o[2 * d + 1], a, bh);
      }
    }
    __syncthreads();
  }
  // normalise (quad-reduce the row sums) and store bf16
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  const float inv0 = l_run[0] > 0 ? 1.f / l_run[0] : 0.f;
  const float inv1 = l_run[1] > 0 ? 1.f / l_run[1] : 0.f;
  const int ldo = heads * HD;
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    const int col = h * HD + j * 8 + (lane & 3) * 2;
    if (my_row0 < rows)
      *reinterpret_cast<uint32_t*>(out + (int64_t)my_row0 * ldo + col) =
          pack_bf16x2(o[j][0] * inv0, o[j][1] * inv0);
    if (my_row0 + 8 < rows)
      *reinterpret_cast<uint32_t*>(out + (int64_t)(my_row0 + 8) * ldo + col) =
          pack_bf16x2(o[j][2] * inv1, o[j][3] * inv1);
  }
}

// ---------------------------------------------------------------- decode
constexpr int kSplit = 256;      // keys per split
constexpr int kDecThreads = 128;
constexpr int kMaxGroup = 8;     // q heads per kv head handled per CTA

// partial layout per (seq, q head, split): o[HD] (unnormalised), m, l
template <int HD>
__global__ void __launch_bounds__(kDecThreads) attn_decode_kernel(
    const bf16* __restrict__ qkv, KvGeom kv, int layer, const int32_t* __restrict__ seqs,
    const int32_t* __restrict__ pos, int heads, float scale_log2, float* __restrict__ part,
    int n_splits) {
  pdl_trigger();
  pdl_wait();
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int G = heads / kv.kv_heads;
  const int len = pos[b] + 1;  // the new token's K/V is already appended
  const int k_lo = split * kSplit, k_hi = min(len, k_lo + kSplit);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float sq[kMaxGroup][HD];
  __shared__ float sp[kMaxGroup][kSplit];
  __shared__ float so[kDecThreads / 32][kMaxGroup][HD];
  __shared__ float sm[kMaxGroup], sl[kMaxGroup];
  const int ldq = (heads + 2 * kv.kv_heads) * HD;
  for (int i = tid; i < G * HD; i += kDecThreads)
    sq[i / HD][i % HD] = bf2f(qkv[(int64_t)b * ldq + (kvh * G + i / HD) * HD + i % HD]);
  __syncthreads();
  const int32_t* bt = kv.block_tables + (int64_t)seqs[b] * kv.max_blocks;
  const int64_t k_plane = kv.plane(layer, 0, kvh), v_plane = kv.plane(layer, 1, kvh);
  // scores: half-warp per key, 16 lanes x (HD/16) dims
  constexpr int DPL = HD / 16;
  const int half = lane >> 4, hl = lane & 15;
  // warp-uniform trip count: both half-warps iterate together (full-mask shuffles)
  for (int kb = k_lo + warp * 2; kb < k_hi; kb += kDecThreads / 16) {
    const int key = kb + half;
    const bool valid = key < k_hi;
    float kf[DPL];
    if (valid) {
      const int32_t page = bt[key / kv.tpb];
      const bf16* kr = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) +
                       k_plane + (int64_t)(key % kv.tpb) * HD + hl * DPL;
#pragma unroll
      for (int d = 0; d < DPL; ++d) kf[d] = bf2f(kr[d]);
    } else {
#pragma unroll
      for (int d = 0; d < DPL; ++d) kf[d] = 0.f;
    }
    for (int g = 0; g < G; ++g) {
      float acc = 0.f;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc += kf[d] * sq[g][hl * DPL + d];
      acc += __shfl_xor_sync(0xffffffffu, acc, 8);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (hl == 0 && valid) sp[g][key - k_lo] = acc * scale_log2;
    }
  }
  __syncthreads();
  // per-head max / exp / sum over this split (warp g handles head g, g+4..)
  for (int g = warp; g < G; g += kDecThreads / 32) {
    float mx = -INFINITY;
    for (int k = lane; k < k_hi - k_lo; k += 32) mx = fmaxf(mx, sp[g][k]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int k = lane; k < k_hi - k_lo; k += 32) {
      const float p = exp2f(sp[g][k] - mx);
      sp[g][k] = p;
      s += p;
    }
    s = warp_sum(s);
    if (lane == 0) {
      sm[g] = mx;
      sl[g] = s;
    }
  }
  __syncthreads();
  // O = sum_k p_k V_k : warp w takes keys w, w+4, ...; lane owns HD/32 dims
  constexpr int DV = HD / 32;
  float acc[kMaxGroup][DV];
#pragma unroll
  for (int g = 0; g < kMaxGroup; ++g)
#pragma unroll
    for (int d = 0; d < DV; ++d) acc[g][d] = 0.f;
  for (int key = k_lo + warp; key < k_hi; key += kDecThreads / 32) {
    const int32_t page = bt[key / kv.tpb];
    const bf16* vr = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) + v_plane +
                     (int64_t)(key % kv.tpb) * HD + lane * DV;
    float vf[DV];
#pragma unroll
    for (int d = 0; d < DV; ++d) vf[d] = bf2f(vr[d]);
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
      if (g < G) {
        const float p = sp[g][key - k_lo];
#pragma unroll
        for (int d = 0; d < DV; ++d) acc[g][d] += p * vf[d];
      }
    }
  }
#pragma unroll
  for (int g = 0; g < kMaxGroup; ++g)
    if (g < G)
#pragma unroll
      for (int d = 0; d < DV; ++d) so[warp][g][lane * DV + d] = acc[g][d];
  __syncthreads();
  for (int i = tid; i < G * HD; i += kDecThreads) {
    const int g = i / HD, d = i % HD;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) v += so[w][g][d];
    float* dst = part + (((int64_t)b * heads + kvh * G + g) * n_splits + split) * (HD + 2);
    dst[d] = v;
    if (d == 0) {
      dst[HD] = k_hi > k_lo ? sm[g] : -INFINITY;
      dst[HD + 1] = k_hi > k_lo ? sl[g] : 0.f;
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(HD) attn_combine_kernel(const float* __restrict__ part,
                                                          bf16* __restrict__ out, int heads,
                                                          int n_splits) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
  const float* p = part + ((int64_t)b * heads + h) * n_splits * (HD + 2);
  float mx = -INFINITY;
  for (int s = 0; s < n_splits; ++s) mx = fmaxf(mx, p[s * (HD + 2) + HD]);
  float num = 0.f, den = 0.f;
  for (int s = 0; s < n_splits; ++s) {
    const float m = p[s * (HD + 2) + HD];
    if (m == -INFINITY) continue;
    const float w = exp2f(m - mx);
    num += w * p[s * (HD + 2) + d];
    den += w * p[s * (HD + 2) + HD + 1];
  }
  out[(int64_t)b * heads * HD + h * HD + d] = f2bf(den > 0 ? num / den : 0.f);
}

template <int HD>
void prefill_impl(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                  int pos0, int heads, float scale, cudaStream_t st) {
  const int smem = PrefillSmem<HD>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((rows + kQTile - 1) / kQTile, heads);
  count_launch();
  launch_pdl(attn_prefill_kernel<HD>, dim3(grid), dim3(kWarps * 32), smem, st, qkv, out, kv, layer, seq, rows, pos0,
                                                           heads, scale * 1.4426950408889634f);
}

template <int HD>
void decode_impl(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, const int32_t* seqs,
                 const int32_t* ctx, int n_seqs, int heads, int max_ctx, float scale, float* scratch,
                 cudaStream_t st) {
  const int n_splits = (max_ctx + kSplit - 1) / kSplit;
  dim3 grid(n_splits, kv.kv_heads, n_seqs);
  count_launch(2);
  launch_pdl(attn_decode_kernel<HD>, dim3(grid), dim3(kDecThreads), 0, st, qkv, kv, layer, seqs, ctx, heads,
                                                       scale * 1.4426950408889634f, scratch, n_splits);
  launch_pdl(attn_combine_kernel<HD>, dim3(heads, n_seqs), dim3(HD), 0, st, scratch, out, heads, n_splits);
}

}  // namespace

void launch_attn_prefill(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                         int pos0, int heads, float scale, cudaStream_t st) {
  switch (kv.head_dim) {
    case 64: prefill_impl<64>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    case 96: prefill_impl<96>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    case 128: prefill_impl<128>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    default: break;
  }
}

void launch_attn_decode(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, const int32_t* seqs,
                        const int32_t* ctx, int n_seqs, int heads, int max_ctx, float scale,
                        float* scratch, cudaStream_t st) {
  switch (kv.head_dim) {
    case 64: decode_impl<64>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st); break;
    case 96: decode_impl<96>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st); break;
    case 128: decode_impl<128>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st); break;
    default: break;
  }
}

int decode_scratch_floats(int n_seqs, int heads, int head_dim, int max_ctx) {
  return n_seqs * heads * ((max_ctx + kSplit - 1) / kSplit) * (head_dim + 2);
}

}  // namespace ws

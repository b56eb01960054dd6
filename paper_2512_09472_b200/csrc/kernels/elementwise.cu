// HBM-bound per-token kernels: embedding gather, RMSNorm, SwiGLU, RoPE +
// paged KV append, argmax. Each moves 16-byte vectors with one row (or one
// token x head) per CTA/warp; grids cover all rows so every SM streams.
#include <algorithm>

#include "../common.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {
namespace {

using namespace dev;

// x[r, :] = float(E[tok[r], :])
__global__ void __launch_bounds__(256) embed_kernel(const int32_t* __restrict__ tok,
                                                    const bf16* __restrict__ table,
                                                    float* __restrict__ x, int d) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int64_t t = tok[r];
  const uint4* src = reinterpret_cast<const uint4*>(table + t * d);
  float4* dst = reinterpret_cast<float4*>(x + (int64_t)r * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    uint4 v = __ldg(src + i);
    float2 a = unpack_bf16x2(v.x), b = unpack_bf16x2(v.y), c = unpack_bf16x2(v.z),
           e = unpack_bf16x2(v.w);
    dst[2 * i] = make_float4(a.x, a.y, b.x, b.y);
    dst[2 * i + 1] = make_float4(c.x, c.y, e.x, e.y);
  }
}

// out = bf16(x * rsqrt(mean(x^2) + eps) * w), fp32 math. One CTA per row;
// the row stays in registers (kVec float4 per thread, d <= 4*kT*kVec), so x
// is read from memory exactly once. Few rows (decode) use wide CTAs for
// memory parallelism, many rows (prefill) narrow ones.
template <int kT, int kVec>
__global__ void __launch_bounds__(kT) rmsnorm_kernel(const float* __restrict__ x,
                                                     const bf16* __restrict__ w,
                                                     bf16* __restrict__ out, int d, float eps) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, n4 = d / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)r * d);
  float4 v[kVec];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = threadIdx.x + k * kT;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
  }
  __shared__ float red[kT / 32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < kT / 32; ++k) tot += red[k];
  const float inv = rsqrtf(tot / (float)d + eps);
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  uint2* orow = reinterpret_cast<uint2*>(out + (int64_t)r * d);
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = threadIdx.x + k * kT;
    if (i >= n4) break;
    const uint2 wv = __ldg(wr + i);
    const float2 w0 = unpack_bf16x2(wv.x), w1 = unpack_bf16x2(wv.y);
    uint2 o;
    o.x = pack_bf16x2(v[k].x * inv * w0.x, v[k].y * inv * w0.y);
    o.y = pack_bf16x2(v[k].z * inv * w1.x, v[k].w * inv * w1.y);
    orow[i] = o;
  }
}

// act[r, j] = silu(g) * u. Gate/up rows of Wgu are interleaved in 128-row
// blocks (layout of ws_model_layout), so g = gu[r, 256*(j/128) + j%128] and
// u = gu[r, 256*(j/128) + 128 + j%128]. Used for the skinny (decode) path; the
// tcgen05 GEMM applies SwiGLU in its epilogue instead.
__global__ void __launch_bounds__(256) silu_mul_kernel(const bf16* __restrict__ gu,
                                                       bf16* __restrict__ act, int ffn) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // 8-element group
  if (i >= ffn / 8) return;
  const int j = i * 8;
  const int64_t g_off = (int64_t)r * 2 * ffn + (j >> 7) * 256 + (j & 127);
  const uint4 g = __ldg(reinterpret_cast<const uint4*>(gu + g_off));
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(gu + g_off + 128));
  const uint32_t* gp = &g.x;
  const uint32_t* up = &u.x;
  uint4 o;
  uint32_t* op = &o.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 gv = unpack_bf16x2(gp[k]), uv = unpack_bf16x2(up[k]);
    float s0 = silu(gv.x), s1 = silu(gv.y);
    op[k] = pack_bf16x2(s0 * uv.x, s1 * uv.y);
  }
  reinterpret_cast<uint4*>(act + (int64_t)r * ffn)[i] = o;
}

// One warp per (row, head slot); head slots: [0,H) q heads, [H, H+KV) k heads,
// [H+KV, H+2KV) v heads. rotate_half RoPE on q and k (pairs i, i+hd/2),
// k and v written to the paged cache.
__global__ void __launch_bounds__(256) rope_kv_kernel(bf16* __restrict__ qkv,
                                                      const float2* __restrict__ rope, KvGeom kv,
                                                      int layer, int rows, int heads,
                                                      const int32_t* __restrict__ seq_arr,
                                                      const int32_t* __restrict__ pos_arr, int seq0,
                                                      int pos0) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int slots = heads + 2 * kv.kv_heads;
  const int r = warp / slots, hs = warp % slots;
  if (r >= rows) return;
  const int hd = kv.head_dim, half = hd / 2;
  const int pos = pos_arr ? pos_arr[r] : pos0 + r;
  const int seq = seq_arr ? seq_arr[r] : seq0;
  bf16* vec = qkv + (int64_t)r * slots * hd + (int64_t)hs * hd;
  const bool is_v = hs >= heads + kv.kv_heads;
  const float2* cs = rope + (int64_t)pos * half;
  bf16* dst = nullptr;
  if (hs >= heads) {
    const int kind = is_v ? 1 : 0;
    const int h = is_v ? hs - heads - kv.kv_heads : hs - heads;
    const int32_t page = kv.block_tables[(int64_t)seq * kv.max_blocks + pos / kv.tpb];
    dst = reinterpret_cast<bf16*>(kv.window + (int64_t)page * kv.page_size) + kv.plane(layer, kind, h) +
          (int64_t)(pos % kv.tpb) * hd;
  }
  for (int i = lane; i < half; i += 32) {
    float a = bf2f(vec[i]), b = bf2f(vec[i + half]);
    if (!is_v) {
      const float2 c = cs[i];  // (cos, sin)
      const float ra = a * c.x - b * c.y, rb = b * c.x + a * c.y;
      a = ra;
      b = rb;
      vec[i] = f2bf(a);
      vec[i + half] = f2bf(b);
    }
    if (dst) {
      dst[i] = f2bf(a);
      dst[i + half] = f2bf(b);
    }
  }
}

// Row-wise argmax over fp32 logits (first index on ties, like torch.argmax).
// A row is split over gridDim.x CTAs (a decode step's 128k-entry row on one
// CTA took ~60 us); each CTA reduces its chunk to one 64-bit key =
// (order-preserving float bits << 32) | ~index, so max(key) is the largest
// logit at the smallest index; the last CTA of the row (arrival counter,
// reset by that CTA, so CUDA-graph replays stay valid) reduces the keys.
__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | (uint32_t)(~(uint32_t)i);
}
__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, k, o);
    k = x > k ? x : k;
  }
  __shared__ unsigned long long sk[32];
  if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x < 32) {
    k = threadIdx.x < blockDim.x / 32 ? sk[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, k, o);
      k = x > k ? x : k;
    }
  }
  return k;  // valid in thread 0
}

__global__ void __launch_bounds__(256) argmax_kernel(const float* __restrict__ logits, int V, int chunk,
                                                     int32_t* __restrict__ out, unsigned long long* part,
                                                     unsigned int* count) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y, nb = gridDim.x, b = blockIdx.x;
  const float* row = logits + (int64_t)r * V;
  const int lo = b * chunk, hi = min(V, lo + chunk);
  unsigned long long k = 0ull;
  if ((V & 3) == 0) {  // rows 16-byte aligned, chunk a multiple of 4
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int i = lo / 4 + threadIdx.x; i < hi / 4; i += blockDim.x) {
      const float4 v = __ldcs(r4 + i);
      unsigned long long x = argmax_key(v.x, 4 * i);
      x = max(x, argmax_key(v.y, 4 * i + 1));
      x = max(x, argmax_key(v.z, 4 * i + 2));
      x = max(x, argmax_key(v.w, 4 * i + 3));
      k = max(k, x);
    }
  } else {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) k = max(k, argmax_key(row[i], i));
  }
  k = block_max_u64(k);
  if (nb == 1) {
    if (threadIdx.x == 0) out[r] = (int32_t)~(uint32_t)k;
    return;
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[(int64_t)r * nb + b] = k;
    __threadfence();
    last = atomicAdd(count + r, 1u) == (unsigned)nb - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  unsigned long long m = 0ull;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) m = max(m, __ldcg(part + (int64_t)r * nb + i));
  m = block_max_u64(m);
  if (threadIdx.x == 0) {
    out[r] = (int32_t)~(uint32_t)m;
    count[r] = 0u;  // ready for the next launch (graph replays included)
  }
}

__global__ void __launch_bounds__(256) add_f32_kernel(float4* __restrict__ x, const float4* __restrict__ p,
                                                      int64_t n4) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = x[i];
    const float4 b = p[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    x[i] = a;
  }
}

__global__ void __launch_bounds__(256) gather_vocab_kernel(const float* __restrict__ g, float* __restrict__ out,
                                                           int tp, int rows, int vs) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y, shard = blockIdx.z;
  const float* src = g + ((int64_t)shard * rows + r) * vs;
  float* dst = out + (int64_t)r * tp * vs + (int64_t)shard * vs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < vs; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

}  // namespace

void launch_add_f32(float* x, const float* p, int64_t count, cudaStream_t st) {
  count_launch();
  const int64_t n4 = count / 4;  // hidden sizes are multiples of 32
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  launch_pdl(add_f32_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<float4*>(x), reinterpret_cast<const float4*>(p), n4);
}

// x (fp32 residual) += p (bf16 row-parallel partial, already summed over the TP group)
__global__ void __launch_bounds__(256) add_bf16_f32_kernel(float4* __restrict__ x, const uint2* __restrict__ p,
                                                           int64_t n4) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = x[i];
    const uint2 b = p[i];
    a.x += __uint_as_float(b.x << 16);
    a.y += __uint_as_float(b.x & 0xffff0000u);
    a.z += __uint_as_float(b.y << 16);
    a.w += __uint_as_float(b.y & 0xffff0000u);
    x[i] = a;
  }
}

void launch_add_bf16_f32(float* x, const bf16* p, int64_t count, cudaStream_t st) {
  count_launch();
  const int64_t n4 = count / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  launch_pdl(add_bf16_f32_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<float4*>(x),
             reinterpret_cast<const uint2*>(p), n4);
}

void launch_gather_vocab(const float* g, float* out, int tp, int rows, int vs, cudaStream_t st) {
  count_launch();
  dim3 grid((vs + 1023) / 1024, rows, tp);
  launch_pdl(gather_vocab_kernel, dim3(grid), dim3(256), 0, st, g, out, tp, rows, vs);
}

void launch_embed(const int32_t* tokens, const bf16* table, float* x, int n, int d, cudaStream_t st) {
  count_launch();
  launch_pdl(embed_kernel, dim3(n), dim3(256), 0, st, tokens, table, x, d);
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* out, int rows, int d, float eps,
                    cudaStream_t st) {
  count_launch();
  if (rows < 2 * kNumSMs) {  // decode rows
    if (d <= 4096)
      launch_pdl(rmsnorm_kernel<512, 2>, dim3(rows), dim3(512), 0, st, x, w, out, d, eps);
    else
      launch_pdl(rmsnorm_kernel<512, 4>, dim3(rows), dim3(512), 0, st, x, w, out, d, eps);
  } else if (d <= 1024) {
    launch_pdl(rmsnorm_kernel<128, 2>, dim3(rows), dim3(128), 0, st, x, w, out, d, eps);
  } else if (d <= 4096) {
    // 128 threads x 8 float4. 256 x 4 measured 11.7 -> 10.1 us per 2048-row
    // launch (ncu) but sums each row's squares in a different order, which
    // flipped two bf16 near-tie greedy tokens of the parity suite (Llama-3-8B
    // full depth seed 8, Phi-3 full width): not worth 0.4% of a prefill.
    launch_pdl(rmsnorm_kernel<128, 8>, dim3(rows), dim3(128), 0, st, x, w, out, d, eps);
  } else {
    launch_pdl(rmsnorm_kernel<128, 16>, dim3(rows), dim3(128), 0, st, x, w, out, d, eps);
  }
}

void launch_silu_mul(const bf16* gu, bf16* act, int rows, int ffn, cudaStream_t st) {
  dim3 grid((ffn / 8 + 255) / 256, rows);
  count_launch();
  launch_pdl(silu_mul_kernel, dim3(grid), dim3(256), 0, st, gu, act, ffn);
}

void launch_rope_kv(bf16* qkv, const float2* rope, const KvGeom& kv, int layer, int rows, int heads,
                    const int32_t* seq, const int32_t* pos, int seq0, int pos0, cudaStream_t st) {
  const int64_t warps = (int64_t)rows * (heads + 2 * kv.kv_heads);
  const int blocks = (int)((warps * 32 + 255) / 256);
  count_launch();
  launch_pdl(rope_kv_kernel, dim3(blocks), dim3(256), 0, st, qkv, rope, kv, layer, rows, heads, seq, pos, seq0, pos0);
}

void launch_argmax(const float* logits, int M, int V, int32_t* out, void* scratch, cudaStream_t st) {
  // enough CTAs to stream the logits from every SM: ~2 per SM over all rows,
  // chunks of >= 2048 logits, at most kArgmaxMaxSplit per row
  int nb = scratch ? std::min({kArgmaxMaxSplit, std::max(1, 2 * kNumSMs / M), (V + 2047) / 2048}) : 1;
  const int chunk = ((V + nb - 1) / nb + 3) / 4 * 4;
  nb = (V + chunk - 1) / chunk;
  auto* part = static_cast<unsigned long long*>(scratch);
  auto* count = reinterpret_cast<unsigned int*>(part + (int64_t)kArgmaxMaxRows * kArgmaxMaxSplit);
  count_launch();
  launch_pdl(argmax_kernel, dim3(nb, M), dim3(256), 0, st, logits, V, chunk, out, part, count);
}

}  // namespace ws

// Baseline tensor-core GEMM (mma.sync m16n8k16 bf16 -> fp32, cp.async
// 4-stage pipeline, XOR-swizzled smem, 128x128x32 CTA tile, 8 warps of 64x32).
// This is the legacy-path kernel the tcgen05 GEMM (gemm_tc.cu) must beat; it
// also serves as its parity reference in the GPU tests. Plus the skinny
// weight-streaming GEMV used for decode rows and the lm_head.
#include "../common.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {
namespace {

using namespace dev;

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 4, THREADS = 256;
constexpr int TILE_ELEMS = BM * BK;  // A and B tiles have the same shape

// element offset of 16B chunk `c` (0..3) of row `r` in a swizzled [128][32] tile
__device__ __forceinline__ int swz(int r, int c) { return r * BK + ((c ^ ((r >> 1) & 3)) << 3); }

__global__ void __launch_bounds__(THREADS) gemm_mma_kernel(const bf16* __restrict__ A,
                                                           const bf16* __restrict__ B, int M, int N,
                                                           int K, int epi, void* __restrict__ Cout,
                                                           const bf16* __restrict__ bias) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sA = reinterpret_cast<bf16*>(smem_raw);
  bf16* sB = sA + STAGES * TILE_ELEMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, 64 x 32 each
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int n_k = K / BK;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * THREADS;  // 0..511
      const int r = idx >> 2, c = idx & 3;
      const int gm = m0 + r, gn = n0 + r;
      const bf16* srcA = A + (int64_t)(gm < M ? gm : 0) * K + k0 + c * 8;
      const bf16* srcB = B + (int64_t)(gn < N ? gn : 0) * K + k0 + c * 8;
      cp_async16(sA + stage * TILE_ELEMS + swz(r, c), srcA, gm < M);
      cp_async16(sB + stage * TILE_ELEMS + swz(r, c), srcB, gn < N);
    }
  };

  float acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < n_k) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < n_k; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < n_k) load_stage(nxt % STAGES, nxt);
    cp_async_commit();
    const bf16* tA = sA + (kt % STAGES) * TILE_ELEMS;
    const bf16* tB = sB + (kt % STAGES) * TILE_ELEMS;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t af[4][4], bfr[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 64 + i * 16 + (lane & 15);
        ldmatrix_x4(af[i][0], af[i][1], af[i][2], af[i][3], tA + swz(r, kk * 2 + (lane >> 4)));
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = wn * 32 + j * 16 + (lane & 7) + ((lane >> 4) << 3);
        uint32_t r0, r1, r2, r3;
        ldmatrix_x4(r0, r1, r2, r3, tB + swz(r, kk * 2 + ((lane >> 3) & 1)));
        bfr[2 * j][0] = r0;
        bfr[2 * j][1] = r1;
        bfr[2 * j + 1][0] = r2;
        bfr[2 * j + 1][1] = r3;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_bf16_16816(acc[i][j], af[i], bfr[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue straight from registers: c0,c1 at (row, col..col+1), c2,c3 at row+8.
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + wn * 32 + j * 8 + (lane & 3) * 2;
      if (col >= N) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m0 + wm * 64 + i * 16 + (lane >> 2) + h * 8;
        if (row >= M) continue;
        float v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
        if (epi == (int)Epi::kAddF32) {
          float2* c = reinterpret_cast<float2*>(static_cast<float*>(Cout) + (int64_t)row * N + col);
          float2 o = *c;
          o.x += v0;
          o.y += v1;
          *c = o;
        } else if (epi == 3) {
          *reinterpret_cast<float2*>(static_cast<float*>(Cout) + (int64_t)row * N + col) =
              make_float2(v0, v1);
        } else {
          if (epi == (int)Epi::kBiasBf16) {
            v0 += bf2f(bias[col]);
            v1 += bf2f(bias[col + 1]);
          }
          *reinterpret_cast<uint32_t*>(static_cast<bf16*>(Cout) + (int64_t)row * N + col) =
              pack_bf16x2(v0, v1);
        }
      }
    }
}

// ---- skinny GEMM: M <= 16 rows of A against all N rows of B (HBM bound).
// One warp owns 2 output columns at a time; lanes split K in 16 B vectors.
template <int MR>
__global__ void __launch_bounds__(256) gemv_kernel(const bf16* __restrict__ A,
                                                   const bf16* __restrict__ B, int M, int N, int K,
                                                   int epi, void* __restrict__ Cout,
                                                   const bf16* __restrict__ bias) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_warps = (gridDim.x * blockDim.x) >> 5;
  const int kv = K / 8;  // 16-byte vectors per row
  for (int n = gw * 2; n < N; n += n_warps * 2) {
    const bool two = n + 1 < N;
    const uint4* b0 = reinterpret_cast<const uint4*>(B + (int64_t)n * K);
    const uint4* b1 = reinterpret_cast<const uint4*>(B + (int64_t)(two ? n + 1 : n) * K);
    float acc0[MR], acc1[MR];
#pragma unroll
    for (int m = 0; m < MR; ++m) acc0[m] = acc1[m] = 0.f;
    for (int i = lane; i < kv; i += 32) {
      const uint4 w0 = __ldg(b0 + i), w1 = __ldg(b1 + i);
      float2 wa[4], wb[4];
      wa[0] = unpack_bf16x2(w0.x); wa[1] = unpack_bf16x2(w0.y);
      wa[2] = unpack_bf16x2(w0.z); wa[3] = unpack_bf16x2(w0.w);
      wb[0] = unpack_bf16x2(w1.x); wb[1] = unpack_bf16x2(w1.y);
      wb[2] = unpack_bf16x2(w1.z); wb[3] = unpack_bf16x2(w1.w);
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        if (m < M) {
          const uint4 xv = __ldg(reinterpret_cast<const uint4*>(A + (int64_t)m * K) + i);
          float2 x[4] = {unpack_bf16x2(xv.x), unpack_bf16x2(xv.y), unpack_bf16x2(xv.z),
                         unpack_bf16x2(xv.w)};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc0[m] += x[q].x * wa[q].x + x[q].y * wa[q].y;
            acc1[m] += x[q].x * wb[q].x + x[q].y * wb[q].y;
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (m >= M) break;
      float v0 = dev::warp_sum(acc0[m]);
      float v1 = dev::warp_sum(acc1[m]);
      if (lane == 0) {
        for (int t = 0; t < (two ? 2 : 1); ++t) {
          const int col = n + t;
          float v = t ? v1 : v0;
          if (epi == (int)Epi::kAddF32) {
            static_cast<float*>(Cout)[(int64_t)m * N + col] += v;
          } else if (epi == 3) {
            static_cast<float*>(Cout)[(int64_t)m * N + col] = v;
          } else {
            if (epi == (int)Epi::kBiasBf16) v += bf2f(bias[col]);
            static_cast<bf16*>(Cout)[(int64_t)m * N + col] = f2bf(v);
          }
        }
      }
    }
  }
}

}  // namespace

void launch_gemm_mma(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                     const bf16* bias, cudaStream_t st) {
  const int smem = STAGES * 2 * TILE_ELEMS * (int)sizeof(bf16);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  count_launch();
  launch_pdl(gemm_mma_kernel, dim3(grid), dim3(THREADS), smem, st, A, B, M, N, K, (int)epi, C, bias);
}

void launch_gemm(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                 const bf16* bias, cudaStream_t st) {
  if (M <= 128) {
    TcEpilogue e;
    e.mode = epi;
    e.C = C;
    e.bias = bias;
    if (launch_gemm_skinny(A, B, M, N, K, e, st)) return;
  }
  if (M < 16) {
    count_fallback(kFallbackGemv, "GEMM with < 16 rows outside the skinny tcgen05 tiling runs the CUDA-core GEMV");
    launch_gemv(A, B, M, N, K, epi, C, bias, st);
  } else if (!launch_gemm_tc(A, B, M, N, K, epi, C, bias, st)) {
    count_fallback(kFallbackGemmMma, "GEMM shape outside the tcgen05 tiling runs the mma.sync kernel");
    launch_gemm_mma(A, B, M, N, K, epi, C, bias, st);
  }
}

void launch_gemv(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C,
                 const bf16* bias, cudaStream_t st) {
  const int warps_needed = (N + 1) / 2;
  int blocks = (warps_needed + 7) / 8;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  count_launch();
  if (M <= 1)
    launch_pdl(gemv_kernel<1>, dim3(blocks), dim3(256), 0, st, A, B, M, N, K, (int)epi, C, bias);
  else if (M <= 4)
    launch_pdl(gemv_kernel<4>, dim3(blocks), dim3(256), 0, st, A, B, M, N, K, (int)epi, C, bias);
  else if (M <= 8)
    launch_pdl(gemv_kernel<8>, dim3(blocks), dim3(256), 0, st, A, B, M, N, K, (int)epi, C, bias);
  else
    launch_pdl(gemv_kernel<16>, dim3(blocks), dim3(256), 0, st, A, B, M, N, K, (int)epi, C, bias);
}

}  // namespace ws

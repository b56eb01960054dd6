// Lossless bf16 weight unpacking for the packed layer stream (cold start).
//
// Format 1 (Huffman, the default): lo[n] as below, then the exponents as a
// length-limited (<= 12 bit) canonical Huffman code, LSB-first, in blocks of
// 1024 weights whose bitstreams start on 32-bit words:
//   lo [n] | lut [4096] u16 (symbol | length << 8, indexed by the next 12 bits)
//        | block word offsets [ceil(n/1024)] u32 | words [] u32
// ~10.6 bits per weight (the exponent entropy is ~2.6 bits). One thread
// decodes one block through a shared-memory LUT and writes 16-byte vectors.
//
// Format 0 (fixed 4-bit codes):
// A bf16 weight is sign(1) | exponent(8) | mantissa(7). Trained and
// synthetic weights use a narrow band of exponents (entropy ~2.5 bits), so
// the host image of each streamed range is stored as
//   lo    [n]          uint8  sign << 7 | mantissa
//   codes [ceil(n/2)]  uint8  two 4-bit codes: exponent - e_base (0..14), 15 = escape
//   idx   [n_esc]      uint32 positions of the escaped values (ascending)
//   exp   [n_esc]      uint8  their exponents
// (sections 16-byte aligned): 12 bits per weight plus escapes, so the PCIe
// stream carries ~25% fewer bytes. The copy engine moves the packed range
// into a device staging buffer and these kernels rebuild the exact bf16 bits
// in the slot — HBM-bound, ~0.1 ms per 436 MB layer, on their own stream.
#include <algorithm>
#include <cstdint>

#include "../common.h"
#include "ops.cuh"

namespace ws {
namespace {

__device__ __forceinline__ uint32_t bf16_bits(uint32_t lo, uint32_t e) {
  return ((lo & 0x80u) << 8) | ((e & 0xFFu) << 7) | (lo & 0x7Fu);
}

// 16 weights per thread per step: 16 lo bytes + 8 code bytes -> 32 output bytes
__global__ void __launch_bounds__(256) unpack_bf16_kernel(uint16_t* __restrict__ dst, const uint8_t* __restrict__ lo,
                                                          const uint8_t* __restrict__ codes, int64_t n, int e_base) {
  const int64_t groups = n / 16;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const uint4 L = __ldg(reinterpret_cast<const uint4*>(lo) + g);
    const uint2 C = __ldg(reinterpret_cast<const uint2*>(codes) + g);
    const uint32_t lw[4] = {L.x, L.y, L.z, L.w}, cw[2] = {C.x, C.y};
    uint32_t out[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // values 2k, 2k+1
      const uint32_t l0 = (lw[k >> 1] >> (16 * (k & 1))) & 0xFFu, l1 = (lw[k >> 1] >> (16 * (k & 1) + 8)) & 0xFFu;
      const uint32_t cb = (cw[k >> 2] >> (8 * (k & 3))) & 0xFFu;  // code byte of values 2k, 2k+1
      out[k] = bf16_bits(l0, e_base + (cb & 0xFu)) | (bf16_bits(l1, e_base + (cb >> 4)) << 16);
    }
    uint4* d = reinterpret_cast<uint4*>(dst) + 2 * g;
    d[0] = make_uint4(out[0], out[1], out[2], out[3]);
    d[1] = make_uint4(out[4], out[5], out[6], out[7]);
  }
  // tail (n % 16 values), one thread each
  const int64_t t = groups * 16 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    const uint32_t c = (codes[t >> 1] >> (4 * (t & 1))) & 0xFu;
    dst[t] = (uint16_t)bf16_bits(lo[t], e_base + c);
  }
}

constexpr int kHuffBlock = 1024, kHuffBits = 12;

__global__ void __launch_bounds__(128) unpack_huff_kernel(uint16_t* __restrict__ dst, const uint8_t* __restrict__ lo,
                                                          const uint16_t* __restrict__ lut_g,
                                                          const uint32_t* __restrict__ offs,
                                                          const uint32_t* __restrict__ words, int64_t n) {
  __shared__ uint16_t lut[1 << kHuffBits];
  for (int i = threadIdx.x; i < (1 << kHuffBits); i += blockDim.x) lut[i] = lut_g[i];
  __syncthreads();
  const int64_t nb = (n + kHuffBlock - 1) / kHuffBlock;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint32_t* w = words + offs[b];
  uint64_t buf = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  int have = 64, next = 2;
  const int64_t v0 = b * kHuffBlock;
  const int cnt = (int)(n - v0 < kHuffBlock ? n - v0 : kHuffBlock);
  const uint8_t* l = lo + v0;
  uint16_t* d = dst + v0;
  int v = 0;
  for (; v + 8 <= cnt; v += 8) {
    const uint2 L = *reinterpret_cast<const uint2*>(l + v);
    uint32_t out[4];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t ent = lut[buf & ((1u << kHuffBits) - 1)];
      const int len = ent >> 8;
      buf >>= len;
      have -= len;
      if (have < 32) {
        buf |= (uint64_t)w[next++] << have;
        have += 32;
      }
      const uint32_t lb = ((k < 4 ? L.x : L.y) >> (8 * (k & 3))) & 0xFFu;
      const uint32_t bits = bf16_bits(lb, ent & 0xFFu);
      if (k & 1)
        out[k >> 1] |= bits << 16;
      else
        out[k >> 1] = bits;
    }
    *reinterpret_cast<uint4*>(d + v) = make_uint4(out[0], out[1], out[2], out[3]);
  }
  for (; v < cnt; ++v) {  // last block's tail
    const uint32_t ent = lut[buf & ((1u << kHuffBits) - 1)];
    const int len = ent >> 8;
    buf >>= len;
    have -= len;
    if (have < 32) {
      buf |= (uint64_t)w[next++] << have;
      have += 32;
    }
    d[v] = (uint16_t)bf16_bits(l[v], ent & 0xFFu);
  }
}

// escaped values carry their own exponent (runs after the bulk pass)
__global__ void __launch_bounds__(256) unpack_escapes_kernel(uint16_t* __restrict__ dst, const uint8_t* __restrict__ lo,
                                                             const uint32_t* __restrict__ idx,
                                                             const uint8_t* __restrict__ exps, int64_t n_esc) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_esc; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx[j];
    dst[i] = (uint16_t)bf16_bits(lo[i], exps[j]);
  }
}

}  // namespace

int64_t packed_align16(int64_t v) { return (v + 15) / 16 * 16; }

void packed_sections(int64_t n, int64_t n_esc, int64_t* codes_off, int64_t* idx_off, int64_t* exp_off,
                     int64_t* total) {
  *codes_off = packed_align16(n);
  *idx_off = packed_align16(*codes_off + (n + 1) / 2);
  *exp_off = packed_align16(*idx_off + 4 * n_esc);
  *total = packed_align16(*exp_off + n_esc);
}

void huff_sections(int64_t n, int64_t* lut_off, int64_t* offs_off, int64_t* words_off) {
  *lut_off = packed_align16(n);
  *offs_off = *lut_off + 2 * (1 << kHuffBits);
  *words_off = packed_align16(*offs_off + 4 * ((n + kHuffBlock - 1) / kHuffBlock));
}

void launch_unpack_huff(void* dst, const void* packed, int64_t n, cudaStream_t st) {
  int64_t lut_off, offs_off, words_off;
  huff_sections(n, &lut_off, &offs_off, &words_off);
  const uint8_t* p = static_cast<const uint8_t*>(packed);
  const int64_t nb = (n + kHuffBlock - 1) / kHuffBlock;
  count_launch();
  unpack_huff_kernel<<<(unsigned)((nb + 127) / 128), 128, 0, st>>>(
      static_cast<uint16_t*>(dst), p, reinterpret_cast<const uint16_t*>(p + lut_off),
      reinterpret_cast<const uint32_t*>(p + offs_off), reinterpret_cast<const uint32_t*>(p + words_off), n);
}

void launch_unpack_bf16(void* dst, const void* packed, int64_t n, int e_base, int64_t n_esc, cudaStream_t st) {
  int64_t codes_off, idx_off, exp_off, total;
  packed_sections(n, n_esc, &codes_off, &idx_off, &exp_off, &total);
  const uint8_t* p = static_cast<const uint8_t*>(packed);
  const int blocks = (int)std::min<int64_t>(kNumSMs * 8, (n / 16 + 255) / 256 + 1);
  count_launch();
  unpack_bf16_kernel<<<blocks, 256, 0, st>>>(static_cast<uint16_t*>(dst), p, p + codes_off, n, e_base);
  if (n_esc > 0) {
    count_launch();
    unpack_escapes_kernel<<<(int)std::min<int64_t>(kNumSMs * 4, (n_esc + 255) / 256), 256, 0, st>>>(
        static_cast<uint16_t*>(dst), p, reinterpret_cast<const uint32_t*>(p + idx_off), p + exp_off, n_esc);
  }
}

}  // namespace ws

// tcgen05 flash-attention prefill over the paged KV pool (sm_100a).
//
// One CTA = 128 queries of one q head (GQA: its kv head = h / group), K/V
// tiles of 128 keys gathered page by page. Warp roles (416 threads):
//   warps 0-7  softmax + correction: warps w and w+4 share TMEM lanes
//              32(w%4).. (query rows) and split the 128 key columns of S_j
//              in halves, so two warps per SM sub-partition issue the
//              exp2/max/sum stream. The row max is exchanged through smem
//              each tile; P_j goes to SMEM as bf16 (K-major SW128); the TMEM
//              output accumulator is rescaled only when the running max grows
//              by more than 2^8 (exact: the final O/l uses the same max).
//   warps 9-12 producers: Q (cp.async, once); K_j/V_j by TMA page-row boxes
//              from the block table (or a cp.async gather when pages do not
//              hold 16-token runs) into SWIZZLE_128B smem tiles.
//   warp 8     TMEM allocator + single-thread MMA issuer:
//              S_j = Q K_j^T   (M=128, N=128, K=hd; both operands K-major)
//              O  += P_j V_j   (M=128, N=hd, K=128; V is MN-major — no transpose)
//              S is double-buffered in TMEM so QK^T of tile j+1 overlaps the
//              softmax of tile j. TMEM: S0 [0,128) S1 [128,256) O [256,256+hd).
#include <cuda.h>

#include <mutex>

#include "../common.h"
#include "../driver.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {
namespace {

using namespace dev;

constexpr int kRows = 128, kKeys = 128, kThreads = 416;

#ifdef WS_ATTN_TRACE
// debug timeline of block (0,0): [event][j] = clock64 (events: 0 S issued,
// 1 PV issued, 2 softmax got S, 3 softmax released P)
__device__ long long g_attn_trace[8][64];
#define TRACE(ev, j) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 64) g_attn_trace[ev][j] = clock64(); } while (0)
// per-CTA [start (after pdl_wait), end, smid] in globaltimer ns, grid order
__device__ long long g_attn_cta[4096][3];
__device__ __forceinline__ long long attn_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define TRACE(ev, j) do { } while (0)
#endif

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#ifdef WS_DEBUG_WAIT
  // watchdog build: report the stuck barrier instead of hanging
  for (long long spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin == 20000000 && (threadIdx.x & 31) == 0)
      printf("attn_tc stuck: block (%d,%d) thread %d bar@%u parity %u\n", blockIdx.x, blockIdx.y, threadIdx.x,
             bar & 0xFFF, parity);
    if (spin == 400000000) asm volatile("trap;");
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ float fast_exp2(float x) {  // one MUFU op, no range fix-up branches
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ bool mbar_ready(uint32_t bar, uint32_t parity) {  // non-blocking probe
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A operand from TMEM (the P tile, 128 lanes x 8 packed columns per K=16 step)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// SWIZZLE_128B smem descriptor (version 1); LBO only matters for MN-major.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, M=128
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kRows >> 4) << 24);
}

#define TLD32(taddr, v)                                                                            \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"             \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),   \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),             \
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),             \
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])              \
      : "r"(taddr))
#define TST32(taddr, v)                                                                            \
  asm volatile(                                                                                    \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr), \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),     \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),          \
      "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),          \
      "r"(v[30]), "r"(v[31]))

constexpr int NS = 3;  // K and V ring stages (TMA page gathers take ~2 us; 3 tiles in flight hide them)

template <int HD>
struct Smem {
  static constexpr int kTile = kRows * HD * 2;     // Q, K or V tile: [HD/64 blocks][128 rows][128 B]
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;            // NS stages
  static constexpr int kV = kK + NS * kTile;       // NS stages
  static constexpr int kX = kV + NS * kTile;       // [2 halves][128 rows] fp32 row-max / row-sum exchange
  static constexpr int kBar = kX + 2 * kRows * 4;
  static constexpr int kBytes = kBar + 256 + 1024;  // barriers + alignment slack
};

// barrier indices
constexpr int kQFull = 0, kKFull = 1, kKEmpty = kKFull + NS, kVFull = kKEmpty + NS, kVEmpty = kVFull + NS,
              kSFull = kVEmpty + NS, kSEmpty = kSFull + 2, kPFull = kSEmpty + 2, kPvDone = kPFull + 2,
              kTmemSlot = kPvDone + 1;

// byte offset of 16-byte chunk c (0 .. 2*HD/16-1 across the row) of row r in a
// [blocks][128][128 B] SWIZZLE_128B tile
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 3) * (kRows * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int HD, bool TMA>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ out, KvGeom kv, int layer, int seq,
                   int rows, int pos0, int heads, float scale_log2, const __grid_constant__ CUtensorMap kvmap) {
  using S = Smem<HD>;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);  // generic pointer to the aligned base
  const uint32_t bar = base + S::kBar;
  // K_j is released right after S_j (QK^T) retires, V_j after PV_j, so the
  // gathers of K_{j+3} / V_{j+3} overlap the softmax of tile j.
  auto B = [&](int i) { return bar + 8 * i; };
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + S::kBar + kTmemSlot * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (rows + kRows - 1) / kRows;
  // grid = (heads, q tiles): CTAs launch in blockIdx order, so every head's
  // heaviest (latest) query tile goes first and the tail holds the light ones
  const int qt = n_qt - 1 - blockIdx.y;
  const int h = blockIdx.x;
  const int kvh = h / (heads / kv.kv_heads);
  const int q0 = qt * kRows;
  const int n_keys = pos0 + min(rows, q0 + kRows);
  const int n_kt = (n_keys + kKeys - 1) / kKeys;
  // HD is the smem / TMEM tile width; the model's head_dim may be smaller
  // (Phi-3: 96 in 128-wide tiles): Q/K/V columns past it are zero, so S and
  // the first hd columns of O are exact and the rest is never stored.
  const int hd = kv.head_dim;
  const int ldq = (heads + 2 * kv.kv_heads) * hd;

  if (threadIdx.x == 0) {
    mbar_init(B(kQFull), 128);
    for (int i = 0; i < NS; ++i) {
      mbar_init(B(kKFull + i), TMA ? 1 : 64);  // TMA thread (expect_tx) or 64 cp.async threads
      mbar_init(B(kKEmpty + i), 1);            // MMA commit after S_j
      mbar_init(B(kVFull + i), TMA ? 1 : 64);
      mbar_init(B(kVEmpty + i), 1);            // MMA commit after PV_j
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(B(kSFull + i), 1);     // MMA commit
      mbar_init(B(kSEmpty + i), 256);  // softmax threads read S
      mbar_init(B(kPFull + i), 256);   // softmax threads wrote P (into the same TMEM columns)
    }
    mbar_init(B(kPvDone), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if constexpr (TMA) {
    // K/V rows a tile does not load keep stale data; start from finite zeros
    for (int i = threadIdx.x; i < 2 * NS * S::kTile / 16; i += kThreads)
      reinterpret_cast<uint4*>(gbase + S::kK)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(B(kTmemSlot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // everything above is prologue; global data from here on
#ifdef WS_ATTN_TRACE
  const int cta_id = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0 && cta_id < 4096) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_attn_cta[cta_id][0] = attn_gtimer();
    g_attn_cta[cta_id][2] = smid;
  }
#endif

  if (warp >= 9) {
    // ===================== producers: warps 9-10 gather K, warps 11-12 gather V =====================
    const int t = threadIdx.x - 288;
    for (int i = t; i < kRows * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const int gr = q0 + r;
      const bf16* src = qkv + (int64_t)(gr < rows ? gr : 0) * ldq + h * hd + (c * 8 < hd ? c * 8 : 0);
      cp_async16(gbase + S::kQ + swz(r, c), src, gr < rows && c * 8 < hd);
    }
    cp_async_arrive(B(kQFull));
    const bool is_v = t >= 64;
    const int u = t & 63;  // rows u and u + 64 of every tile
    const int32_t* bt = kv.block_tables + (int64_t)seq * kv.max_blocks;
    const int64_t plane = kv.plane(layer, is_v ? 1 : 0, kvh);
    const uint32_t ring = is_v ? S::kV : S::kK;
    const int full0 = is_v ? kVFull : kKFull, empty0 = is_v ? kVEmpty : kKEmpty;
    if constexpr (TMA) {
      // One thread per ring issues 8-row TMA boxes (one per run of 8 tokens of
      // a page; tokens-per-block is a multiple of 8): 16 x HD/64 bulk copies
      // per tile instead of 2048 16-byte LDGSTS. Groups past the last key are
      // skipped (their smem rows hold finite stale data and are masked).
      if (u < 32) {  // the first warp of the ring's producer pair
        const int rows_pp = (int)(kv.page_size / (HD * 2));
        const int plane_rows = (int)(plane / HD);
        // lane g resolves group g's page (16 block-table loads in parallel,
        // one tile ahead), lane 0 issues the bulk copies
        auto row_of = [&](int j) {
          const int key0 = j * kKeys + (u & 7) * 16;
          const int blk = key0 / kv.tpb, slot = key0 - blk * kv.tpb;
          return key0 < n_keys ? bt[blk] * rows_pp + plane_rows + slot : 0;
        };
        int y_next = row_of(0);
        for (int j = 0; j < n_kt; ++j) {
          const int st = j % NS;
          const int y = y_next;
          if (j + 1 < n_kt) y_next = row_of(j + 1);
          const int groups = min(kKeys / 16, (n_keys - j * kKeys + 15) / 16);
          if (u == 0) {
            mbar_wait(B(empty0 + st), ((j / NS) & 1) ^ 1);
            tma_expect(B(full0 + st), (uint32_t)(groups * (HD / 64) * 2048));
          }
          for (int g = 0; g < groups; ++g) {
            const int yg = __shfl_sync(0xffffffffu, y, g);
            if (u == 0) {
#pragma unroll
              for (int hh = 0; hh < HD / 64; ++hh)
                tma_load_2d(base + ring + st * S::kTile + hh * (kRows * 128) + g * 2048, &kvmap,
                            B(full0 + st), hh * 64, yg);
            }
          }
        }
      }
    } else {
    for (int j = 0; j < n_kt; ++j) {
      const int st = j % NS;
      mbar_wait(B(empty0 + st), ((j / NS) & 1) ^ 1);
      uint8_t* dst = gbase + ring + st * S::kTile;
      // CH consecutive lanes cover one key row (HD*2 contiguous bytes, coalesced);
      // this thread walks rows r, r+RS, ... with its (block, slot) position
      // advanced incrementally — one integer division per tile, not per chunk.
      constexpr int RS = 64 / CH;
      const int c = u % CH;
      int r = u / CH;
      int key = j * kKeys + r;
      int blk = key / kv.tpb, slot = key - blk * kv.tpb;
      const char* wbase = kv.window;
#pragma unroll 4
      for (int k = 0; k < kKeys / RS; ++k) {
        const bool ok = key < n_keys;
        const int32_t page = bt[ok ? blk : 0];
        const bf16* row = reinterpret_cast<const bf16*>(wbase + (int64_t)page * kv.page_size) + plane +
                          (int64_t)(ok ? slot : 0) * hd;
        cp_async16(dst + swz(r, c), row + (c * 8 < hd ? c * 8 : 0), ok && c * 8 < hd);
        r += RS;
        key += RS;
        slot += RS;
        while (slot >= kv.tpb) {
          slot -= kv.tpb;
          ++blk;
        }
      }
      cp_async_arrive(B(full0 + st));
    }
    }
  } else if (warp == 8) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(kKeys, false), id_pv = idesc(HD, true);
      const uint32_t tO = tmem + 256;
      mbar_wait(B(kQFull), 0);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      auto issue_s = [&](int j) {  // S_j = Q K_j^T into TMEM columns [128 (j&1), +128)
        const int ks = j % NS;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fence_after();
        const uint32_t qa = base + S::kQ, ka = base + S::kK + ks * S::kTile;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kRows * 128) + (k & 3) * 32;
          mma(tmem + (j & 1) * 128, sdesc(qa + off, 16), sdesc(ka + off, 16), id_s, k > 0);
        }
        commit(B(kSFull + (j & 1)));  // S_j ready (also: every earlier PV has retired)
        commit(B(kKEmpty + ks));      // K stage free
      };
      auto issue_pv = [&](int j) {  // O += P_j V_j, P_j bf16 in TMEM (aliasing S_j's columns)
        const int vs = j % NS;
        fence_after();
        const uint32_t pa = tmem + (j & 1) * 128, va = base + S::kV + vs * S::kTile;
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k)  // 16 keys = 8 packed bf16x2 TMEM columns
          mma_ts(tO, pa + k * 8, sdesc(va + k * 16 * 128, kRows * 128), id_pv, (j | k) != 0);
        commit(B(kVEmpty + vs));  // V stage free
        commit(B(kPvDone));       // O updated through tile j
      };
      // In-order issue with blocking (HW-suspending) waits: S_{j+1} first (its K
      // tile is prefetched NS tiles ahead, so it is normally already there),
      // then PV_j once softmax has written P_j. S_{j+2} (same TMEM columns as
      // P_j) is issued after PV_j, and tcgen05 MMAs of one thread run in order.
      for (int j = 0; j < n_kt; ++j) {
        if (j == 0) {
          mbar_wait(B(kKFull), 0);
          TRACE(0, 0);
          issue_s(0);
        }
        if (j + 1 < n_kt) {
          mbar_wait(B(kKFull + (j + 1) % NS), ((j + 1) / NS) & 1);
          mbar_wait(B(kSEmpty + ((j + 1) & 1)), (((j + 1) >> 1) & 1) ^ 1);
          TRACE(0, j + 1);
          issue_s(j + 1);
        }
        mbar_wait(B(kPFull + (j & 1)), (j >> 1) & 1);
        mbar_wait(B(kVFull + j % NS), (j / NS) & 1);
        TRACE(1, j);
        issue_pv(j);
      }
    }
    __syncwarp();  // reconverge before the CTA-wide (aligned) barrier below
  } else {
    // ===================== softmax / correction (warps 0-7) =====================
    constexpr int HK = kKeys / 2;  // key columns per half
    const int qd = warp & 3, hf = warp >> 2;
    const int r = qd * 32 + lane;  // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int qpos = pos0 + q0 + r;
    float* xch = reinterpret_cast<float*>(gbase + S::kX);  // [half][row]
    // the two warps of a row quarter meet on named barrier 1 + qd (64 threads)
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;\n" ::"r"(1 + qd) : "memory"); };
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int st = j & 1;
      mbar_wait(B(kSFull + st), (j >> 1) & 1);
      if (threadIdx.x == 0) TRACE(2, j);
      fence_after();
      const uint32_t ts = tmem + lane_off + st * 128 + hf * HK;
      const int key0 = j * kKeys + hf * HK;
      const bool diag = j * kKeys + kKeys - 1 > pos0 + q0 || j * kKeys + kKeys > n_keys;
      uint32_t v[HK];
      TLD32(ts + 0, (v + 0));
      TLD32(ts + 32, (v + 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      fence_before();
      mbar_arrive(B(kSEmpty + st));  // S[st] read: S_{j+2} may be issued (it runs after PV_j)
      // row max over raw scores (scale > 0 commutes with max), 8 independent chains
      float m8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = -INFINITY;
      if (diag) {
#pragma unroll
        for (int i = 0; i < HK; ++i) {
          const int key = key0 + i;
          if (key > qpos || key >= n_keys) v[i] = __float_as_uint(-INFINITY);
          m8[i & 7] = fmaxf(m8[i & 7], __uint_as_float(v[i]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < HK; ++i) m8[i & 7] = fmaxf(m8[i & 7], __uint_as_float(v[i]));
      }
      const float mh = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                             fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      xch[hf * kRows + r] = mh;
      pair_sync();
      const float mx = fmaxf(mh, xch[(hf ^ 1) * kRows + r]) * scale_log2;
      pair_sync();  // both halves read before either overwrites its slot next tile
      // lazy rescale: move the reference max only when it grows by > 8 (log2);
      // both halves see the same mx, so they agree on m_used and alpha
      float alpha = 1.f;
      if (mx > m_used + 8.f) {
        alpha = m_used == -INFINITY ? 0.f : fast_exp2(m_used - mx);
        m_used = mx;
      }
      const float mref = m_used == -INFINITY ? 0.f : m_used;
      // P_j (bf16 pairs) overwrites this half's 32 TMEM columns of S_j's
      // buffer: both halves have loaded S_j (the max exchange above), and
      // PV_{j-2}, the last reader of these columns, retired before S_j landed.
      float s8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) s8[i] = 0.f;
      uint32_t pk[HK / 2];
#pragma unroll
      for (int i = 0; i < HK; i += 2) {
        // exp2(s * scale - mref): one FFMA + one MUFU; masked keys give exp2(-inf) = 0
        const float p0 = fast_exp2(fmaf(__uint_as_float(v[i]), scale_log2, -mref));
        const float p1 = fast_exp2(fmaf(__uint_as_float(v[i + 1]), scale_log2, -mref));
        s8[i & 7] += p0;
        s8[(i + 1) & 7] += p1;
        pk[i / 2] = pack_bf16x2(p0, p1);
      }
      TST32(tmem + lane_off + st * 128 + hf * (HK / 2), pk);
      l = l * alpha + (((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7])));
      // Wait for PV_{j-1} every iteration (keeps this waiter at most one phase
      // behind pv_done, so parity waits stay unambiguous), then rescale this
      // half's O columns if the reference max moved: O holds P_0..P_{j-1} V.
      if (j > 0) {
        mbar_wait(B(kPvDone), (j - 1) & 1);
        fence_after();
      }
      // tcgen05.ld/st are warp-collective (.sync.aligned): rescale when ANY lane
      // of the warp needs it (the others multiply by 1)
      if (__any_sync(0xffffffffu, alpha != 1.f) && j > 0) {
#pragma unroll 1
        for (int c = 0; c < HD / 64; ++c) {
          uint32_t o[32];
          const uint32_t to = tmem + lane_off + 256 + hf * (HD / 2) + c * 32;
          TLD32(to, o);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          TST32(to, o);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");  // P (and any O rescale) in TMEM
      fence_before();
      mbar_arrive(B(kPFull + st));
      if (threadIdx.x == 0) TRACE(3, j);
    }
    // epilogue: O / (l_0 + l_1) -> bf16, each half writes its HD/2 columns
    xch[hf * kRows + r] = l;
    pair_sync();
    const float lt = l + xch[(hf ^ 1) * kRows + r];
    mbar_wait(B(kPvDone), (n_kt - 1) & 1);
    fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const int grow = q0 + r;
#pragma unroll 1
    for (int c = 0; c < HD / 64; ++c) {
      uint32_t o[32];
      TLD32(tmem + lane_off + 256 + hf * (HD / 2) + c * 32, o);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (grow < rows && hf * (HD / 2) + c * 32 < hd) {
        uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)grow * heads * hd + h * hd + hf * (HD / 2) + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
#ifdef WS_ATTN_TRACE
  if (threadIdx.x == 0 && cta_id < 4096) g_attn_cta[cta_id][1] = attn_gtimer();
#endif
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- packed fp32 helpers (sm_100 FFMA2 / FADD2 / 3-input FMNMX) and a
// polynomial exp2 on the FMA pipe: a share of the softmax exponentials skip
// the MUFU unit, which is the softmax's throughput limit (FA4's trick).
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for a pair: x = n + f, n = round(x), f in [-0.5, 0.5]; 2^f by a cubic
// (max rel. error 7.7e-5, far below bf16's 3.9e-3 for P); 2^n added to the
// exponent field. x is clamped at -125 (2^-125 ~ 0 next to the row sum >= 1).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  const float2 xf = up2(x);
  const uint64_t xm = pk2(fmaxf(xf.x, -125.f), fmaxf(xf.y, -125.f));
  const uint64_t t = fadd2(xm, pk2(12582912.f, 12582912.f));  // 1.5 * 2^23: rounds to an integer
  const uint64_t n = fadd2(t, pk2(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(n, pk2(-1.f, -1.f), xm);
  uint64_t p = ffma2(f, pk2(0.05508868f, 0.05508868f), pk2(0.24260405f, 0.24260405f));
  p = ffma2(p, f, pk2(0.69327624f, 0.69327624f));
  p = ffma2(p, f, pk2(0.99992894f, 0.99992894f));
  const float2 tf = up2(t), pf = up2(p);
  return pk2(__uint_as_float(__float_as_uint(pf.x) + (__float_as_uint(tf.x) << 23)),
             __uint_as_float(__float_as_uint(pf.y) + (__float_as_uint(tf.y) << 23)));
}

// ---------------------------------------------------------------------------
// Persistent attention, two q heads of one GQA group per work item (even
// group sizes, TMA page gathers). An item = the same 128 query positions of
// heads h0 and h0 + 1 (tiles A and B), so every K_j / V_j tile gathered from
// the pool feeds 256 query rows. Items run heaviest first (latest query tile)
// and are dealt to the resident CTAs in a snake order (round r: CTA c takes
// item r*G + c, or r*G + G-1-c on odd rounds), which balances the causal
// triangle like LPT without atomics. Across items nothing drains: the K/V
// rings keep streaming, the next item's Q is loaded as soon as the last QK^T
// of the current one retired, and its first QK^T runs while the softmax warps
// still store the previous output.
// TMEM: S_A [0,128) S_B [128,256) O_A [256, 256+HD) O_B [256+HD, 256+2HD);
// P_X (bf16) overwrites S_X in place and PV reads it from TMEM. The MMA warp
// ping-pongs the tiles — PV_A(j), S_A(j+1), PV_B(j), S_B(j+1) — so the exp2
// stream of one tile runs under the tensor work of the other.
// Softmax warps first (tile A then B; thread = query row; with the column
// split two warps per 32 rows, 64 key columns each), then one warp each for
// TMEM alloc + MMA issue, the K gather, the V gather and the Q loads.
namespace pair2 {
#ifndef WS_ATTN_POLY
#define WS_ATTN_POLY 3
#endif
// 3/8 on the polynomial. A/B at 8B / 2048 tokens (tools/ab_attn_poly.sh):
// 0-6 of 8 -> 46.5 / 46.5 / 45.0 / 46.9 / 48.1 / 49.4 / 51.2 us. 2/8 is 0.25%
// of a prefill faster but rounds P differently enough to flip the greedy
// token of the full-depth parity prompt that sits at a bf16 near-tie (fp32
// margin 0.045; the bf16-floor emulation flips it too), so 3/8 stays.
constexpr int kPolyPairs = WS_ATTN_POLY;
#ifndef WS_ATTN_SPLIT
#define WS_ATTN_SPLIT 0
#endif
// Column split (off by default; A/B variant): two softmax warps per (tile,
// 32-row quarter), each over 64 of the 128 key columns — 16 softmax warps, 4
// per SM sub-partition, row maxima exchanged through shared memory. Measured
// 45.7 vs 45.0 us at 8B / 2048 tokens: the per-tile softmax drops from ~2200
// to ~1850 clocks but the exchange and the busier MUFU pipe eat the gain
// (prefill attention).
constexpr int kHalves = WS_ATTN_SPLIT ? 2 : 1;
constexpr int kCols = kKeys / kHalves;
constexpr int kSoftWarps = 8 * kHalves;
constexpr int kMmaWarp = kSoftWarps, kKWarp = kSoftWarps + 1, kVWarp = kSoftWarps + 2, kQWarp = kSoftWarps + 3;
constexpr int kThreads2 = (kSoftWarps + 4) * 32;
constexpr int NSK = kHalves == 2 ? 2 : 3, NSV = 2;  // K tiles are needed a full softmax earlier than V tiles
template <int HD>
struct Smem {
  static constexpr int kTile = kRows * HD * 2;
  static constexpr int kQ = 0;                      // Q_A, Q_B
  static constexpr int kK = kQ + 2 * kTile;         // NSK stages
  static constexpr int kV = kK + NSK * kTile;       // NSV stages
  static constexpr int kBar = kV + NSV * kTile;
  static constexpr int kX = kBar + 256;             // column split: row max / row sum exchange
  static constexpr int kBytes = kX + (kHalves == 2 ? (2 * 2 * 2 + 2 * 2) * kRows * 4 : 0) + 1024;
};
constexpr int kQFull = 0, kQEmpty = 2, kKFull = 4, kKEmpty = kKFull + NSK, kVFull = kKEmpty + NSK,
              kVEmpty = kVFull + NSV, kSFull = kVEmpty + NSV, kPFull = kSFull + 2, kPvDone = kPFull + 2,
              kOFree = kPvDone + 2, kTmemSlot = kOFree + 2;

struct Item {
  int qt, h0, q0, n_keys, n_kt;
};
__device__ __forceinline__ bool item_of(int r, int c, int G, int n_items, int n_hp, int n_qt, int rows, int pos0,
                                        Item& it) {
  const int i = r * G + ((r & 1) ? G - 1 - c : c);
  if (i >= n_items) return false;
  it.qt = n_qt - 1 - i / n_hp;
  it.h0 = 2 * (i % n_hp);
  it.q0 = it.qt * kRows;
  it.n_keys = pos0 + min(rows, it.q0 + kRows);
  it.n_kt = (it.n_keys + kKeys - 1) / kKeys;
  return true;
}
}  // namespace pair2

template <int HD>
__global__ void __launch_bounds__(pair2::kThreads2, 1)
    attn_tc2_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ out, KvGeom kv, int layer, int seq, int rows,
                    int pos0, int heads, float scale_log2, const __grid_constant__ CUtensorMap kvmap) {
  using namespace pair2;
  using S = pair2::Smem<HD>;
  constexpr int CH = HD / 8;
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar = base + S::kBar;
  auto B = [&](int i) { return bar + 8 * i; };
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + S::kBar + pair2::kTmemSlot * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (rows + kRows - 1) / kRows, n_hp = heads / 2, n_items = n_qt * n_hp;
  const int G = gridDim.x, c = blockIdx.x;
  const int group = heads / kv.kv_heads;
  const int ldq = (heads + 2 * kv.kv_heads) * HD;

  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(B(pair2::kQFull + x), 32);
      mbar_init(B(pair2::kQEmpty + x), 1);
    }
    for (int i = 0; i < NSK; ++i) {
      mbar_init(B(pair2::kKFull + i), 1);
      mbar_init(B(pair2::kKEmpty + i), 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(B(pair2::kVFull + i), 1);
      mbar_init(B(pair2::kVEmpty + i), 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(B(pair2::kSFull + x), 1);
      mbar_init(B(pair2::kPFull + x), 128 * kHalves);
      mbar_init(B(pair2::kPvDone + x), 1);
      mbar_init(B(pair2::kOFree + x), 128 * kHalves);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // K/V rows a tile does not load keep stale (finite) data; start from zeros
  for (int i = threadIdx.x; i < (NSK + NSV) * S::kTile / 16; i += pair2::kThreads2)
    reinterpret_cast<uint4*>(gbase + S::kK)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(B(pair2::kTmemSlot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) TRACE(0, 0);  // CTA start (after the PDL wait)

  Item it;
  if (warp == kQWarp) {
    // ===================== Q loads (one warp) =====================
    for (int r = 0; item_of(r, c, G, n_items, n_hp, n_qt, rows, pos0, it); ++r) {
      for (int x = 0; x < 2; ++x) {
        // Q_x is free once the previous item's last QK^T on tile x retired
        if (r > 0) mbar_wait(B(pair2::kQEmpty + x), (r - 1) & 1);
        for (int i = lane; i < kRows * CH; i += 32) {
          const int rr = i / CH, cc = i % CH;
          const int gr = it.q0 + rr;
          const bf16* src = qkv + (int64_t)(gr < rows ? gr : 0) * ldq + (it.h0 + x) * HD + cc * 8;
          cp_async16(gbase + S::kQ + x * S::kTile + swz(rr, cc), src, gr < rows);
        }
        cp_async_arrive(B(pair2::kQFull + x));
      }
    }
  } else if (warp == kKWarp || warp == kVWarp) {
    // ===================== K / V page gathers (one warp each) =====================
    const bool is_v = warp == kVWarp;
    const int32_t* bt = kv.block_tables + (int64_t)seq * kv.max_blocks;
    const uint32_t ring = is_v ? S::kV : S::kK;
    const int full0 = is_v ? pair2::kVFull : pair2::kKFull, empty0 = is_v ? pair2::kVEmpty : pair2::kKEmpty;
    const int rows_pp = (int)(kv.page_size / (HD * 2));
    const int ns = is_v ? NSV : NSK;
    int g = 0;  // tiles issued so far (ring position)
    for (int r = 0; item_of(r, c, G, n_items, n_hp, n_qt, rows, pos0, it); ++r) {
      const int plane_rows = (int)(kv.plane(layer, is_v ? 1 : 0, it.h0 / group) / HD);
      auto row_of = [&](int j) {  // lane u: page row of key group u (16 tokens) of tile j
        const int key0 = j * kKeys + (lane & 7) * 16;
        const int blk = key0 / kv.tpb, slot = key0 - blk * kv.tpb;
        return key0 < it.n_keys ? bt[blk] * rows_pp + plane_rows + slot : 0;
      };
      int y_next = row_of(0);
      for (int j = 0; j < it.n_kt; ++j, ++g) {
        const int st = g % ns;
        const int y = y_next;
        if (j + 1 < it.n_kt) y_next = row_of(j + 1);
        const int groups = min(kKeys / 16, (it.n_keys - j * kKeys + 15) / 16);
        if (lane == 0) {
          mbar_wait(B(empty0 + st), ((g / ns) & 1) ^ 1);
          tma_expect(B(full0 + st), (uint32_t)(groups * (HD / 64) * 2048));
        }
        for (int gg = 0; gg < groups; ++gg) {
          const int yg = __shfl_sync(0xffffffffu, y, gg);
          if (lane == 0) {
#pragma unroll
            for (int hh = 0; hh < HD / 64; ++hh)
              tma_load_2d(base + ring + st * S::kTile + hh * (kRows * 128) + gg * 2048, &kvmap, B(full0 + st),
                          hh * 64, yg);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(kKeys, false), id_pv = idesc(HD, true);
      auto issue_s = [&](int x, int kt) {  // S_x = Q_x K^T (K ring tile kt)
        fence_after();
        const uint32_t qa = base + S::kQ + x * S::kTile, ka = base + S::kK + (kt % NSK) * S::kTile;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kRows * 128) + (k & 3) * 32;
          mma(tmem + x * 128, sdesc(qa + off, 16), sdesc(ka + off, 16), id_s, k > 0);
        }
        commit(B(pair2::kSFull + x));
      };
      auto issue_pv = [&](int x, int kt, bool first) {  // O_x += P_x V (P_x bf16 in S_x's TMEM columns)
        fence_after();
        const uint32_t pa = tmem + x * 128, va = base + S::kV + (kt % NSV) * S::kTile;
        const uint32_t to = tmem + 256 + x * HD;
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k)
          mma_ts(to, pa + k * 8, sdesc(va + k * 16 * 128, kRows * 128), id_pv, (!first || k != 0) ? 1u : 0u);
        commit(B(pair2::kPvDone + x));
      };
      int g = 0;  // global tile counter (ring position and per-step barrier parity)
      for (int r = 0; item_of(r, c, G, n_items, n_hp, n_qt, rows, pos0, it); ++r) {
        const bool single = it.n_kt == 1;
        mbar_wait(B(pair2::kKFull + g % NSK), (g / NSK) & 1);
        if (r == 0) TRACE(2, 63);
        // S_X(0) may overwrite the previous item's P_X: its PV was issued earlier (in-order pipe)
        mbar_wait(B(pair2::kQFull + 0), r & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue_s(0, g);
        if (single) commit(B(pair2::kQEmpty + 0));
        mbar_wait(B(pair2::kQFull + 1), r & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue_s(1, g);
        if (single) commit(B(pair2::kQEmpty + 1));
        commit(B(pair2::kKEmpty + g % NSK));
        for (int j = 0; j < it.n_kt; ++j, ++g) {
          const bool more = j + 1 < it.n_kt;
          mbar_wait(B(pair2::kVFull + g % NSV), (g / NSV) & 1);
          mbar_wait(B(pair2::kPFull + 0), g & 1);
          if (j == 0 && r > 0) mbar_wait(B(pair2::kOFree + 0), (r - 1) & 1);  // previous O_A read out
          if (r == 0) TRACE(1, j);
          issue_pv(0, g, j == 0);
          if (more) {
            mbar_wait(B(pair2::kKFull + (g + 1) % NSK), ((g + 1) / NSK) & 1);
            if (r == 0) TRACE(0, j + 1);
            issue_s(0, g + 1);  // after PV_A(j) in the same in-order pipe: P_A(j) is read first
            if (j + 2 == it.n_kt) commit(B(pair2::kQEmpty + 0));  // last QK^T of tile A: Q_A free
          }
          mbar_wait(B(pair2::kPFull + 1), g & 1);
          if (j == 0 && r > 0) mbar_wait(B(pair2::kOFree + 1), (r - 1) & 1);
          issue_pv(1, g, j == 0);
          commit(B(pair2::kVEmpty + g % NSV));
          if (more) {
            issue_s(1, g + 1);
            if (j + 2 == it.n_kt) commit(B(pair2::kQEmpty + 1));
            commit(B(pair2::kKEmpty + (g + 1) % NSK));
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kSoftWarps) {
    // ===================== softmax =====================
    // warp = (tile x, column half hf, row quarter qd): thread = query row
    // qd*32 + lane of tile x, over kCols of the 128 key columns. With the
    // column split the two warps of a (tile, quarter) exchange their row
    // maxima through shared memory (named barrier per pair, parity double-
    // buffered slots) so they agree on the reference max and the rescale.
    const int x = warp / (4 * kHalves), hf = (warp >> 2) % kHalves, qd = warp & 3;
    const int rl = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t tS = tmem + lane_off + x * 128, tO = tmem + lane_off + 256 + x * HD + hf * (HD / kHalves);
    float* xmax = reinterpret_cast<float*>(gbase + S::kX);  // [parity][tile][half][row]
    float* xsum = xmax + 2 * 2 * kHalves * kRows;          // [tile][half][row]
    const uint32_t nb = 1 + x * 4 + qd;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;\n" ::"r"(nb) : "memory"); };
    int g = 0;
    for (int r = 0; item_of(r, c, G, n_items, n_hp, n_qt, rows, pos0, it); ++r) {
      const int qpos = pos0 + it.q0 + rl;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < it.n_kt; ++j, ++g) {
        mbar_wait(B(pair2::kSFull + x), g & 1);
        if (threadIdx.x == 0 && r == 0) TRACE(2, j);
        fence_after();
        const int key0 = j * kKeys + hf * kCols;  // this thread's first key column
        const bool diag = j * kKeys + kKeys - 1 > pos0 + it.q0 || j * kKeys + kKeys > it.n_keys;
        uint32_t v[kCols];
#pragma unroll
        for (int cc = 0; cc < kCols / 32; ++cc) TLD32(tS + hf * kCols + cc * 32, (v + cc * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (threadIdx.x == 0 && r == 0) TRACE(4, j);
        if (diag) {
#pragma unroll
          for (int i = 0; i < kCols; ++i)
            if (key0 + i > qpos || key0 + i >= it.n_keys) v[i] = __float_as_uint(-INFINITY);
        }
        // row max over raw scores (scale > 0 commutes with max): 3-input max, 4 chains
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
        for (int i = 0; i < kCols; i += 8) {
          m0 = fmax3(m0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          m1 = fmax3(m1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
          m2 = fmax3(m2, __uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
          m3 = fmax3(m3, __uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
        }
        float mraw = fmax3(m0, m1, fmaxf(m2, m3));
        if constexpr (kHalves == 2) {
          // both halves have loaded S_j (tcgen05.wait::ld above) once they meet
          // here, so P may overwrite S_j's columns afterwards
          float* slot = xmax + ((g & 1) * 2 + x) * 2 * kRows;
          slot[hf * kRows + rl] = mraw;
          pair_sync();
          mraw = fmaxf(mraw, slot[(hf ^ 1) * kRows + rl]);
        }
        const float mx = mraw * scale_log2;
        float alpha = 1.f;
        if (mx > m_used + 8.f) {  // lazy rescale (exact: O/l share the reference max)
          alpha = m_used == -INFINITY ? 0.f : fast_exp2(m_used - mx);
          m_used = mx;
        }
        const float mref = m_used == -INFINITY ? 0.f : m_used;
        if (threadIdx.x == 0 && r == 0) TRACE(5, j);
        // p = exp2(s * scale - mref) two at a time (FFMA2); kPolyPairs of every 8
        // pairs on the FMA-pipe polynomial, the rest on MUFU; P packed in place
        const uint64_t sc2 = pk2(scale_log2, scale_log2), nm2 = pk2(-mref, -mref);
        uint64_t s2[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) s2[i] = 0;
#pragma unroll
        for (int q = 0; q < kCols / 2; ++q) {
          const uint64_t x2 = ffma2(pk2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1])), sc2, nm2);
          uint64_t p2;
          if ((q & 7) < kPolyPairs) {
            p2 = exp2_poly2(x2);
          } else {
            const float2 xf = up2(x2);
            p2 = pk2(fast_exp2(xf.x), fast_exp2(xf.y));
          }
          s2[q & 3] = fadd2(s2[q & 3], p2);
          const float2 pf = up2(p2);
          v[q] = pack_bf16x2(pf.x, pf.y);
        }
        const float2 sa = up2(fadd2(fadd2(s2[0], s2[1]), fadd2(s2[2], s2[3])));
        l = l * alpha + (sa.x + sa.y);
        if (threadIdx.x == 0 && r == 0) TRACE(6, j);
        // P_j (bf16 pairs) overwrites the first half of S_j's columns: keys
        // [hf*kCols, +kCols) -> packed columns [hf*kCols/2, +kCols/2)
#pragma unroll
        for (int cc = 0; cc < kCols / 64; ++cc) TST32(tS + hf * (kCols / 2) + cc * 32, (v + cc * 32));
        if (j > 0) {  // O_x holds P_0..P_{j-1} V once PV_x(j-1) retired
          mbar_wait(B(pair2::kPvDone + x), (g - 1) & 1);
          fence_after();
        }
        if (threadIdx.x == 0 && r == 0) TRACE(7, j);
        if (__any_sync(0xffffffffu, alpha != 1.f) && j > 0) {  // this warp's O columns
#pragma unroll 1
          for (int cc = 0; cc < HD / kHalves / 32; ++cc) {
            uint32_t o[32];
            TLD32(tO + cc * 32, o);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            TST32(tO + cc * 32, o);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        fence_before();
        mbar_arrive(B(pair2::kPFull + x));
        if (threadIdx.x == 0 && r == 0) TRACE(3, j);
      }
      // epilogue: O_x / l -> bf16 rows of head h0 + x (this warp's columns);
      // O_x is released as soon as it is in registers
      float lt = l;
      if constexpr (kHalves == 2) {
        xsum[(x * 2 + hf) * kRows + rl] = l;
        pair_sync();
        lt += xsum[(x * 2 + (hf ^ 1)) * kRows + rl];
      }
      mbar_wait(B(pair2::kPvDone + x), (g - 1) & 1);
      fence_after();
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      constexpr int OC = HD / kHalves;
      uint32_t o[OC];
#pragma unroll
      for (int cc = 0; cc < OC / 32; ++cc) TLD32(tO + cc * 32, (o + cc * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      fence_before();
      mbar_arrive(B(pair2::kOFree + x));
      const int grow = it.q0 + rl;
      if (grow < rows) {
        uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)grow * heads * HD + (it.h0 + x) * HD + hf * OC);
#pragma unroll
        for (int q = 0; q < OC / 8; ++q)
          dst[q] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
                              pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) TRACE(1, 63);  // CTA done
#ifdef WS_ATTN_TRACE
  if (threadIdx.x == 0 && c < 4096) {
    g_attn_cta[c][1] = attn_gtimer();
  }
#endif
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// 2D view of the page window as rows of HD bf16 (one token of one K or V
// plane per row), 8-row x 64-column boxes with 128B swizzle.
bool window_map(CUtensorMap* map, const KvGeom& kv, int hd) {
  const Driver* d = driver();
  if (!d) return false;
  cuuint64_t dims[2] = {(cuuint64_t)hd, (cuuint64_t)(kv.n_pages * kv.page_size / (hd * 2))};
  cuuint64_t strides[1] = {(cuuint64_t)hd * 2};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t estr[2] = {1, 1};
  return d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.window, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


template <int HD, bool TMA>
void launch_impl(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows, int pos0,
                 int heads, float scale, const CUtensorMap& map, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<HD, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<HD>::kBytes);
    attr = true;
  }
  dim3 grid(heads, (rows + kRows - 1) / kRows);
  count_launch();
  launch_pdl(attn_tc_kernel<HD, TMA>, dim3(grid), dim3(kThreads), Smem<HD>::kBytes, st, qkv, out, kv, layer, seq, rows, pos0, heads,
                                                                    scale * 1.4426950408889634f, map);
}

template <int HD>
void dispatch(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows, int pos0, int heads,
              float scale, cudaStream_t st) {
  // TMA needs 8-token runs inside a block and the window addressable as HD-wide rows
  static CUtensorMap map;
  static const char* map_window = nullptr;
  static int64_t map_pages = 0;
  bool tma = kv.head_dim == HD && kv.tpb % 16 == 0 && kv.page_size % (HD * 2) == 0;
  if (tma && (map_window != kv.window || map_pages != kv.n_pages)) {
    tma = window_map(&map, kv, HD);
    map_window = tma ? kv.window : nullptr;
    map_pages = tma ? kv.n_pages : 0;
  }
  static const bool pair_heads = !(getenv("WS_ATTN_PAIR") && getenv("WS_ATTN_PAIR")[0] == '0');
  if (tma && pair_heads && (heads / kv.kv_heads) % 2 == 0) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(attn_tc2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           pair2::Smem<HD>::kBytes);
      attr = true;
    }
    count_launch();
    const int items = (heads / 2) * ((rows + kRows - 1) / kRows);
    launch_pdl(attn_tc2_kernel<HD>, dim3(items < kNumSMs ? items : kNumSMs), dim3(pair2::kThreads2),
               pair2::Smem<HD>::kBytes, st, qkv, out, kv, layer, seq, rows, pos0, heads, scale * 1.4426950408889634f,
               map);
  } else if (tma)
    launch_impl<HD, true>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, map, st);
  else
    launch_impl<HD, false>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, map, st);
}

}  // namespace

// The page window as a TMA tensor (rows of hd bf16, 64 x 16 boxes, 128B
// swizzle), cached per (window, extent, hd): shared with the decode kernel.
bool kv_window_tmap(const KvGeom& kv, int hd, CUtensorMap* out) {
  struct Entry {
    const char* window;
    int64_t pages;
    int hd;
    bool ok;
    CUtensorMap map;
  };
  static Entry cache[4];
  static int next = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (const Entry& e : cache)
    if (e.window == kv.window && e.pages == kv.n_pages && e.hd == hd) {
      *out = e.map;
      return e.ok;
    }
  Entry& e = cache[next];
  next = (next + 1) % 4;
  e.window = kv.window;
  e.pages = kv.n_pages;
  e.hd = hd;
  e.ok = hd % 64 == 0 && kv.page_size % (hd * 2) == 0 && window_map(&e.map, kv, hd);
  *out = e.map;
  return e.ok;
}

#ifdef WS_ATTN_TRACE
extern "C" int ws_attn_trace(long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace)) == cudaSuccess ? 0 : 6;
}
extern "C" int ws_attn_cta_trace(long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_attn_cta, sizeof(g_attn_cta)) == cudaSuccess ? 0 : 6;
}
#endif

bool attn_prefill_tc_paired(const KvGeom& kv, int heads) {
  static const bool pair_heads = !(getenv("WS_ATTN_PAIR") && getenv("WS_ATTN_PAIR")[0] == '0');
  const int hd = kv.head_dim;
  return (hd == 128 || hd == 64) && kv.tpb % 16 == 0 && kv.page_size % (hd * 2) == 0 && pair_heads &&
         (heads / kv.kv_heads) % 2 == 0;
}

// Warm prefill, same box, whole prompt, ms, tcgen05 -> mma.sync attention:
// Llama-3-8B 64 / 128 / 256 / 384 tokens 4.48 / 5.17 / 7.18 / 8.24 -> 4.35 /
// 4.89 / 7.02 / 8.26 (paired heads); Phi-3-mini 64 / 128: 3.63 / 4.34 ->
// 3.49 / 4.34 (head_dim 96, one head per CTA), Qwen2.5-7B 64 / 256: 4.17 /
// 6.52 -> 4.11 / 6.50 (odd group). WS_ATTN_SHORT_MMA=0 keeps the tcgen05
// kernels for every length.
bool attn_prefill_prefers_mma(const KvGeom& kv, int rows, int heads) {
  static const bool on = !(getenv("WS_ATTN_SHORT_MMA") && getenv("WS_ATTN_SHORT_MMA")[0] == '0');
  return on && rows <= (attn_prefill_tc_paired(kv, heads) ? 256 : 64);
}

bool launch_attn_prefill_tc(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                            int pos0, int heads, float scale, cudaStream_t st) {
  if (kv.head_dim == 128 || kv.head_dim == 96)  // 96 runs in zero-padded 128-wide tiles
    dispatch<128>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st);
  else if (kv.head_dim == 64)
    dispatch<64>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st);
  else
    return false;
  return true;
}

}  // namespace ws

// tcgen05 flash-attention prefill over the paged KV pool (sm_100a).
//
// One CTA = 128 queries of one q head (GQA: its kv head = h / group), K/V
// tiles of 128 keys gathered page by page. Warp roles (288 threads):
//   warps 0-3  softmax + correction: thread r owns query row r (TMEM lane r).
//              Reads S_j from TMEM in 32-column chunks (two passes: row max,
//              then exp2/sum), writes P_j as bf16 into SMEM (K-major SW128),
//              rescales the TMEM output accumulator only when the running max
//              grows by more than 2^8 (exact: final O/l uses the same max).
//   warps 4-7  producers: cp.async gather of Q (once) and K_j/V_j rows from
//              the block table into SWIZZLE_128B smem tiles; completion via
//              cp.async.mbarrier.arrive.noinc.
//   warp 8     TMEM allocator + single-thread MMA issuer:
//              S_j = Q K_j^T   (M=128, N=128, K=hd; both operands K-major)
//              O  += P_j V_j   (M=128, N=hd, K=128; V is MN-major — no transpose)
//              S is double-buffered in TMEM so QK^T of tile j+1 overlaps the
//              softmax of tile j. TMEM: S0 [0,128) S1 [128,256) O [256,256+hd).
#include <cuda.h>

#include "../common.h"
#include "../driver.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {
namespace {

using namespace dev;

constexpr int kRows = 128, kKeys = 128, kThreads = 288;

#ifdef WS_ATTN_TRACE
// debug timeline of block (0,0): [event][j] = clock64 (events: 0 S issued,
// 1 PV issued, 2 softmax got S, 3 softmax released P)
__device__ long long g_attn_trace[4][64];
#define TRACE(ev, j) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 64) g_attn_trace[ev][j] = clock64(); } while (0)
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

template <int HD>
struct Smem {
  static constexpr int kTile = kRows * HD * 2;     // Q, K or V tile: [HD/64 blocks][128 rows][128 B]
  static constexpr int kP = kRows * kKeys * 2;     // P tile: [2 blocks][128 rows][128 B]
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;            // 2 stages
  static constexpr int kV = kK + 2 * kTile;        // 2 stages
  static constexpr int kPo = kV + 2 * kTile;       // 2 buffers
  static constexpr int kBar = kPo + 2 * kP;
  static constexpr int kBytes = kBar + 256 + 1024;  // barriers + alignment slack
};

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
  // barriers: 0 q_full | 1,2 k_full | 3,4 k_empty | 5,6 v_full | 7,8 v_empty | 9,10 s_full |
  //           11,12 s_empty | 13,14 p_full | 15,16 p_empty | 17 pv_done | TMEM base slot at +18*8
  // K_j is released right after S_j (QK^T) retires, V_j after PV_j, so the
  // gather of K_{j+2} overlaps the softmax of tile j.
  auto B = [&](int i) { return bar + 8 * i; };
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + S::kBar + 18 * 8);

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
  const int ldq = (heads + 2 * kv.kv_heads) * HD;

  if (threadIdx.x == 0) {
    mbar_init(B(0), 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(B(1 + i), TMA ? 1 : 64);  // k_full: TMA thread (expect_tx) or 64 cp.async threads
      mbar_init(B(3 + i), 1);     // k_empty: MMA commit after S_j
      mbar_init(B(5 + i), TMA ? 1 : 64);  // v_full
      mbar_init(B(7 + i), 1);     // v_empty: MMA commit after PV_j
      mbar_init(B(9 + i), 1);     // s_full: MMA commit
      mbar_init(B(11 + i), 128);  // s_empty: softmax threads
      mbar_init(B(13 + i), 128);  // p_full: softmax threads
      mbar_init(B(15 + i), 1);    // p_empty: MMA commit
    }
    mbar_init(B(17), 1);  // pv_done: MMA commit
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if constexpr (TMA) {
    // K/V rows a tile does not load keep stale data; start from finite zeros
    for (int i = threadIdx.x; i < 4 * S::kTile / 16; i += kThreads)
      reinterpret_cast<uint4*>(gbase + S::kK)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(bar + 18 * 8));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // everything above is prologue; global data from here on

  if (warp >= 4 && warp < 8) {
    // ===================== producers: warps 4-5 gather K, warps 6-7 gather V =====================
    const int t = threadIdx.x - 128;
    for (int i = t; i < kRows * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const int gr = q0 + r;
      const bf16* src = qkv + (int64_t)(gr < rows ? gr : 0) * ldq + h * HD + c * 8;
      cp_async16(gbase + S::kQ + swz(r, c), src, gr < rows);
    }
    cp_async_arrive(B(0));
    const bool is_v = t >= 64;
    const int u = t & 63;  // rows u and u + 64 of every tile
    const int32_t* bt = kv.block_tables + (int64_t)seq * kv.max_blocks;
    const int64_t plane = kv.plane(layer, is_v ? 1 : 0, kvh);
    const uint32_t ring = is_v ? S::kV : S::kK;
    const int full0 = is_v ? 5 : 1, empty0 = is_v ? 7 : 3;
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
          const int st = j & 1;
          const int y = y_next;
          if (j + 1 < n_kt) y_next = row_of(j + 1);
          const int groups = min(kKeys / 16, (n_keys - j * kKeys + 15) / 16);
          if (u == 0) {
            mbar_wait(B(empty0 + st), ((j >> 1) & 1) ^ 1);
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
      const int st = j & 1;
      mbar_wait(B(empty0 + st), ((j >> 1) & 1) ^ 1);
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
                          (int64_t)(ok ? slot : 0) * HD;
        cp_async16(dst + swz(r, c), row + c * 8, ok);
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
      mbar_wait(B(0), 0);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      // Event-driven issue: S_{j+1} = Q K_{j+1}^T and PV_j = P_j V_j are issued
      // in whichever order their inputs become ready (non-blocking polls), so
      // a late K tile never holds back the PV of the previous tile.
      auto issue_s = [&](int j) {
        const int st = j & 1;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fence_after();
        const uint32_t qa = base + S::kQ, ka = base + S::kK + st * S::kTile;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kRows * 128) + (k & 3) * 32;
          mma(tmem + st * 128, sdesc(qa + off, 16), sdesc(ka + off, 16), id_s, k > 0);
        }
        commit(B(9 + st));  // S_j ready
        commit(B(3 + st));  // K stage free
      };
      auto issue_pv = [&](int j) {
        const int st = j & 1;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fence_after();
        const uint32_t pa = base + S::kPo + st * S::kP, va = base + S::kV + st * S::kTile;
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          const uint32_t a_off = (k >> 2) * (kRows * 128) + (k & 3) * 32;
          mma(tO, sdesc(pa + a_off, 16), sdesc(va + k * 16 * 128, kRows * 128), id_pv, (j | k) != 0);
        }
        commit(B(15 + st));  // P buffer free
        commit(B(7 + st));   // V stage free
        commit(B(17));       // O updated through tile j
      };
      // In-order issue with blocking (HW-suspending) waits: S_{j+1} first (its K
      // tile is prefetched two tiles ahead, so it is normally already there),
      // then PV_j once softmax has written P_j.
      for (int j = 0; j < n_kt; ++j) {
        if (j == 0) {
          mbar_wait(B(1), 0);
          TRACE(0, 0);
          issue_s(0);
        }
        if (j + 1 < n_kt) {
          const int s1 = (j + 1) & 1, ph1 = ((j + 1) >> 1) & 1;
          mbar_wait(B(1 + s1), ph1);
          mbar_wait(B(11 + s1), ph1 ^ 1);
          TRACE(0, j + 1);
          issue_s(j + 1);
        }
        mbar_wait(B(13 + (j & 1)), (j >> 1) & 1);
        mbar_wait(B(5 + (j & 1)), (j >> 1) & 1);
        TRACE(1, j);
        issue_pv(j);
      }
      int ns = n_kt, npv = n_kt;  // event-driven variant below disabled
      while (npv < n_kt) {
        // S_ns needs K_ns and a free S buffer (softmax already read S_{ns-2}):
        // it may run ahead of PV so the next softmax never waits on the pipe
        if (ns < n_kt && mbar_ready(B(1 + (ns & 1)), (ns >> 1) & 1) &&
            mbar_ready(B(11 + (ns & 1)), ((ns >> 1) & 1) ^ 1)) {
          TRACE(0, ns);
          issue_s(ns++);
          continue;
        }
        // PV_npv needs P_npv (softmax) and V_npv
        if (npv < ns && mbar_ready(B(13 + (npv & 1)), (npv >> 1) & 1) &&
            mbar_ready(B(5 + (npv & 1)), (npv >> 1) & 1)) {
          TRACE(1, npv);
          issue_pv(npv++);
          continue;
        }
        __nanosleep(64);  // back off: this warp shares an SMSP with a softmax warp
      }
    }
    __syncwarp();  // reconverge before the CTA-wide (aligned) barrier below
  } else {
    // ===================== softmax / correction (warps 0-3) =====================
    const int r = threadIdx.x;  // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const int qpos = pos0 + q0 + r;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int st = j & 1;
      mbar_wait(B(9 + st), (j >> 1) & 1);
      if (threadIdx.x == 0) TRACE(2, j);
      fence_after();
      const uint32_t ts = tmem + lane_off + st * 128;
      const int key0 = j * kKeys;
      const bool diag = key0 + kKeys - 1 > pos0 + q0 || key0 + kKeys > n_keys;
      // the whole 128-column row of S_j in registers: 4 loads, one wait
      uint32_t v[kKeys];
      TLD32(ts + 0, (v + 0));
      TLD32(ts + 32, (v + 32));
      TLD32(ts + 64, (v + 64));
      TLD32(ts + 96, (v + 96));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      fence_before();
      mbar_arrive(B(11 + st));  // S[st] consumed: the next QK^T may overwrite it
      float mx = -INFINITY;
      if (diag) {
#pragma unroll
        for (int i = 0; i < kKeys; ++i) {
          const int key = key0 + i;
          const float x = (key > qpos || key >= n_keys) ? -INFINITY : __uint_as_float(v[i]) * scale_log2;
          v[i] = __float_as_uint(x);
          mx = fmaxf(mx, x);
        }
      } else {
#pragma unroll
        for (int i = 0; i < kKeys; ++i) {
          const float x = __uint_as_float(v[i]) * scale_log2;
          v[i] = __float_as_uint(x);
          mx = fmaxf(mx, x);
        }
      }
      // lazy rescale: move the reference max only when it grows by > 8 (log2)
      float alpha = 1.f;
      if (mx > m_used + 8.f) {
        alpha = m_used == -INFINITY ? 0.f : fast_exp2(m_used - mx);
        m_used = mx;
      }
      const float mref = m_used == -INFINITY ? 0.f : m_used;
      // the P buffer of tile j was last read by PV_{j-2}
      if (j >= 2) mbar_wait(B(15 + st), ((j >> 1) & 1) ^ 1);
      uint8_t* prow = gbase + S::kPo + st * S::kP;
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < kKeys / 8; ++q) {  // 8 keys per 16-byte chunk
        float p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          p[i] = fast_exp2(__uint_as_float(v[8 * q + i]) - mref);  // exp2(-inf) = 0 for masked keys
          sum += p[i];
        }
        *reinterpret_cast<uint4*>(prow + swz(r, q)) =
            make_uint4(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]), pack_bf16x2(p[4], p[5]),
                       pack_bf16x2(p[6], p[7]));
      }
      l = l * alpha + sum;
      // Wait for PV_{j-1} every iteration (keeps this waiter at most one phase
      // behind pv_done, so parity waits stay unambiguous), then rescale O if
      // the reference max moved: O holds P_0..P_{j-1} V.
      if (j > 0) {
        mbar_wait(B(17), (j - 1) & 1);
        fence_after();
      }
      // tcgen05.ld/st are warp-collective (.sync.aligned): rescale when ANY lane
      // of the warp needs it (the others multiply by 1)
      if (__any_sync(0xffffffffu, alpha != 1.f) && j > 0) {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t v[32];
          TLD32(tmem + lane_off + 256 + c * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          TST32(tmem + lane_off + 256 + c * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P visible to the tensor core
      fence_before();
      mbar_arrive(B(13 + st));
      if (threadIdx.x == 0) TRACE(3, j);
    }
    // epilogue: O / l -> bf16
    mbar_wait(B(17), (n_kt - 1) & 1);
    fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int grow = q0 + r;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      TLD32(tmem + lane_off + 256 + c * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (grow < rows) {
        uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)grow * heads * HD + h * HD + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * q]) * inv, __uint_as_float(v[8 * q + 1]) * inv),
                              pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv),
                              pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv),
                              pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv));
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
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
  bool tma = kv.tpb % 16 == 0 && kv.page_size % (HD * 2) == 0;
  if (tma && (map_window != kv.window || map_pages != kv.n_pages)) {
    tma = window_map(&map, kv, HD);
    map_window = tma ? kv.window : nullptr;
    map_pages = tma ? kv.n_pages : 0;
  }
  if (tma)
    launch_impl<HD, true>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, map, st);
  else
    launch_impl<HD, false>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, map, st);
}

}  // namespace

#ifdef WS_ATTN_TRACE
extern "C" int ws_attn_trace(long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace)) == cudaSuccess ? 0 : 6;
}
#endif

bool launch_attn_prefill_tc(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                            int pos0, int heads, float scale, cudaStream_t st) {
  if (kv.head_dim == 128)
    dispatch<128>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st);
  else if (kv.head_dim == 64)
    dispatch<64>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st);
  else
    return false;
  return true;
}

}  // namespace ws

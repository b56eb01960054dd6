// sm_100a memory-switch kernel (SURVEY.md §2 "block-table rewrite /
// slot-evict kernel"): the device half of switch_memory().
//
// One launch does three things that the host ledger already decided
// (single writer, cluster.py:200-201):
//   1. bulk owner-map rules over all pages   (evict slot -> free, free -> KV…)
//   2. explicit owner writes                  (pages given to a new slot)
//   3. live-block migration + block-table rewrite for KV pages being
//      returned to the weight pool (reclaim_on_completion, cluster.py:351-365)
// Bytes are tiny except migrations (2 MiB each, HBM-bound copy); the launch is
// latency-bound, so the grid is sized to the work, not to the SM count.
#include "common.h"
#include "switch.cuh"

namespace ws {
namespace {

constexpr int kThreads = 256;
constexpr int kMigCtasPerPage = 16;  // 2 MiB / 16 = 128 KiB per CTA, 32 B per thread-iter x 16

__global__ void __launch_bounds__(kThreads) switch_kernel(SwitchArgs a, int n_rule_ctas,
                                                          int n_set_ctas) {
  const int cta = blockIdx.x;
  if (cta < n_rule_ctas) {
    if (a.rules.n == 0) return;
    const int64_t hi = a.rules.hi ? a.rules.hi : a.n_pages;
    for (int64_t p = a.rules.lo + (int64_t)cta * kThreads + threadIdx.x; p < hi;
         p += (int64_t)n_rule_ctas * kThreads) {
      int32_t o = a.owner[p];
#pragma unroll
      for (int i = 0; i < kMaxRules; ++i) {
        if (i < a.rules.n && o == a.rules.from[i]) {
          a.owner[p] = a.rules.to[i];
          break;
        }
      }
    }
    return;
  }
  if (cta < n_rule_ctas + n_set_ctas) {
    // Explicit writes are disjoint from pages touched by rules (host ledger
    // guarantees it), so no ordering between the two groups is needed.
    int i = (cta - n_rule_ctas) * kThreads + threadIdx.x;
    if (i < a.n_set) a.owner[a.set_pages[i]] = a.set_owner[i];
    return;
  }
  // Migration CTAs: kMigCtasPerPage per migrated page, 16-byte vector copies.
  int m = (cta - n_rule_ctas - n_set_ctas) / kMigCtasPerPage;
  int part = (cta - n_rule_ctas - n_set_ctas) % kMigCtasPerPage;
  if (m >= a.n_mig) return;
  Migration mg = a.migs[m];
  const int64_t span = a.page_size / kMigCtasPerPage;
  const int4* src = reinterpret_cast<const int4*>(a.window + (int64_t)mg.src * a.page_size + part * span);
  int4* dst = reinterpret_cast<int4*>(a.window + (int64_t)mg.dst * a.page_size + part * span);
  const int64_t n16 = span / 16;
  for (int64_t i = threadIdx.x; i < n16; i += kThreads * 4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * kThreads < n16) v[u] = __ldg(src + i + u * kThreads);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * kThreads < n16) dst[i + u * kThreads] = v[u];
  }
  // The src page's new owner comes from the explicit writes; only the table
  // entry is rewritten here. Readers run later on the same stream.
  if (part == 0 && threadIdx.x == 0)
    a.block_tables[(int64_t)mg.seq * a.max_blocks + mg.block] = mg.dst;
}

}  // namespace

void launch_switch(const SwitchArgs& a, cudaStream_t stream) {
  int n_rule_ctas = 0;
  if (a.rules.n > 0) {
    int64_t need = ((a.rules.hi ? a.rules.hi : a.n_pages) - a.rules.lo + kThreads - 1) / kThreads;
    n_rule_ctas = (int)(need < 2 * kNumSMs ? need : 2 * kNumSMs);
  }
  int n_set_ctas = (a.n_set + kThreads - 1) / kThreads;
  int n_mig_ctas = a.n_mig * kMigCtasPerPage;
  int grid = n_rule_ctas + n_set_ctas + n_mig_ctas;
  if (grid == 0) grid = 1;
  count_launch();
  switch_kernel<<<grid, kThreads, 0, stream>>>(a, n_rule_ctas, n_set_ctas);
}

}  // namespace ws

// Switch kernel interface: one launch applies a memory switch to the device
// page-ownership map, migrates live KV blocks off pages leaving the KV pool,
// and rewrites the block tables that pointed at them.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace ws {

constexpr int kMaxRules = 4;
constexpr int32_t kOwnerFree = -1;
constexpr int32_t kOwnerKV = -2;

// owner[p] = to[i] for the first i with owner[p] == from[i] (bulk moves such
// as "free -> KV" on promotion or "slot s -> free" on eviction).
struct SwitchRules {
  int32_t n;
  int32_t from[kMaxRules];
  int32_t to[kMaxRules];
  int64_t lo, hi;  // rules apply to pages [lo, hi) only (hi = 0: up to n_pages)
};

// Live KV block relocation: copy page src -> dst, then table[seq][block] = dst.
struct Migration {
  int32_t src, dst, seq, block;
};

struct SwitchArgs {
  int32_t* owner;            // [n_pages]
  int64_t n_pages;
  SwitchRules rules;
  const int32_t* set_pages;  // explicit owner writes (applied after rules)
  const int32_t* set_owner;
  int32_t n_set;
  const Migration* migs;
  int32_t n_mig;
  char* window;              // page window base
  int64_t page_size;
  int32_t* block_tables;     // [max_seqs, max_blocks]
  int32_t max_blocks;
};

void launch_switch(const SwitchArgs& a, cudaStream_t stream);

}  // namespace ws

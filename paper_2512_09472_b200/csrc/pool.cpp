// Per-GPU page pool: the page ledger of a universal worker and the CUDA VMM
// memory behind it.
//
// Host ledger (single writer, mutated synchronously before device work is
// enqueued — cluster.py:200-201) replaces GpuWorker's page counters
// (cluster.py:110-129) and adds page identities.
//
// Physical memory: the ledger's 2 MiB pages are backed by physical handles of
// `hpages` pages each (default 64 = 128 MiB; cuMemCreate), all mapped once,
// in page order, into one "page window" VA at init — page p lives at
// window + p * page. The driver's cost is per handle, not per byte (on this
// B200: create + map + set-access ~0.3-1.8 ms per 2 MiB handle vs ~4 us per
// 2 MiB with 128 MiB handles, profiles/r1_vmm_granularity.json), so large
// handles make a full-HBM pool cheap to build: 86,906 pages (170 GiB) in
// 0.2-1.5 s with 64-page handles vs 1.4-8 s with 16-page ones
// (profiles/r2_pool_init.txt).
//
// KV blocks address pages through the window: weight<->KV conversion is a
// ledger update + the switch kernel, never a driver call.
//
// Prewarm slots: a slot is placed, by a deterministic rule
// the host ledger and the device agree on, as
//   * WINDOWED  — the lowest contiguous run of free pages: the slot's VA is
//                 window + first * page, zero driver calls to create or evict;
//   * COMPOSITE — when no run is long enough: [free suffix of one handle] +
//                 whole free handles + [free prefix of one handle], each
//                 handle mapped whole into a private VA reservation (with one
//                 handle of slack either side) — driver cost per handle, and
//                 evicted composite slots are unmapped by a background worker
//                 (async-unmap contract, engine.py:615-632);
//   * a ledger-only pool (no device) falls back to the lowest free pages when
//     even a composite placement does not exist; a device pool refuses
//     (WS_ERR_FRAGMENTED) before any state changes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "driver.h"
#include "switch.cuh"

using ws::kOwnerFree;
using ws::kOwnerKV;

namespace {

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

enum SlotKind { kWindowed = 0, kComposite = 1, kScattered = 2 };

// One whole physical handle mapped into a composite slot's VA, at slot page
// offset `off` (negative for the head handle, whose first pages are not the
// slot's).
struct Seg {
  int32_t handle;
  int64_t off;
};

struct Slot {
  std::vector<int32_t> pages;  // slot page j -> physical page id
  int64_t mapped = 0;          // pages [0, mapped) addressable through the slot VA
  int kind = kWindowed;
  int va = -1;                 // composite: index into ws_pool::vas
  CUdeviceptr base = 0;        // slot VA (device pools)
  std::vector<Seg> segs;       // composite: handle mappings in slot-page order
  size_t segs_mapped = 0;      // segments [0, segs_mapped) are mapped
  uint64_t key = 0;
};

struct VaRange {
  CUdeviceptr base = 0;
  bool busy = false;
};

struct UnmapJob {
  int va;
  std::vector<std::pair<CUdeviceptr, size_t>> maps;  // (address, bytes) of every mapped handle
  cudaEvent_t fence;
};

#define DRV(expr)                                                           \
  do {                                                                      \
    CUresult _r = (expr);                                                   \
    if (_r != CUDA_SUCCESS) {                                               \
      const char* _s = "?";                                                 \
      if (ws::driver()) ws::driver()->cuGetErrorString(_r, &_s);            \
      WS_FAIL(WS_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, _s, __FILE__, __LINE__); \
    }                                                                       \
  } while (0)

}  // namespace

struct ws_pool {
  int dev = -1;
  int64_t n = 0, page = 0;
  // ---- host ledger ----
  std::vector<int32_t> owner;   // -1 free, -2 KV, >=0 slot id
  std::vector<int32_t> kv_seq;  // KV page -> sequence holding a block on it (-1 none)
  std::vector<int32_t> kv_blk;  //          -> block index in that sequence
  std::unordered_map<int64_t, Slot> slots;
  int64_t n_free = 0, n_slot = 0, n_kv = 0, kv_cap = 0, kv_used = 0, n_alloc = 0;
  // ---- sequences / block tables ----
  int32_t max_seqs = 0, max_blocks = 0;
  std::vector<int32_t> seq_len;
  std::vector<char> seq_live;
  int32_t* bt_host = nullptr;  // host mirror of the block tables
  int32_t* bt_dev = nullptr;
  // Block-table uploads go through a ring of pinned staging slots, each
  // guarded by an event, so a later host write can never race an earlier
  // queued copy (the mirror itself is rewritten freely).
  static constexpr int kBtSlots = 4;
  char* bt_stage = nullptr;
  cudaEvent_t bt_ev[kBtSlots] = {};
  int bt_next = 0;
  // ---- device ----
  const ws::Driver* drv = nullptr;
  std::vector<CUmemGenericAllocationHandle> handles;  // handle h backs pages [h*hpages, ...)
  int64_t hpages = 64;                                // ledger pages per physical handle
  bool exportable = false;                            // handles carry a POSIX-fd shareable type
  CUdeviceptr window = 0;
  int32_t* owner_dev = nullptr;
  char* stage_host = nullptr;  // pinned staging for switch lists
  char* stage_dev = nullptr;
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev = nullptr, sw_start = nullptr, sw_stop = nullptr;
  bool sw_recorded = false;
  int64_t sw_entries = 0;
  std::vector<VaRange> vas;                           // composite-slot VA reservations
  std::unordered_map<uint64_t, int64_t> last_first;   // keyed windowed slot -> its last first page
  int64_t remapped_pages = 0, reused_pages = 0;       // slot pages mapped by the driver / by the window
  int64_t placed_pages = 0;                           // device slot pages placed (for the per-page cost)
  double map_ms_total = 0;
  // ---- background unmap worker ----
  std::mutex mu;
  std::condition_variable cv, cv_done;
  std::deque<UnmapJob> jobs;
  std::thread worker;
  bool stop = false;
  int64_t pending = 0;
  double init_ms = 0, map_ms_per_page = 0, unmap_ms_per_page = 0;

  bool on_device() const { return dev >= 0; }
  int64_t n_handles() const { return (n + hpages - 1) / hpages; }
  int64_t handle_size(int64_t h) const { return std::min(hpages, n - h * hpages); }  // in pages
  size_t va_bytes() const { return (size_t)((n + 2 * hpages) * page); }
};

namespace {

int check_pool(ws_pool* p) {
  if (!p) WS_FAIL(WS_ERR_INVALID, "null pool");
  return WS_OK;
}

// Apply a switch on the device: rules + explicit writes + migrations.
int device_switch(ws_pool* p, const ws::SwitchRules& rules, const std::vector<int32_t>& set_pages,
                  int32_t set_owner, const std::vector<ws::Migration>& migs, cudaStream_t stream) {
  if (!p->on_device()) return WS_OK;
  WS_CUDA(cudaSetDevice(p->dev));
  size_t n_set = set_pages.size();
  size_t need = n_set * 8 + migs.size() * sizeof(ws::Migration) + 64;
  if (need > p->stage_bytes) WS_FAIL(WS_ERR_INVALID, "switch staging overflow");
  // The staging buffer is reused: wait until the previous upload consumed it.
  WS_CUDA(cudaEventSynchronize(p->stage_ev));
  int32_t* h_pages = reinterpret_cast<int32_t*>(p->stage_host);
  int32_t* h_owner = h_pages + n_set;
  ws::Migration* h_migs = reinterpret_cast<ws::Migration*>(
      p->stage_host + ((n_set * 8 + 15) / 16) * 16);
  if (n_set) {
    memcpy(h_pages, set_pages.data(), n_set * 4);
    for (size_t i = 0; i < n_set; ++i) h_owner[i] = set_owner;
  }
  if (!migs.empty()) memcpy(h_migs, migs.data(), migs.size() * sizeof(ws::Migration));
  size_t used = (size_t)((char*)(h_migs + migs.size()) - p->stage_host);
  WS_CUDA(cudaEventRecord(p->sw_start, stream));
  if (n_set || !migs.empty())
    WS_CUDA(cudaMemcpyAsync(p->stage_dev, p->stage_host, used, cudaMemcpyHostToDevice, stream));
  WS_CUDA(cudaEventRecord(p->stage_ev, stream));
  ws::SwitchArgs a{};
  a.owner = p->owner_dev;
  a.n_pages = p->n;
  a.rules = rules;
  a.set_pages = reinterpret_cast<const int32_t*>(p->stage_dev);
  a.set_owner = a.set_pages + n_set;
  a.n_set = (int32_t)n_set;
  a.migs = reinterpret_cast<const ws::Migration*>(p->stage_dev + ((char*)h_migs - p->stage_host));
  a.n_mig = (int32_t)migs.size();
  a.window = reinterpret_cast<char*>(p->window);
  a.page_size = p->page;
  a.block_tables = p->bt_dev;
  a.max_blocks = p->max_blocks;
  ws::launch_switch(a, stream);
  WS_CUDA(cudaGetLastError());
  WS_CUDA(cudaEventRecord(p->sw_stop, stream));
  p->sw_recorded = true;
  p->sw_entries = (int64_t)n_set + (int64_t)migs.size() + (rules.n ? (rules.hi ? rules.hi : p->n) - rules.lo : 0);
  return WS_OK;
}

ws::SwitchRules one_rule(int32_t from, int32_t to) {
  ws::SwitchRules r{};
  r.n = 1;
  r.from[0] = from;
  r.to[0] = to;
  return r;
}

void unmap_worker(ws_pool* p) {
  cudaSetDevice(p->dev);
  for (;;) {
    UnmapJob job;
    {
      std::unique_lock<std::mutex> lk(p->mu);
      p->cv.wait(lk, [&] { return p->stop || !p->jobs.empty(); });
      if (p->jobs.empty()) return;
      job = std::move(p->jobs.front());
      p->jobs.pop_front();
    }
    if (job.fence) {
      cudaEventSynchronize(job.fence);
      cudaEventDestroy(job.fence);
    }
    double t0 = now_ms();
    int64_t pages = 0;
    for (const auto& m : job.maps) {
      p->drv->cuMemUnmap(m.first, m.second);
      pages += (int64_t)(m.second / (size_t)p->page);
    }
    double t1 = now_ms();
    std::lock_guard<std::mutex> lk(p->mu);
    if (pages) p->unmap_ms_per_page = (t1 - t0) / (double)pages;
    p->vas[job.va].busy = false;
    p->pending -= 1;
    p->cv_done.notify_all();
  }
}

int acquire_va(ws_pool* p, int* out) {
  std::lock_guard<std::mutex> lk(p->mu);
  for (size_t i = 0; i < p->vas.size(); ++i)
    if (!p->vas[i].busy) {
      p->vas[i].busy = true;
      *out = (int)i;
      return WS_OK;
    }
  VaRange r;
  DRV(p->drv->cuMemAddressReserve(&r.base, p->va_bytes(), (size_t)(p->hpages * p->page), 0, 0));
  r.busy = true;
  p->vas.push_back(r);
  *out = (int)p->vas.size() - 1;
  return WS_OK;
}

// Make slot pages [first, first + count) addressable through the slot VA
// (memswitch.py:78-88 per-chunk map step). Windowed slots alias the page
// window: nothing to do. Composite slots map every handle segment that
// covers a page of the range and is not mapped yet, then grant access to the
// newly mapped span in one call.
int map_range(ws_pool* p, Slot& s, int64_t first, int64_t count) {
  if (first != s.mapped) WS_FAIL(WS_ERR_INVALID, "slot pages must be mapped in order");
  if (first + count > (int64_t)s.pages.size()) WS_FAIL(WS_ERR_INVALID, "map beyond slot");
  s.mapped += count;
  if (!p->on_device() || count == 0 || s.kind != kComposite) return WS_OK;
  const double t0 = now_ms();
  const size_t seg0 = s.segs_mapped;
  int64_t lo = INT64_MAX, hi = INT64_MIN, pages = 0;
  while (s.segs_mapped < s.segs.size() && s.segs[s.segs_mapped].off < s.mapped) {
    const Seg& g = s.segs[s.segs_mapped];
    const int64_t hs = p->handle_size(g.handle);
    DRV(p->drv->cuMemMap(s.base + g.off * p->page, (size_t)(hs * p->page), 0, p->handles[g.handle], 0));
    lo = std::min(lo, g.off);
    hi = std::max(hi, g.off + hs);
    pages += hs;
    ++s.segs_mapped;
  }
  if (s.segs_mapped > seg0) {
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = p->dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV(p->drv->cuMemSetAccess(s.base + lo * p->page, (size_t)((hi - lo) * p->page), &acc, 1));
    p->remapped_pages += pages;
  }
  p->map_ms_total += now_ms() - t0;
  return WS_OK;
}

// Slot placement (the identity rule; host ledger only, no side effects).
// Returns WS_OK and fills `s.pages`, `s.kind`, `s.segs`, or
// WS_ERR_FRAGMENTED when a device pool has no placement.
int place_slot(const ws_pool* p, int64_t n, uint64_t key, Slot& s) {
  s.pages.clear();
  s.segs.clear();
  const auto& own = p->owner;
  auto run_free = [&](int64_t f) {
    if (f < 0 || f + n > p->n) return false;
    for (int64_t q = f; q < f + n; ++q)
      if (own[q] != kOwnerFree) return false;
    return true;
  };
  auto windowed = [&](int64_t f) {
    s.kind = kWindowed;
    for (int64_t q = f; q < f + n; ++q) s.pages.push_back((int32_t)q);
    return WS_OK;
  };
  if (n == 0) return windowed(0);
  // 1. a keyed slot takes back the run it held last time if it is free
  if (key) {
    auto it = p->last_first.find(key);
    if (it != p->last_first.end() && run_free(it->second)) return windowed(it->second);
  }
  // 2. the lowest contiguous free run
  for (int64_t q = 0, run = 0; q < p->n; ++q) {
    run = own[q] == kOwnerFree ? run + 1 : 0;
    if (run == n) return windowed(q - n + 1);
  }
  // 3. composite: [free suffix of one handle] + whole free handles + [free prefix of one handle]
  const int64_t G = p->hpages, H = p->n_handles();
  std::vector<int64_t> whole, fs(H), fp(H);
  for (int64_t h = 0; h < H; ++h) {
    const int64_t b = h * G, gs = p->handle_size(h);
    int64_t nf = 0;
    for (int64_t q = b; q < b + gs; ++q) nf += own[q] == kOwnerFree;
    while (fp[h] < gs && own[b + fp[h]] == kOwnerFree) ++fp[h];
    while (fs[h] < gs && own[b + gs - 1 - fs[h]] == kOwnerFree) ++fs[h];
    if (nf == gs && gs == G) whole.push_back(h);
  }
  auto is_whole = [&](int64_t h) { return fp[h] == G; };
  int64_t head = -1;  // the partial (or short last) handle with the longest free suffix
  for (int64_t h = 0; h < H; ++h)
    if (!is_whole(h) && fs[h] > 0 && (head < 0 || fs[h] > fs[head])) head = h;
  int64_t got = head >= 0 ? fs[head] : 0;
  if (got >= n) head = -1, got = 0;  // cannot happen (step 2 found no run) — defensive
  const int64_t nw = std::min<int64_t>((n - got) / G, (int64_t)whole.size());
  got += nw * G;
  int64_t rem = n - got, tail = -1;
  if (rem > 0) {
    for (int64_t h = 0; h < H; ++h)  // best-fit partial prefix
      if (h != head && !is_whole(h) && fp[h] >= rem && (tail < 0 || fp[h] < fp[tail])) tail = h;
    if (tail < 0 && (int64_t)whole.size() > nw) tail = whole[nw];  // first rem pages of one more whole handle
  }
  if (rem > 0 && tail < 0) {
    if (p->on_device())
      WS_FAIL(WS_ERR_FRAGMENTED,
              "slot of %lld pages cannot be placed: free pages are fragmented below the %lld-page physical "
              "handle granularity", (long long)n, (long long)G);
    s.kind = kScattered;  // ledger-only pool: identities only, lowest free pages
    for (int64_t q = 0; q < p->n && (int64_t)s.pages.size() < n; ++q)
      if (own[q] == kOwnerFree) s.pages.push_back((int32_t)q);
    return WS_OK;
  }
  s.kind = kComposite;
  int64_t off = 0;
  if (head >= 0) {
    const int64_t gs = p->handle_size(head), r = gs - fs[head];
    s.segs.push_back({(int32_t)head, -r});
    for (int64_t q = 0; q < fs[head]; ++q) s.pages.push_back((int32_t)(head * G + r + q));
    off = fs[head];
  }
  for (int64_t i = 0; i < nw; ++i) {
    s.segs.push_back({(int32_t)whole[i], off});
    for (int64_t q = 0; q < G; ++q) s.pages.push_back((int32_t)(whole[i] * G + q));
    off += G;
  }
  if (rem > 0) {
    s.segs.push_back({(int32_t)tail, off});
    for (int64_t q = 0; q < rem; ++q) s.pages.push_back((int32_t)(tail * G + q));
  }
  return WS_OK;
}

// Remove n KV pages (highest ids), relocating live blocks. Host ledger first,
// then one switch launch. The victims are exactly the KV pages with id >=
// the lowest victim, so the device applies them as one ranged rule (KV ->
// free on [lowest, n)) instead of an uploaded page list.
int kv_shrink(ws_pool* p, int64_t n, cudaStream_t stream) {
  if (n <= 0) return WS_OK;
  if (n > p->n_kv) WS_FAIL(WS_ERR_INVALID, "shrink %lld > kv %lld", (long long)n, (long long)p->n_kv);
  int32_t* own = p->owner.data();
  int64_t lowest = p->n, seen = 0;
  std::vector<int32_t> live;  // victims holding a live block, descending
  while (seen < n) {
    --lowest;
    if (own[lowest] == kOwnerKV) {
      ++seen;
      if (p->kv_seq[lowest] >= 0) live.push_back((int32_t)lowest);
    }
  }
  std::vector<ws::Migration> migs;
  int64_t cursor = 0;
  for (auto it = live.rbegin(); it != live.rend(); ++it) {  // ascending page order
    const int32_t v = *it;
    while (cursor < lowest && !(own[cursor] == kOwnerKV && p->kv_seq[cursor] < 0)) ++cursor;
    if (cursor >= lowest)
      WS_FAIL(WS_ERR_KV_BUSY, "KV shrink by %lld pages would drop live blocks", (long long)n);
    migs.push_back({v, (int32_t)cursor, p->kv_seq[v], p->kv_blk[v]});
    ++cursor;
  }
  for (const auto& m : migs) {
    p->kv_seq[m.dst] = m.seq;
    p->kv_blk[m.dst] = m.block;
    p->bt_host[(int64_t)m.seq * p->max_blocks + m.block] = m.dst;
  }
  for (int32_t v : live) {
    p->kv_seq[v] = -1;
    p->kv_blk[v] = -1;
  }
  for (int64_t q = lowest; q < p->n; ++q) own[q] = own[q] == kOwnerKV ? kOwnerFree : own[q];
  p->n_kv -= n;
  p->n_free += n;
  ws::SwitchRules r = one_rule(kOwnerKV, kOwnerFree);
  r.lo = lowest;
  return device_switch(p, r, {}, 0, migs, stream);
}

int kv_grow(ws_pool* p, int64_t n, cudaStream_t stream) {
  if (n <= 0) return WS_OK;
  if (n > p->n_free) WS_FAIL(WS_ERR_INSUFFICIENT, "insufficient pages (need %lld, free %lld)",
                             (long long)n, (long long)p->n_free);
  std::vector<int32_t> got;
  for (int64_t q = 0; q < p->n && (int64_t)got.size() < n; ++q)
    if (p->owner[q] == kOwnerFree) got.push_back((int32_t)q);
  for (int32_t q : got) p->owner[q] = kOwnerKV;
  p->n_free -= n;
  p->n_kv += n;
  ws::SwitchRules none{};
  return device_switch(p, none, got, kOwnerKV, {}, stream);
}

}  // namespace

extern "C" {

int ws_pool_create(int32_t device, int64_t total_pages, int64_t page_size, ws_pool** out) {
  return ws_pool_create_ex(device, total_pages, page_size, 64, out);
}

int ws_pool_create_ex(int32_t device, int64_t total_pages, int64_t page_size, int64_t handle_pages,
                      ws_pool** out) {
  if (total_pages < 1 || page_size < 1) WS_FAIL(WS_ERR_INVALID, "pool needs pages and a page size");
  if (total_pages > (int64_t)INT32_MAX) WS_FAIL(WS_ERR_INVALID, "too many pages");
  if (handle_pages < 1) WS_FAIL(WS_ERR_INVALID, "handle_pages must be >= 1");
  ws_pool* p = new ws_pool();
  p->dev = device;
  p->n = total_pages;
  p->page = page_size;
  p->hpages = handle_pages;
  p->owner.assign(total_pages, kOwnerFree);
  p->kv_seq.assign(total_pages, -1);
  p->kv_blk.assign(total_pages, -1);
  p->n_free = total_pages;
  if (device >= 0) {
    double t0 = now_ms();
    auto fail = [&](int code) {
      ws_pool_destroy(p);
      return code;
    };
    p->drv = ws::driver();
    if (!p->drv) return fail(WS_ERR_NO_DEVICE);
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(0) != cudaSuccess) {
      ws::set_error("cudaSetDevice failed");
      return fail(WS_ERR_NO_DEVICE);
    }
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    if (p->drv->cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) !=
            CUDA_SUCCESS ||
        page_size % (int64_t)gran != 0) {
      ws::set_error("page size is not a multiple of the VMM granularity");
      return fail(WS_ERR_INVALID);
    }
    if (p->drv->cuMemAddressReserve(&p->window, (size_t)(total_pages * page_size),
                                    (size_t)(handle_pages * page_size), 0, 0) != CUDA_SUCCESS) {
      ws::set_error("cuMemAddressReserve(window) failed");
      return fail(WS_ERR_CUDA);
    }
    const int64_t H = p->n_handles();
    p->handles.reserve(H);
    // Exportable handles (POSIX fd) so a peer process can map this pool's
    // slots as its cold-start weight source; plain handles if unsupported.
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    for (int64_t h = 0; h < H; ++h) {
      const size_t bytes = (size_t)(p->handle_size(h) * page_size);
      CUmemGenericAllocationHandle hd;
      CUresult r = p->drv->cuMemCreate(&hd, bytes, &prop, 0);
      if (r != CUDA_SUCCESS && h == 0 && prop.requestedHandleTypes != CU_MEM_HANDLE_TYPE_NONE) {
        prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
        r = p->drv->cuMemCreate(&hd, bytes, &prop, 0);
      }
      p->exportable = prop.requestedHandleTypes == CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      if (r == CUDA_SUCCESS) {
        p->handles.push_back(hd);
        r = p->drv->cuMemMap(p->window + h * handle_pages * page_size, bytes, 0, hd, 0);
      }
      if (r != CUDA_SUCCESS) {
        // destroy unmaps and releases only the fully mapped handles
        if ((int64_t)p->handles.size() == h + 1) {
          p->drv->cuMemRelease(p->handles.back());
          p->handles.pop_back();
        }
        ws::set_error("cuMemCreate/cuMemMap of the page window failed (out of HBM?)");
        return fail(WS_ERR_CUDA);
      }
    }
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (p->drv->cuMemSetAccess(p->window, (size_t)(total_pages * page_size), &acc, 1) !=
        CUDA_SUCCESS) {
      ws::set_error("cuMemSetAccess(window) failed");
      return fail(WS_ERR_CUDA);
    }
    // Zero every page once: afterwards a page only ever holds finite bf16
    // (weights or KV), so kernels may read stale-but-finite rows and mask them.
    if (cudaMemset(reinterpret_cast<void*>(p->window), 0, (size_t)(total_pages * page_size)) != cudaSuccess) {
      ws::set_error("zeroing the page window failed");
      return fail(WS_ERR_CUDA);
    }
    p->stage_bytes = (size_t)total_pages * 24 + 4096;
    if (cudaMalloc(&p->owner_dev, total_pages * 4) != cudaSuccess ||
        cudaMemcpy(p->owner_dev, p->owner.data(), total_pages * 4, cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaHostAlloc(&p->stage_host, p->stage_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaMalloc(&p->stage_dev, p->stage_bytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->stage_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&p->sw_start) != cudaSuccess || cudaEventCreate(&p->sw_stop) != cudaSuccess) {
      ws::set_error("pool device buffers allocation failed");
      return fail(WS_ERR_CUDA);
    }
    cudaEventRecord(p->stage_ev, 0);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      ws::set_error("pool init synchronize failed");
      return fail(WS_ERR_CUDA);
    }
    p->worker = std::thread(unmap_worker, p);
    p->init_ms = now_ms() - t0;
  }
  *out = p;
  return WS_OK;
}

namespace {
void unmap_slot_now(ws_pool* p, const Slot& s) {
  for (size_t i = 0; i < s.segs_mapped; ++i)
    p->drv->cuMemUnmap(s.base + s.segs[i].off * p->page, (size_t)(p->handle_size(s.segs[i].handle) * p->page));
}
}  // namespace

int ws_pool_destroy(ws_pool* p) {
  if (!p) return WS_OK;
  if (p->worker.joinable()) {
    {
      std::lock_guard<std::mutex> lk(p->mu);
      p->stop = true;
    }
    p->cv.notify_all();
    p->worker.join();
  }
  if (p->on_device() && p->drv) {
    cudaSetDevice(p->dev);
    cudaDeviceSynchronize();
    for (auto& kv : p->slots)
      if (kv.second.kind == kComposite) unmap_slot_now(p, kv.second);
    for (auto& v : p->vas) p->drv->cuMemAddressFree(v.base, p->va_bytes());
    for (size_t h = 0; h < p->handles.size(); ++h)
      p->drv->cuMemUnmap(p->window + h * p->hpages * p->page, (size_t)(p->handle_size(h) * p->page));
    for (auto h : p->handles) p->drv->cuMemRelease(h);
    if (p->window) p->drv->cuMemAddressFree(p->window, (size_t)(p->n * p->page));
    if (p->owner_dev) cudaFree(p->owner_dev);
    if (p->stage_dev) cudaFree(p->stage_dev);
    if (p->stage_host) cudaFreeHost(p->stage_host);
    if (p->bt_dev) cudaFree(p->bt_dev);
    if (p->bt_stage) cudaFreeHost(p->bt_stage);
    for (cudaEvent_t e : p->bt_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {p->stage_ev, p->sw_start, p->sw_stop})
      if (e) cudaEventDestroy(e);
  }
  free(p->bt_host);
  delete p;
  return WS_OK;
}

int ws_pool_counts_get(ws_pool* p, ws_pool_counts* o) {
  if (int e = check_pool(p)) return e;
  o->total_pages = p->n;
  o->free_pages = p->n_free;
  o->slot_pages = p->n_slot;
  o->kv_pages_mapped = p->n_kv;
  o->kv_pages_used = p->kv_used;
  o->kv_capacity_pages = p->kv_cap;
  o->kv_pages_allocated = p->n_alloc;
  o->n_slots = (int64_t)p->slots.size();
  std::lock_guard<std::mutex> lk(p->mu);
  o->pending_unmaps = p->pending;
  return WS_OK;
}

int ws_pool_owner_map(ws_pool* p, int32_t* out, int64_t n) {
  if (int e = check_pool(p)) return e;
  if (n < p->n) WS_FAIL(WS_ERR_INVALID, "buffer too small");
  memcpy(out, p->owner.data(), p->n * 4);
  return WS_OK;
}

int ws_pool_device_owner_map(ws_pool* p, int32_t* out, int64_t n) {
  if (int e = check_pool(p)) return e;
  if (!p->on_device()) WS_FAIL(WS_ERR_NO_DEVICE, "ledger-only pool");
  if (n < p->n) WS_FAIL(WS_ERR_INVALID, "buffer too small");
  WS_CUDA(cudaSetDevice(p->dev));
  WS_CUDA(cudaDeviceSynchronize());
  WS_CUDA(cudaMemcpy(out, p->owner_dev, p->n * 4, cudaMemcpyDeviceToHost));
  return WS_OK;
}

int ws_pool_window(ws_pool* p, void** base) {
  if (int e = check_pool(p)) return e;
  if (!p->on_device()) WS_FAIL(WS_ERR_NO_DEVICE, "ledger-only pool");
  *base = reinterpret_cast<void*>(p->window);
  return WS_OK;
}

int ws_pool_timing(ws_pool* p, double* init_ms, double* map_pp, double* unmap_pp) {
  if (int e = check_pool(p)) return e;
  std::lock_guard<std::mutex> lk(p->mu);
  *init_ms = p->init_ms;
  *map_pp = p->placed_pages ? p->map_ms_total / (double)p->placed_pages : 0.0;
  *unmap_pp = p->unmap_ms_per_page;
  return WS_OK;
}

int ws_pool_sync_unmaps(ws_pool* p) {
  if (int e = check_pool(p)) return e;
  std::unique_lock<std::mutex> lk(p->mu);
  p->cv_done.wait(lk, [&] { return p->pending == 0; });
  return WS_OK;
}

int ws_pool_handle_pages(ws_pool* p, int64_t* handle_pages) {
  if (int e = check_pool(p)) return e;
  *handle_pages = p->hpages;
  return WS_OK;
}

int ws_slot_create(ws_pool* p, int64_t slot_id, int64_t pages, int32_t map_now, void** va_out) {
  return ws_slot_create_keyed(p, slot_id, pages, map_now, 0, va_out);
}

int ws_slot_create_keyed(ws_pool* p, int64_t slot_id, int64_t pages, int32_t map_now, uint64_t key,
                         void** va_out) {
  if (int e = check_pool(p)) return e;
  if (slot_id < 0 || slot_id > INT32_MAX) WS_FAIL(WS_ERR_INVALID, "slot id out of range");
  if (p->slots.count(slot_id)) WS_FAIL(WS_ERR_DUPLICATE, "already holds slot %lld", (long long)slot_id);
  if (pages < 0) WS_FAIL(WS_ERR_INVALID, "negative page count");
  if (pages > p->n_free)
    WS_FAIL(WS_ERR_INSUFFICIENT, "insufficient pages (need %lld, free %lld)", (long long)pages,
            (long long)p->n_free);
  Slot s;
  if (int e = place_slot(p, pages, key, s)) return e;
  s.key = key;
  if (p->on_device()) {
    WS_CUDA(cudaSetDevice(p->dev));
    if (s.kind == kComposite) {
      if (int e = acquire_va(p, &s.va)) return e;
      s.base = p->vas[s.va].base + (CUdeviceptr)(p->hpages * p->page);
    } else {
      s.base = p->window + (CUdeviceptr)(pages ? (int64_t)s.pages[0] * p->page : 0);
    }
    p->placed_pages += pages;
    if (s.kind == kWindowed) p->reused_pages += pages;
  }
  if (key && s.kind == kWindowed && pages) p->last_first[key] = s.pages[0];
  for (int32_t q : s.pages) p->owner[q] = (int32_t)slot_id;
  p->n_free -= pages;
  p->n_slot += pages;
  Slot& ref = p->slots[slot_id] = std::move(s);
  if (ref.kind == kWindowed && pages) {  // a contiguous run: one ranged rule, no page list
    ws::SwitchRules r = one_rule(kOwnerFree, (int32_t)slot_id);
    r.lo = ref.pages[0];
    r.hi = ref.pages[0] + pages;
    if (int e = device_switch(p, r, {}, 0, {}, 0)) return e;
  } else {
    ws::SwitchRules none{};
    if (int e = device_switch(p, none, ref.pages, (int32_t)slot_id, {}, 0)) return e;
  }
  if (map_now)
    if (int e = map_range(p, ref, 0, pages)) return e;
  if (va_out) *va_out = p->on_device() ? reinterpret_cast<void*>(ref.base) : nullptr;
  return WS_OK;
}

int ws_slot_map_chunk(ws_pool* p, int64_t slot_id, int64_t first, int64_t count) {
  if (int e = check_pool(p)) return e;
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  return map_range(p, it->second, first, count);
}

int ws_slot_evict(ws_pool* p, int64_t slot_id, void* fence_stream) {
  if (int e = check_pool(p)) return e;
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  Slot s = std::move(it->second);
  p->slots.erase(it);
  for (int32_t q : s.pages) p->owner[q] = kOwnerFree;
  p->n_free += (int64_t)s.pages.size();
  p->n_slot -= (int64_t)s.pages.size();
  if (!p->on_device()) return WS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(fence_stream);
  if (int e = device_switch(p, one_rule((int32_t)slot_id, kOwnerFree), {}, 0, {}, st)) return e;
  if (s.kind != kComposite) return WS_OK;  // windowed: the window mapping stays, nothing to undo
  UnmapJob job;
  job.va = s.va;
  for (size_t i = 0; i < s.segs_mapped; ++i)
    job.maps.emplace_back(s.base + s.segs[i].off * p->page, (size_t)(p->handle_size(s.segs[i].handle) * p->page));
  WS_CUDA(cudaEventCreateWithFlags(&job.fence, cudaEventDisableTiming));
  WS_CUDA(cudaEventRecord(job.fence, st));
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->jobs.push_back(std::move(job));
    p->pending += 1;
  }
  p->cv.notify_all();
  return WS_OK;
}

int ws_slot_info(ws_pool* p, int64_t slot_id, int64_t* pages, int64_t* mapped, void** va) {
  if (int e = check_pool(p)) return e;
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  if (pages) *pages = (int64_t)it->second.pages.size();
  if (mapped) *mapped = it->second.mapped;
  if (va) *va = p->on_device() ? reinterpret_cast<void*>(it->second.base) : nullptr;
  return WS_OK;
}

int ws_slot_placement(ws_pool* p, int64_t slot_id, int32_t* kind, int64_t* handles_mapped) {
  if (int e = check_pool(p)) return e;
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  *kind = it->second.kind;
  *handles_mapped = (int64_t)it->second.segs.size();
  return WS_OK;
}

int ws_slot_pages(ws_pool* p, int64_t slot_id, int32_t* ids, int64_t cap, int64_t* n_out) {
  if (int e = check_pool(p)) return e;
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  int64_t n = (int64_t)it->second.pages.size();
  *n_out = n;
  if (ids) memcpy(ids, it->second.pages.data(), std::min(n, cap) * 4);
  return WS_OK;
}

int ws_kv_map_all(ws_pool* p, void* stream, int64_t* kv_out) {
  if (int e = check_pool(p)) return e;
  int32_t* own = p->owner.data();
  for (int64_t q = 0; q < p->n; ++q)  // branch-free: vectorises (89k pages in a few us)
    own[q] = own[q] == kOwnerFree ? kOwnerKV : own[q];
  p->n_kv += p->n_free;
  p->n_free = 0;
  p->kv_cap = p->n_kv;
  if (kv_out) *kv_out = p->n_kv;
  return device_switch(p, one_rule(kOwnerFree, kOwnerKV), {}, 0, {},
                       reinterpret_cast<cudaStream_t>(stream));
}

int ws_kv_reclaim(ws_pool* p, int32_t inflight, int32_t max_batch, double kv_used_bytes,
                  void* stream, int64_t* freed_out) {
  if (int e = check_pool(p)) return e;
  // cluster.py:358-363. capacity is an exact integer byte count; `used` is
  // min(kv_used, capacity), whichever type wins in the reference.
  const int64_t cap_bytes = p->kv_cap * p->page;
  const double used = (double)cap_bytes < kv_used_bytes ? (double)cap_bytes : kv_used_bytes;
  // The reference records kv_pages_used before Eq. 1 validates its inputs.
  p->kv_used = (int64_t)std::ceil(used / (double)p->page);
  if (inflight < 0 || inflight > max_batch)
    WS_FAIL(WS_ERR_INVALID, "inflight %d outside [0, %d]", inflight, max_batch);
  if (used < 0) WS_FAIL(WS_ERR_INVALID, "kv_used %.17g outside [0, %lld]", used, (long long)cap_bytes);
  // Eq. 1 with M an exact integer: M*R is exact, then one rounding per op.
  const double expect = (double)(cap_bytes * (int64_t)inflight) / (double)max_batch;
  const double buffer = used + (double)cap_bytes / (double)max_batch;
  const double target = expect >= buffer ? expect : buffer;
  const double reserved = (double)(p->n_kv * p->page);
  int64_t freed = (int64_t)std::floor((reserved - target) / (double)p->page);
  if (freed < 0) freed = 0;
  if (int e = kv_shrink(p, freed, reinterpret_cast<cudaStream_t>(stream))) return e;
  *freed_out = freed * p->page;
  return WS_OK;
}

int ws_kv_resize(ws_pool* p, int64_t kv_pages, void* stream) {
  if (int e = check_pool(p)) return e;
  if (kv_pages < 0) WS_FAIL(WS_ERR_INVALID, "negative KV size");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (kv_pages < p->n_kv) return kv_shrink(p, p->n_kv - kv_pages, st);
  return kv_grow(p, kv_pages - p->n_kv, st);
}

int ws_kv_release(ws_pool* p, void* stream) {
  if (int e = check_pool(p)) return e;
  if (p->n_alloc) WS_FAIL(WS_ERR_KV_BUSY, "KV release with %lld live blocks", (long long)p->n_alloc);
  int32_t* own = p->owner.data();
  for (int64_t q = 0; q < p->n; ++q)
    own[q] = own[q] == kOwnerKV ? kOwnerFree : own[q];
  p->n_free += p->n_kv;
  p->n_kv = p->kv_cap = p->kv_used = 0;
  return device_switch(p, one_rule(kOwnerKV, kOwnerFree), {}, 0, {},
                       reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- sequences

int ws_pool_seq_config(ws_pool* p, int32_t max_seqs, int32_t max_blocks) {
  if (int e = check_pool(p)) return e;
  if (max_seqs < 1 || max_blocks < 1) WS_FAIL(WS_ERR_INVALID, "bad sequence table shape");
  if (p->n_alloc) WS_FAIL(WS_ERR_STATE, "sequences still hold KV blocks");
  size_t bytes = (size_t)max_seqs * max_blocks * 4;
  free(p->bt_host);
  p->bt_host = static_cast<int32_t*>(malloc(bytes));
  if (p->on_device()) {
    WS_CUDA(cudaSetDevice(p->dev));
    WS_CUDA(cudaDeviceSynchronize());
    if (p->bt_dev) cudaFree(p->bt_dev);
    if (p->bt_stage) cudaFreeHost(p->bt_stage);
    p->bt_dev = nullptr;
    p->bt_stage = nullptr;
    WS_CUDA(cudaMalloc(&p->bt_dev, bytes));
    WS_CUDA(cudaMemset(p->bt_dev, 0xff, bytes));
    WS_CUDA(cudaHostAlloc(&p->bt_stage, (size_t)ws_pool::kBtSlots * max_blocks * 4, cudaHostAllocDefault));
    for (auto& e : p->bt_ev) {
      if (!e) WS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      WS_CUDA(cudaEventRecord(e, 0));
    }
  }
  memset(p->bt_host, 0xff, bytes);
  p->max_seqs = max_seqs;
  p->max_blocks = max_blocks;
  p->seq_len.assign(max_seqs, 0);
  p->seq_live.assign(max_seqs, 0);
  return WS_OK;
}

int ws_seq_open(ws_pool* p, int32_t* seq_out) {
  if (int e = check_pool(p)) return e;
  for (int32_t s = 0; s < p->max_seqs; ++s)
    if (!p->seq_live[s]) {
      p->seq_live[s] = 1;
      p->seq_len[s] = 0;
      *seq_out = s;
      return WS_OK;
    }
  WS_FAIL(WS_ERR_INSUFFICIENT, "no free sequence rows (max %d)", p->max_seqs);
}

int ws_seq_reserve(ws_pool* p, int32_t seq, int32_t n_blocks, void* stream) {
  if (int e = check_pool(p)) return e;
  if (seq < 0 || seq >= p->max_seqs || !p->seq_live[seq]) WS_FAIL(WS_ERR_INVALID, "bad sequence %d", seq);
  if (n_blocks > p->max_blocks) WS_FAIL(WS_ERR_INVALID, "sequence exceeds %d blocks", p->max_blocks);
  int32_t have = p->seq_len[seq];
  if (n_blocks <= have) return WS_OK;
  std::vector<int32_t> got;
  for (int64_t q = 0; q < p->n && (int32_t)got.size() < n_blocks - have; ++q)
    if (p->owner[q] == kOwnerKV && p->kv_seq[q] < 0) got.push_back((int32_t)q);
  if ((int32_t)got.size() < n_blocks - have)
    WS_FAIL(WS_ERR_INSUFFICIENT, "insufficient pages (need %d KV blocks, free %d)", n_blocks - have,
            (int)got.size());
  int32_t* row = p->bt_host + (int64_t)seq * p->max_blocks;
  for (int32_t i = 0; i < (int32_t)got.size(); ++i) {
    p->kv_seq[got[i]] = seq;
    p->kv_blk[got[i]] = have + i;
    row[have + i] = got[i];
  }
  p->n_alloc += (int64_t)got.size();
  p->seq_len[seq] = n_blocks;
  if (p->on_device()) {
    WS_CUDA(cudaSetDevice(p->dev));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int slot = p->bt_next;
    p->bt_next = (p->bt_next + 1) % ws_pool::kBtSlots;
    WS_CUDA(cudaEventSynchronize(p->bt_ev[slot]));  // the copy that last used this slot ran
    int32_t* stage = reinterpret_cast<int32_t*>(p->bt_stage) + (int64_t)slot * p->max_blocks;
    memcpy(stage, row + have, (size_t)(n_blocks - have) * 4);
    WS_CUDA(cudaMemcpyAsync(p->bt_dev + (int64_t)seq * p->max_blocks + have, stage,
                            (size_t)(n_blocks - have) * 4, cudaMemcpyHostToDevice, st));
    WS_CUDA(cudaEventRecord(p->bt_ev[slot], st));
  }
  return WS_OK;
}

int ws_seq_close(ws_pool* p, int32_t seq) {
  if (int e = check_pool(p)) return e;
  if (seq < 0 || seq >= p->max_seqs || !p->seq_live[seq]) WS_FAIL(WS_ERR_INVALID, "bad sequence %d", seq);
  int32_t* row = p->bt_host + (int64_t)seq * p->max_blocks;
  for (int32_t i = 0; i < p->seq_len[seq]; ++i) {
    p->kv_seq[row[i]] = -1;
    p->kv_blk[row[i]] = -1;
    row[i] = -1;
  }
  p->n_alloc -= p->seq_len[seq];
  p->seq_len[seq] = 0;
  p->seq_live[seq] = 0;
  return WS_OK;  // stale device entries are never read: the row is dead
}

int ws_seq_blocks(ws_pool* p, int32_t seq, int32_t* ids, int32_t cap, int32_t* n_out) {
  if (int e = check_pool(p)) return e;
  if (seq < 0 || seq >= p->max_seqs) WS_FAIL(WS_ERR_INVALID, "bad sequence %d", seq);
  *n_out = p->seq_len[seq];
  if (ids) memcpy(ids, p->bt_host + (int64_t)seq * p->max_blocks, std::min(cap, p->seq_len[seq]) * 4);
  return WS_OK;
}

int ws_pool_block_tables(ws_pool* p, int32_t** dev_out, int32_t* max_blocks_out) {
  if (int e = check_pool(p)) return e;
  *dev_out = p->bt_dev;
  *max_blocks_out = p->max_blocks;
  return WS_OK;
}

int ws_pool_last_switch(ws_pool* p, double* kernel_ms, int64_t* entries) {
  if (int e = check_pool(p)) return e;
  if (!p->on_device() || !p->sw_recorded) {
    *kernel_ms = 0;
    *entries = 0;
    return WS_OK;
  }
  WS_CUDA(cudaEventSynchronize(p->sw_stop));
  float ms = 0;
  WS_CUDA(cudaEventElapsedTime(&ms, p->sw_start, p->sw_stop));
  *kernel_ms = ms;
  *entries = p->sw_entries;
  return WS_OK;
}

}  // extern "C"

namespace ws {
// Internal accessor for the model driver (not part of the C-ABI).
int pool_kv_view(ws_pool* p, char** window, int64_t* page_size, int32_t** block_tables,
                 int32_t* max_blocks, int64_t* n_pages) {
  if (!p || !p->on_device()) WS_FAIL(WS_ERR_NO_DEVICE, "model forward needs a device pool");
  if (!p->bt_dev) WS_FAIL(WS_ERR_STATE, "sequence table not configured (ws_pool_seq_config)");
  *n_pages = p->n;
  *window = reinterpret_cast<char*>(p->window);
  *page_size = p->page;
  *block_tables = p->bt_dev;
  *max_blocks = p->max_blocks;
  return WS_OK;
}
}  // namespace ws

// ---------------------------------------------------------------- peer source
// Export the physical handles that cover slot pages [0, pages) of a windowed
// slot as POSIX fds (the caller passes them to the peer process, e.g. over a
// Unix socket with SCM_RIGHTS, and closes its copies). `offset_out` is the
// slot's byte offset inside the first exported handle.
extern "C" int ws_pool_export_slot(ws_pool* p, int64_t slot_id, int32_t* fds, int64_t* sizes, int64_t cap,
                                   int64_t* n_out, int64_t* offset_out) {
  if (int e = check_pool(p)) return e;
  if (!p->on_device()) WS_FAIL(WS_ERR_NO_DEVICE, "ledger-only pool");
  if (!p->exportable) WS_FAIL(WS_ERR_STATE, "pool handles are not exportable on this system");
  auto it = p->slots.find(slot_id);
  if (it == p->slots.end()) WS_FAIL(WS_ERR_NO_SLOT, "no slot %lld", (long long)slot_id);
  const Slot& s = it->second;
  if (s.kind != kWindowed || s.pages.empty()) WS_FAIL(WS_ERR_STATE, "only windowed slots are exported");
  const int64_t first = s.pages.front(), last = s.pages.back();
  const int64_t h0 = first / p->hpages, h1 = last / p->hpages;
  if (h1 - h0 + 1 > cap) WS_FAIL(WS_ERR_INVALID, "fd buffer too small (%lld handles)", (long long)(h1 - h0 + 1));
  for (int64_t h = h0; h <= h1; ++h) {
    int fd = -1;
    DRV(p->drv->cuMemExportToShareableHandle(&fd, p->handles[h], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    fds[h - h0] = fd;
    sizes[h - h0] = p->handle_size(h) * p->page;
  }
  *n_out = h1 - h0 + 1;
  *offset_out = (first - h0 * p->hpages) * p->page;
  return WS_OK;
}

extern "C" int ws_pool_map_stats(ws_pool* p, int64_t* remapped, int64_t* reused) {
  if (int e = check_pool(p)) return e;
  *remapped = p->remapped_pages;
  *reused = p->reused_pages;
  return WS_OK;
}

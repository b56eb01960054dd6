// Planning math of the universal worker: prewarm-prefix sizing, catch-up
// stall, Eq. 1 reservation target and the two-stage map/copy schedule.
//
// Bit-exact float64 restatements of the reference's analytic model
// (cluster.py:79-197, memswitch.py:59-122, kernels.py:68-77). Built with
// -ffp-contract=off so every product/sum rounds exactly like CPython.
#include <cmath>
#include <vector>

#include "common.h"

namespace {

// Reference evaluation order: layer_bytes = partition/layers (int/int true
// division, cluster.py:85-88); t_load = layer_bytes/bw; t_comp =
// (a*tokens + b)/layers (cluster.py:158-159).
struct LayerTimes {
  double t_load, t_comp;
};

bool layer_times(int64_t weight_bytes, int32_t parallelism, int32_t layers, double a, double b,
                 double bandwidth, int32_t tokens, LayerTimes* out) {
  if (parallelism < 1 || layers < 1 || weight_bytes < 1) return false;
  int64_t part = weight_bytes / parallelism + (weight_bytes % parallelism ? 1 : 0);
  double layer_bytes = (double)part / (double)layers;
  out->t_load = layer_bytes / bandwidth;
  out->t_comp = (a * (double)tokens + b) / (double)layers;
  return true;
}

}  // namespace

extern "C" {

int ws_required_prewarm_layers(int64_t weight_bytes, int32_t parallelism, int32_t layers,
                               double prefill_a_ms, double prefill_b_ms, double bandwidth,
                               int32_t ref_input_tokens, int32_t* k_out) {
  if (!(bandwidth > 0)) WS_FAIL(WS_ERR_INVALID, "bandwidth must be > 0");
  LayerTimes t;
  if (!layer_times(weight_bytes, parallelism, layers, prefill_a_ms, prefill_b_ms, bandwidth,
                   ref_input_tokens, &t))
    WS_FAIL(WS_ERR_INVALID, "invalid model spec");
  // Stall-free iff for every l in (k, L]: (l-k)*t_load <= (l-1)*t_comp. The
  // condition gets easier as k grows, so scan k upward and stop at the first.
  for (int32_t k = 1; k < layers; ++k) {
    bool ok = true;
    for (int32_t l = k + 1; l <= layers && ok; ++l)
      ok = (double)(l - k) * t.t_load <= (double)(l - 1) * t.t_comp;
    if (ok) {
      *k_out = k;
      return WS_OK;
    }
  }
  *k_out = layers;
  return WS_OK;
}

int ws_catchup_stall_ms(int64_t weight_bytes, int32_t parallelism, int32_t layers,
                        double prefill_a_ms, double prefill_b_ms, int32_t layers_loaded,
                        double bandwidth, int32_t ref_input_tokens, double* stall_out) {
  if (layers_loaded >= layers) {
    *stall_out = 0.0;
    return WS_OK;
  }
  LayerTimes t;
  if (!layer_times(weight_bytes, parallelism, layers, prefill_a_ms, prefill_b_ms, bandwidth,
                   ref_input_tokens, &t))
    WS_FAIL(WS_ERR_INVALID, "invalid model spec");
  double worst = -INFINITY;
  for (int32_t l = layers_loaded + 1; l <= layers; ++l) {
    double lag = (double)(l - layers_loaded) * t.t_load - (double)(l - 1) * t.t_comp;
    if (lag > worst) worst = lag;
  }
  *stall_out = worst > 0.0 ? worst : 0.0;
  return WS_OK;
}

int ws_reservation_target(double m, int32_t c, int32_t r, double k, double* target_out) {
  if (r < 0 || r > c) WS_FAIL(WS_ERR_INVALID, "inflight %d outside [0, %d]", r, c);
  if (k < 0 || k > m) WS_FAIL(WS_ERR_INVALID, "kv_used %.17g outside [0, %.17g]", k, m);
  double expect = m * (double)r / (double)c;
  double buffer = k + m / (double)c;
  *target_out = expect >= buffer ? expect : buffer;
  return WS_OK;
}

int ws_partition_pages(int64_t weight_bytes, int32_t parallelism, int64_t page_size,
                       int64_t* partition_bytes_out, int64_t* partition_pages_out) {
  if (parallelism < 1 || page_size < 1 || weight_bytes < 1)
    WS_FAIL(WS_ERR_INVALID, "invalid partition arguments");
  int64_t part = weight_bytes / parallelism + (weight_bytes % parallelism ? 1 : 0);
  if (partition_bytes_out) *partition_bytes_out = part;
  if (partition_pages_out) *partition_pages_out = part / page_size + (part % page_size ? 1 : 0);
  return WS_OK;
}

int ws_pipelined_load(int64_t total_bytes, double bandwidth, double mu, int64_t chunk_pages,
                      int64_t page_size, ws_transfer_plan* out) {
  if (!(bandwidth > 0)) WS_FAIL(WS_ERR_INVALID, "bandwidth must be > 0");
  if (total_bytes <= 0) WS_FAIL(WS_ERR_INVALID, "total_bytes must be > 0");
  if (chunk_pages < 1) WS_FAIL(WS_ERR_INVALID, "chunk_pages must be >= 1");
  // memswitch.py:78-79 divides in float then ceils; keep that rounding path.
  int64_t pages = (int64_t)std::ceil((double)total_bytes / (double)page_size);
  int64_t n_chunks = (int64_t)std::ceil((double)pages / (double)chunk_pages);
  double mapped = 0.0, done = 0.0, first_map = 0.0;
  int64_t pages_before = 0, bytes_before = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    int64_t cp = c + 1 < n_chunks ? chunk_pages : pages - chunk_pages * (n_chunks - 1);
    int64_t end = (pages_before + cp) * page_size;
    if (end > total_bytes) end = total_bytes;
    double map_ms = (double)cp * mu;
    double copy_ms = (double)(end - bytes_before) / bandwidth;
    if (c == 0) first_map = map_ms;
    mapped += map_ms;  // maps run back to back on the map engine
    done = (mapped > done ? mapped : done) + copy_ms;  // copy c after map c and copy c-1
    pages_before += cp;
    bytes_before = end;
  }
  double stall = done - (double)total_bytes / bandwidth - first_map;
  out->total_bytes = total_bytes;
  out->bandwidth = bandwidth;
  out->chunk_pages = chunk_pages;
  out->page_size = page_size;
  out->n_chunks = n_chunks;
  out->first_chunk_map_ms = first_map;
  out->finish_ms = done;
  out->critical_path_stall_ms = stall > 0.0 ? stall : 0.0;
  return WS_OK;
}

int ws_background_kv_mapping(int64_t pages, double mu, double rate, double* stall_out) {
  if (pages < 0) WS_FAIL(WS_ERR_INVALID, "pages must be >= 0");
  if (!(mu > 0) || !(rate > 0)) WS_FAIL(WS_ERR_INVALID, "rates must be positive");
  double deficit = mu - 1.0 / rate;
  *stall_out = deficit > 0 ? (double)pages * deficit : 0.0;
  return WS_OK;
}

}  // extern "C"

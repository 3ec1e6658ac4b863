// kcache_api.cpp -- the reference's C++ operator API (include/kcache/*.hpp)
// implemented over the C ABI (include/kcache_c.h). Each method restates the
// reference's argument checks in the reference's order and rethrows the C
// status codes as the reference's exception types; the work itself runs in
// libkcache_b200.so's CUDA path -- there is no CPU compute path here.
#include <cstring>
#include <stdexcept>
#include <string>

#include "kcache/attention.hpp"
#include "kcache/b200.hpp"
#include "kcache/checked.hpp"
#include "kcache/errors.hpp"
#include "kcache/kv_cache.hpp"
#include "kcache/matrix.hpp"
#include "kcache/model.hpp"
#include "kcache_c.h"

namespace kcache {

namespace {

void check(int rc) {
  if (rc == KC_OK) return;
  const std::string msg = kc_last_error();
  switch (rc) {
    case KC_ESHAPE: throw ShapeError(msg);
    case KC_ESTATE: throw StateError(msg);
    case KC_ECAPACITY: throw CapacityError(msg);
    case KC_EARG: throw std::invalid_argument(msg);
    case KC_ERANGE: throw std::out_of_range(msg);
    case KC_EOVERFLOW: throw std::overflow_error(msg);
    default: throw std::runtime_error(msg);
  }
}


}  // namespace

// ---- model.hpp (model.cpp:13-53) -----------------------------------------
void ModelConfig::validate() const {
  if (n_layers == 0 || d_model == 0 || n_heads == 0 || head_dim == 0 || max_seq == 0) {
    throw ShapeError("ModelConfig: all counts must be >= 1");
  }
  if (ffn_hidden < 1) throw ShapeError("ModelConfig: ffn_hidden must be >= 1");
  if (vocab < 2) throw ShapeError("ModelConfig: vocab must be >= 2");
  if (d_model != n_heads * head_dim) {
    throw ShapeError("ModelConfig: d_model must equal n_heads * head_dim");
  }
}

std::size_t ModelConfig::default_ffn_hidden(std::size_t d) {
  const std::size_t eight_thirds = (8 * d + 2) / 3;
  return (eight_thirds + 15) / 16 * 16;
}

ModelConfig ModelConfig::toy() { return ModelConfig{4, 64, 4, 16, 176, 256, 4096}; }

ModelConfig ModelConfig::shape_7b() {
  return ModelConfig{32, 4096, 32, 128, default_ffn_hidden(4096), 32000, 32768};
}

std::uint64_t param_count(const ModelConfig& c) {
  const std::uint64_t d = c.d_model, f = c.ffn_hidden;
  const std::uint64_t layer = 2 * d + 4 * d * d + 3 * d * f;
  return checked_mul({c.vocab, d}) + checked_mul({c.n_layers, layer}) + d + checked_mul({d, c.vocab});
}

// ---- matrix.hpp ------------------------------------------------------------
std::vector<std::size_t> arg_topk(std::span<const float> values, std::size_t k) {
  if (k == 0) throw std::invalid_argument("arg_topk: k must be >= 1");
  std::vector<std::uint32_t> tmp(std::min(k, values.size()));
  std::uint64_t count = 0;
  check(kc_arg_topk(values.data(), values.size(), k, tmp.data(), &count));
  return std::vector<std::size_t>(tmp.begin(), tmp.begin() + count);
}

// ---- kv_cache.hpp ------------------------------------------------------------
const char* to_string(CacheMode mode) { return mode == CacheMode::baseline ? "baseline" : "kcache"; }
const char* to_string(TransferDir dir) { return dir == TransferDir::d2h ? "D2H" : "H2D"; }
const char* to_string(EnginePhase phase) {
  return phase == EnginePhase::prefill ? "prefill" : "decode";
}

void TransferLedger::record(EnginePhase phase, std::size_t layer, TransferDir dir,
                            std::uint64_t bytes, std::uint64_t elements) {
  events_.push_back({phase, layer, dir, bytes, elements});
  (dir == TransferDir::d2h ? d2h_bytes_ : h2d_bytes_) += bytes;
}

void TransferLedger::write_jsonl(std::ostream& out) const {
  for (const TransferEvent& e : events_) {
    out << "{\"phase\":\"" << to_string(e.phase) << "\",\"layer\":" << e.layer << ",\"dir\":\""
        << to_string(e.dir) << "\",\"bytes\":" << e.bytes << ",\"elements\":" << e.elements
        << "}\n";
  }
}

void TierPlacement::validate() const {
  if (resident_layers > n_layers) {
    throw ShapeError("TierPlacement: resident_layers must be <= n_layers");
  }
  if (bytes_per_element == 0) throw ShapeError("TierPlacement: bytes_per_element must be >= 1");
}

FootprintBytes memory_footprint(const ModelConfig& config, std::size_t batch, std::size_t seq_len,
                                CacheMode mode, std::size_t resident_layers,
                                std::size_t bytes_per_element) {
  const std::uint64_t per_layer = checked_mul({bytes_per_element, batch, seq_len, config.d_model});
  FootprintBytes fp;
  if (mode == CacheMode::baseline) {
    fp.fast_bytes = checked_mul({2, per_layer, config.n_layers});
  } else {
    if (resident_layers > config.n_layers) {
      throw ShapeError("memory_footprint: resident_layers > n_layers");
    }
    fp.fast_bytes = checked_mul({per_layer, config.n_layers + resident_layers});
    fp.slow_bytes = checked_mul({per_layer, config.n_layers - resident_layers});
  }
  fp.weight_bytes = checked_mul({param_count(config), bytes_per_element});
  return fp;
}

TieredKVCache::TieredKVCache(const ModelConfig& config, std::size_t batch, TierPlacement placement,
                             std::optional<std::uint64_t> fast_capacity_bytes, int device)
    : config_(config), batch_(batch), placement_(placement) {
  config_.validate();
  placement_.validate();
  if (placement_.n_layers != config_.n_layers) {
    throw ShapeError("TieredKVCache: placement layer count differs from config");
  }
  if (batch_ == 0) throw ShapeError("TieredKVCache: batch must be >= 1");
  const std::size_t kv = placement_.kv_heads(config_);
  if (kv == 0 || config_.n_heads % kv != 0) {
    throw ShapeError("TierPlacement: n_kv_heads must divide n_heads");
  }
  kc_config c{config_.n_layers, config_.d_model, config_.n_heads, kv, config_.head_dim, config_.max_seq};
  check(kc_cache_create(&c, batch_, placement_.resident_layers, placement_.bytes_per_element,
                        static_cast<int>(placement_.storage), fast_capacity_bytes.has_value() ? 1 : 0,
                        fast_capacity_bytes.value_or(0), device, -1, &handle_));
}

TieredKVCache::~TieredKVCache() {
  if (handle_) kc_cache_destroy(handle_);
}

TieredKVCache::TieredKVCache(TieredKVCache&& o) noexcept
    : config_(o.config_),
      batch_(o.batch_),
      placement_(o.placement_),
      handle_(o.handle_),
      ledger_(std::move(o.ledger_)),
      ledger_seen_(o.ledger_seen_) {
  o.handle_ = nullptr;
}

TieredKVCache& TieredKVCache::operator=(TieredKVCache&& o) noexcept {
  if (this != &o) {
    if (handle_) kc_cache_destroy(handle_);
    config_ = o.config_;
    batch_ = o.batch_;
    placement_ = o.placement_;
    handle_ = o.handle_;
    ledger_ = std::move(o.ledger_);
    ledger_seen_ = o.ledger_seen_;
    o.handle_ = nullptr;
  }
  return *this;
}

void TieredKVCache::sync_ledger() {
  std::uint64_t n = 0;
  check(kc_ledger_size(handle_, &n));
  for (; ledger_seen_ < n; ++ledger_seen_) {
    int phase = 0, dir = 0;
    std::uint64_t layer = 0, bytes = 0, elements = 0;
    check(kc_ledger_event(handle_, ledger_seen_, &phase, &layer, &dir, &bytes, &elements));
    ledger_.record(phase == KC_PREFILL ? EnginePhase::prefill : EnginePhase::decode, layer,
                   dir == KC_D2H ? TransferDir::d2h : TransferDir::h2d, bytes, elements);
  }
}

void TieredKVCache::append_kv(std::size_t layer, const Matrix& k_rows, const Matrix& v_rows) {
  if (layer >= config_.n_layers) {
    throw std::out_of_range("TieredKVCache: layer " + std::to_string(layer) + " out of range");
  }
  const std::size_t w = placement_.kv_heads(config_) * config_.head_dim;
  if (k_rows.cols != w || v_rows.cols != w) {
    throw ShapeError("append_kv: row width must equal d_model");
  }
  if (k_rows.rows != v_rows.rows || k_rows.rows == 0 || k_rows.rows % batch_ != 0) {
    throw ShapeError("append_kv: need a positive multiple of batch rows for K and V");
  }
  const int rc = kc_append_kv(handle_, layer, k_rows.data.data(), v_rows.data.data(), k_rows.rows);
  sync_ledger();
  check(rc);
}

void TieredKVCache::offload_prefill_v(std::size_t layer) {
  const int rc = kc_offload_prefill_v(handle_, layer);
  sync_ledger();
  check(rc);
}

void TieredKVCache::begin_decode() { check(kc_begin_decode(handle_)); }

GatheredV TieredKVCache::gather_v(std::size_t layer, const SelectionIndices& selection) {
  if (layer >= config_.n_layers) {
    throw std::out_of_range("TieredKVCache: layer " + std::to_string(layer) + " out of range");
  }
  if (selection.size() != batch_ * config_.n_heads) {
    throw ShapeError("gather_v: selection must cover batch * n_heads slots");
  }
  std::vector<std::uint64_t> counts(selection.size());
  std::vector<std::uint32_t> flat;
  for (std::size_t s = 0; s < selection.size(); ++s) {
    counts[s] = selection[s].size();
    flat.insert(flat.end(), selection[s].begin(), selection[s].end());
  }
  const std::size_t h = config_.head_dim;
  std::vector<float> rows(flat.size() * h);
  GatheredV out;
  out.head_dim = h;
  const int rc = kc_gather_v(handle_, layer, flat.data(), counts.data(), rows.data(), &out.h2d_bytes);
  sync_ledger();
  check(rc);
  out.blocks.resize(selection.size());
  std::size_t off = 0;
  for (std::size_t s = 0; s < selection.size(); ++s) {
    out.blocks[s].assign(rows.begin() + off * h, rows.begin() + (off + counts[s]) * h);
    off += counts[s];
  }
  return out;
}

std::span<const float> TieredKVCache::k_row(std::size_t layer, std::size_t pos,
                                            std::size_t batch_idx) const {
  row_stage_.resize(placement_.kv_heads(config_) * config_.head_dim);
  check(kc_read_row(handle_, layer, pos, batch_idx, 0, row_stage_.data()));
  return {row_stage_.data(), row_stage_.size()};
}

std::span<const float> TieredKVCache::v_row(std::size_t layer, std::size_t pos,
                                            std::size_t batch_idx) const {
  row_stage_.resize(placement_.kv_heads(config_) * config_.head_dim);
  check(kc_read_row(handle_, layer, pos, batch_idx, 1, row_stage_.data()));
  return {row_stage_.data(), row_stage_.size()};
}

std::size_t TieredKVCache::current_len() const {
  std::uint64_t len = 0;
  check(kc_current_len(handle_, &len));
  return len;
}

EnginePhase TieredKVCache::phase() const {
  int p = 0;
  check(kc_phase(handle_, &p));
  return p == KC_PREFILL ? EnginePhase::prefill : EnginePhase::decode;
}

std::uint64_t TieredKVCache::fast_bytes_used() const {
  std::uint64_t b = 0;
  check(kc_fast_bytes_used(handle_, &b));
  return b;
}

std::uint64_t TieredKVCache::slow_bytes_used() const {
  std::uint64_t b = 0;
  check(kc_slow_bytes_used(handle_, &b));
  return b;
}

// ---- attention.hpp -----------------------------------------------------------
namespace {

// check_decode_inputs (attention.cpp:80-87)
void check_decode_inputs(const Matrix& q, const TieredKVCache& cache) {
  if (q.rows != cache.batch() || q.cols != cache.config().d_model) {
    throw ShapeError("decode attention: q must be batch x d_model");
  }
  if (cache.current_len() == 0) throw StateError("decode attention: cache is empty");
}

void observe(const Matrix& q, const TieredKVCache& cache, std::size_t layer,
             const ScoreObserver& observer) {
  const std::size_t len = cache.current_len();
  const std::size_t slots = cache.batch() * cache.config().n_heads;
  std::vector<float> probs(slots * len);
  check(kc_score_probs(cache.handle(), layer, q.data.data(), KC_F32, probs.data()));
  for (std::size_t s = 0; s < slots; ++s) {
    observer(s / cache.config().n_heads, s % cache.config().n_heads,
             std::span<const float>(probs.data() + s * len, len));
  }
}

}  // namespace

Matrix decode_attention_full(const Matrix& q, const TieredKVCache& cache, std::size_t layer,
                             const ScoreObserver& observer) {
  check_decode_inputs(q, cache);
  if (observer) observe(q, cache, layer, observer);
  Matrix out(q.rows, q.cols);
  check(kc_decode_full(cache.handle(), layer, q.data.data(), KC_F32, 0, out.data.data(), nullptr));
  return out;
}

Matrix prefill_attention(const Matrix& q, const Matrix& k, const Matrix& v, std::size_t n_heads) {
  // attention.cpp:31-37
  if (!q.same_shape(k) || !q.same_shape(v)) throw ShapeError("prefill_attention: Q/K/V shapes differ");
  if (n_heads == 0 || q.cols % n_heads != 0) throw ShapeError("prefill_attention: cols must divide into heads");
  Matrix out(q.rows, q.cols);
  if (q.rows == 0) return out;
  check(kc_prefill_attention(q.data.data(), k.data.data(), v.data.data(), q.rows, n_heads, q.cols / n_heads,
                             out.data.data(), -1));
  return out;
}

namespace b200 {

Matrix decode_step_attention(const Matrix& q, const Matrix& k_rows, const Matrix& v_rows,
                             TieredKVCache& cache, std::size_t layer, bool use_topn,
                             std::size_t top_n, bool renormalize) {
  if (use_topn && top_n == 0) throw std::invalid_argument("decode_attention_topn: top_n must be >= 1");
  const std::size_t width = cache.placement().kv_heads(cache.config()) * cache.config().head_dim;
  if (k_rows.cols != width || v_rows.cols != width)
    throw ShapeError("append_kv: row width must equal d_model");
  if (k_rows.rows != cache.batch() || v_rows.rows != cache.batch())
    throw ShapeError("append_kv: need a positive multiple of batch rows for K and V");
  if (q.rows != cache.batch() || q.cols != cache.config().d_model)
    throw ShapeError("decode attention: q must be batch x d_model");
  Matrix out(q.rows, q.cols);
  const std::uint32_t flags = (renormalize ? KC_RENORMALIZE : 0u) | (use_topn ? 0u : KC_FULL);
  check(kc_decode_step(cache.handle(), layer, q.data.data(), k_rows.data.data(), v_rows.data.data(), KC_F32,
                       top_n, flags, out.data.data(), nullptr));
  return out;
}

DeviceStepStats read_step_stats(TieredKVCache& cache) {
  kc_step_stats s{};
  check(kc_step_stats_read(cache.handle(), &s, 1));
  DeviceStepStats out;
  out.h2d_bytes = s.h2d_bytes;
  out.d2h_bytes = s.d2h_bytes;
  out.mean_dropped_mass = s.selections ? s.dropped_sum / static_cast<double>(s.selections) : 0.0;
  for (std::size_t i = 0; i < kHistogramBins; ++i) out.position_histogram[i] = s.position_histogram[i];
  return out;
}

}  // namespace b200

TopNResult decode_attention_topn(const Matrix& q, TieredKVCache& cache, std::size_t layer,
                                 std::size_t top_n, bool renormalize, bool ordered_accumulation,
                                 const ScoreObserver& observer) {
  if (top_n == 0) throw std::invalid_argument("decode_attention_topn: top_n must be >= 1");
  check_decode_inputs(q, cache);
  if (observer) observe(q, cache, layer, observer);
  const std::size_t n = cache.config().n_heads;
  const std::size_t slots = cache.batch() * n;
  const std::size_t nc = std::min(top_n, cache.current_len());
  TopNResult res;
  res.out = Matrix(q.rows, q.cols);
  std::vector<std::uint32_t> idx(slots * nc);
  std::vector<float> w(slots * nc);
  res.selection.batch = cache.batch();
  res.selection.n_heads = n;
  res.selection.dropped_mass.resize(slots);
  kc_topn_out o{res.out.data.data(), idx.data(), w.data(), res.selection.dropped_mass.data(), 0, 0};
  std::uint32_t flags = 0;
  if (renormalize) flags |= KC_RENORMALIZE;
  if (!ordered_accumulation) flags |= KC_REVERSE_ACCUM;
  const int rc = kc_decode_topn(cache.handle(), layer, q.data.data(), KC_F32, top_n, flags, &o, nullptr);
  cache.sync_ledger();
  check(rc);
  res.h2d_bytes = o.h2d_bytes;
  res.selection.indices.resize(slots);
  res.selection.weights.resize(slots);
  for (std::size_t s = 0; s < slots; ++s) {
    res.selection.indices[s].assign(idx.begin() + s * nc, idx.begin() + (s + 1) * nc);
    res.selection.weights[s].assign(w.begin() + s * nc, w.begin() + (s + 1) * nc);
  }
  return res;
}

}  // namespace kcache

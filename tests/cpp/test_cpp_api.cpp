// test_cpp_api.cpp -- the reference's C++ operator API, used the way the
// reference's own tests and Engine use it, compiled against include/kcache/
// and linked to libkcache_b200.so. Proves source compatibility of the
// drop-in: this file would compile against the
// reference headers too (except engine_step_cases: kcache/b200.hpp).
// Cases restate proj/tests/test_attention.cpp and test_kv_cache.cpp.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "kcache/attention.hpp"
#include "kcache/b200.hpp"
#include "kcache/errors.hpp"
#include "kcache/kv_cache.hpp"
#include "kcache/matrix.hpp"
#include "kcache/model.hpp"
#include "kcache/rng.hpp"

using namespace kcache;

static int g_fail = 0;
#define CHECK(x)                                                    \
  do {                                                              \
    if (!(x)) {                                                     \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #x);      \
      ++g_fail;                                                     \
    }                                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                    \
  do {                                                              \
    bool ok_ = false;                                               \
    try {                                                           \
      (void)(expr);                                                 \
    } catch (const T&) {                                            \
      ok_ = true;                                                   \
    } catch (...) {                                                 \
    }                                                               \
    if (!ok_) {                                                     \
      std::printf("FAIL %s:%d  %s !throw %s\n", __FILE__, __LINE__, #expr, #T); \
      ++g_fail;                                                     \
    }                                                               \
  } while (0)

static ModelConfig small_config(std::size_t layers, std::size_t d, std::size_t heads) {
  ModelConfig c;
  c.n_layers = layers;
  c.d_model = d;
  c.n_heads = heads;
  c.head_dim = d / heads;
  c.ffn_hidden = ModelConfig::default_ffn_hidden(d);
  c.vocab = 64;
  c.max_seq = 8192;
  return c;
}

static Matrix random_matrix(std::size_t rows, std::size_t cols, SeededRng& rng, float lo = -1.0f,
                            float hi = 1.0f) {
  Matrix m(rows, cols);
  for (float& v : m.data) v = rng.next_uniform(lo, hi);
  return m;
}

static TieredKVCache make_cache(const ModelConfig& c, std::size_t batch, std::size_t resident,
                                const Matrix& k, const Matrix& v) {
  TierPlacement pl = TierPlacement::kcache(resident, c.n_layers);
  TieredKVCache cache(c, batch, pl);
  for (std::size_t layer = 0; layer < c.n_layers; ++layer) {
    cache.append_kv(layer, k, v);
    cache.offload_prefill_v(layer);
  }
  cache.begin_decode();
  return cache;
}

static void hand_checkable() {
  ModelConfig c = small_config(1, 1, 1);
  c.ffn_hidden = 4;
  Matrix k(4, 1);
  k.data = {std::log(0.1f), std::log(0.4f), std::log(0.2f), std::log(0.3f)};
  Matrix v(4, 1);
  v.data = {10.0f, 20.0f, 30.0f, 40.0f};
  TieredKVCache cache = make_cache(c, 1, 0, k, v);
  Matrix q(1, 1);
  q.data = {1.0f};
  TopNResult r = decode_attention_topn(q, cache, 0, 2, false);
  CHECK(r.selection.indices[0].size() == 2);
  CHECK(r.selection.indices[0][0] == 1 && r.selection.indices[0][1] == 3);
  CHECK(std::fabs(r.selection.weights[0][0] - 0.4f) < 1e-5f);
  CHECK(std::fabs(r.selection.dropped_mass[0] - 0.3) < 1e-5);
  CHECK(std::fabs(r.out.at(0, 0) - 20.0f) < 2e-3f);
  TopNResult rn = decode_attention_topn(q, cache, 0, 2, true);
  CHECK(std::fabs(rn.out.at(0, 0) - 20.0f / 0.7f) < 3e-3f);
}

static void topn_equals_full() {
  const ModelConfig c = small_config(3, 64, 4);
  SeededRng rng(3);
  const std::size_t s = 24, batch = 2;
  const Matrix k = random_matrix(s * batch, c.d_model, rng);
  const Matrix v = random_matrix(s * batch, c.d_model, rng);
  TieredKVCache cache = make_cache(c, batch, 1, k, v);
  const Matrix q = random_matrix(batch, c.d_model, rng);
  for (std::size_t layer = 0; layer < c.n_layers; ++layer) {
    const Matrix full = decode_attention_full(q, cache, layer);
    for (std::size_t n : {s, s + 10, std::size_t{4096}}) {
      TopNResult r = decode_attention_topn(q, cache, layer, n, false);
      for (std::size_t i = 0; i < full.data.size(); ++i)
        CHECK(std::fabs(full.data[i] - r.out.data[i]) <= 1e-6f + 1e-5f * std::fabs(full.data[i]));
      for (std::size_t slot = 0; slot < r.selection.indices.size(); ++slot) {
        CHECK(r.selection.indices[slot].size() == s);
        CHECK(std::fabs(r.selection.dropped_mass[slot]) <= 1e-6);
        for (std::uint32_t i = 0; i < s; ++i) CHECK(r.selection.indices[slot][i] == i);
      }
    }
  }
}

static void h2d_accounting_and_errors() {
  const ModelConfig c = small_config(2, 64, 4);
  SeededRng rng(6);
  const std::size_t s = 10;
  const Matrix k = random_matrix(s, c.d_model, rng);
  const Matrix v = random_matrix(s, c.d_model, rng);
  TieredKVCache cache = make_cache(c, 1, 1, k, v);
  const Matrix q = random_matrix(1, c.d_model, rng);
  TopNResult off = decode_attention_topn(q, cache, 1, 64, false);
  CHECK(off.h2d_bytes == 2ull * 1 * c.n_heads * s * c.head_dim);
  TopNResult off4 = decode_attention_topn(q, cache, 1, 4, false);
  CHECK(off4.h2d_bytes == 2ull * 1 * c.n_heads * 4 * c.head_dim);
  TopNResult res = decode_attention_topn(q, cache, 0, 4, false);
  CHECK(res.h2d_bytes == 0);
  CHECK(cache.h2d_bytes_total() == off.h2d_bytes + off4.h2d_bytes);
  CHECK_THROWS_AS(decode_attention_topn(q, cache, 0, 0, false), std::invalid_argument);
  CHECK_THROWS_AS(decode_attention_topn(Matrix(2, c.d_model), cache, 0, 4, false), ShapeError);
  TieredKVCache empty(c, 1, TierPlacement::kcache(0, c.n_layers));
  CHECK_THROWS_AS(decode_attention_full(q, empty, 0), StateError);
}

static void kv_cache_cases() {
  const ModelConfig c = small_config(1, 32, 4);
  TieredKVCache cache(c, 1, TierPlacement::kcache(0, c.n_layers));
  SeededRng rng(12);
  cache.append_kv(0, random_matrix(2, 32, rng), random_matrix(2, 32, rng));
  cache.offload_prefill_v(0);
  std::ostringstream out;
  cache.ledger().write_jsonl(out);
  CHECK(out.str() == "{\"phase\":\"prefill\",\"layer\":0,\"dir\":\"D2H\",\"bytes\":128,\"elements\":64}\n");
  CHECK_THROWS_AS(cache.offload_prefill_v(0), StateError);
  CHECK_THROWS_AS(cache.append_kv(3, random_matrix(1, 32, rng), random_matrix(1, 32, rng)), std::out_of_range);
  CHECK_THROWS_AS(cache.append_kv(0, random_matrix(1, 16, rng), random_matrix(1, 32, rng)), ShapeError);

  const ModelConfig c2 = small_config(2, 64, 4);
  TieredKVCache capped(c2, 1, TierPlacement::kcache(2, c2.n_layers), 4096);
  capped.append_kv(0, random_matrix(8, 64, rng), random_matrix(8, 64, rng));
  CHECK_THROWS_AS(capped.append_kv(1, random_matrix(16, 64, rng), random_matrix(16, 64, rng)), CapacityError);

  const ModelConfig c7 = ModelConfig::shape_7b();
  const FootprintBytes fp = memory_footprint(c7, 8, 32768, CacheMode::baseline, 0, 2);
  CHECK(fp.fast_bytes == 137438953472ull);
  CHECK(memory_footprint(c7, 8, 32768, CacheMode::kcache, 2, 2).fast_bytes == 73014444032ull);

  // gather rows are returned bitwise (fp32 storage)
  const ModelConfig c3 = small_config(1, 64, 4);
  // (fp32 is the default storage: TierPlacement as the reference builds it)
  TieredKVCache g(c3, 2, TierPlacement::kcache(0, c3.n_layers));
  const Matrix k = random_matrix(40, 64, rng);
  const Matrix v = random_matrix(40, 64, rng);
  g.append_kv(0, k, v);
  g.offload_prefill_v(0);
  g.begin_decode();
  SelectionIndices sel(8, std::vector<std::uint32_t>{1, 7, 19});
  const GatheredV got = g.gather_v(0, sel);
  for (std::size_t b = 0; b < 2; ++b)
    for (std::size_t head = 0; head < 4; ++head)
      for (std::size_t r = 0; r < 3; ++r)
        for (std::size_t t = 0; t < 16; ++t)
          CHECK(got.blocks[b * 4 + head][r * 16 + t] == v.at(sel[0][r] * 2 + b, head * 16 + t));
  CHECK(got.h2d_bytes == 2ull * 8 * 3 * 16);
  CHECK(g.ledger().events().size() == 2);
  const auto kr = g.k_row(0, 5, 1);
  for (std::size_t t = 0; t < 64; ++t) CHECK(kr[t] == k.at(5 * 2 + 1, t));
}

static void arg_topk_cases() {
  std::vector<float> vals = {0.1f, 0.4f, 0.2f, 0.3f};
  CHECK(arg_topk(vals, 2) == (std::vector<std::size_t>{1, 3}));
  CHECK(arg_topk(vals, 9) == (std::vector<std::size_t>{0, 1, 2, 3}));
  std::vector<float> ties = {0.5f, 0.5f, 0.1f};
  CHECK(arg_topk(ties, 1) == (std::vector<std::size_t>{0}));
  CHECK_THROWS_AS(arg_topk(vals, 0), std::invalid_argument);
}

// Engine::forward_decode's attention block (engine.cpp:139-160) as one call:
// append + TopN/full + StepStats; the output equals a separate
// append_kv + decode_attention_topn on an identical cache.
static void engine_step_cases() {
  const ModelConfig c = small_config(2, 64, 4);
  SeededRng rng(21);
  const std::size_t s = 40, batch = 2, N = 8;
  const Matrix k = random_matrix(s * batch, c.d_model, rng);
  const Matrix v = random_matrix(s * batch, c.d_model, rng);
  TieredKVCache a = make_cache(c, batch, 1, k, v);
  TieredKVCache b = make_cache(c, batch, 1, k, v);
  b200::read_step_stats(a);
  for (std::size_t layer = 0; layer < c.n_layers; ++layer) {
    const Matrix kr = random_matrix(batch, c.d_model, rng);
    const Matrix vr = random_matrix(batch, c.d_model, rng);
    const Matrix q = random_matrix(batch, c.d_model, rng);
    const bool topn = layer >= 1;
    const Matrix got = b200::decode_step_attention(q, kr, vr, a, layer, topn, N, false);
    b.append_kv(layer, kr, vr);
    if (topn) {
      const TopNResult want = decode_attention_topn(q, b, layer, N, false);
      CHECK(got.data == want.out.data);
    } else {
      CHECK(got.data == decode_attention_full(q, b, layer).data);
    }
  }
  const b200::DeviceStepStats st = b200::read_step_stats(a);
  CHECK(st.h2d_bytes == 2ull * batch * c.n_heads * N * c.head_dim);
  CHECK(st.d2h_bytes == 2ull * batch * c.d_model);  // layer 1's new V row goes to the slow tier
  std::uint64_t total = 0;
  for (auto x : st.position_histogram) total += x;
  CHECK(total == batch * c.n_heads * N);
  CHECK(st.mean_dropped_mass > 0.0 && st.mean_dropped_mass < 1.0);
  CHECK(a.current_len() == s + 1);
  CHECK_THROWS_AS(b200::decode_step_attention(random_matrix(batch, c.d_model, rng), random_matrix(batch, 16, rng),
                                              random_matrix(batch, c.d_model, rng), a, 0, true, N, false),
                  ShapeError);
}

int main() {
  hand_checkable();
  engine_step_cases();
  topn_equals_full();
  h2d_accounting_and_errors();
  kv_cache_cases();
  arg_topk_cases();
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}

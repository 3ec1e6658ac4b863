// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library, so Python tests and
// bench.py can drive the reference's own decode_attention_topn /
// decode_attention_full / arg_topk / TieredKVCache
// (proj/core/include/kcache/{attention,kv_cache,matrix}.hpp). It is compiled
// together with the reference's own sources (proj/core/src/{matrix,model,
// kv_cache,attention}.cpp, read in place from /root/reference) by
// oracle/Makefile into oracle/_ref/libkcache_ref.so. No reference source is
// copied into this repository.
//
// Uses: tests/golden/make_golden.py (golden vectors), tests (oracle pinning)
// and bench.py --impl reference / cpu_baseline (the reference timed on the
// host cores).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "kcache/attention.hpp"
#include "kcache/errors.hpp"
#include "kcache/kv_cache.hpp"
#include "kcache/matrix.hpp"
#include "kcache/model.hpp"
#include "kcache/rng.hpp"

using namespace kcache;

namespace {

thread_local std::string g_err;

int map_exception() {
  try {
    throw;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const StateError& e) {
    g_err = e.what();
    return 2;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 4;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

ModelConfig make_config(std::size_t n_layers, std::size_t n_heads, std::size_t h,
                        std::size_t max_seq) {
  ModelConfig c;
  c.n_layers = n_layers;
  c.d_model = n_heads * h;
  c.n_heads = n_heads;
  c.head_dim = h;
  c.ffn_hidden = ModelConfig::default_ffn_hidden(c.d_model);
  c.vocab = 64;
  c.max_seq = max_seq;
  return c;
}

Matrix from_ptr(std::size_t rows, std::size_t cols, const float* p) {
  Matrix m(rows, cols);
  std::memcpy(m.data.data(), p, rows * cols * sizeof(float));
  return m;
}

uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Same element stream as SeededRng::next_uniform (rng.hpp:22-26), rounded to
// fp16 like the GPU's storage.
float synth_f16(uint64_t seed, uint64_t i, float lo, float hi) {
  const double u = static_cast<double>(splitmix_at(seed, i) >> 11) * 0x1.0p-53;
  const float x = lo + static_cast<float>(u) * (hi - lo);
  return static_cast<float>(static_cast<_Float16>(x));
}

}  // namespace

extern "C" {

const char* kcref_last_error() { return g_err.c_str(); }

// One layer, `batch` rows, cache length s; k/v are [s*batch][n_heads*h]
// position-major. resident=1 keeps V in the fast tier (no ledger charge).
int kcref_decode_topn(std::size_t batch, std::size_t n_heads, std::size_t h, std::size_t s,
                      const float* q, const float* k, const float* v, std::size_t top_n,
                      int renormalize, int ordered, int resident, float* out, uint32_t* idx,
                      float* w, double* dropped, uint64_t* h2d, uint64_t* ledger_h2d_total) {
  try {
    const ModelConfig c = make_config(1, n_heads, h, s > 0 ? s : 1);
    TieredKVCache cache(c, batch, TierPlacement::kcache(resident ? 1 : 0, 1));
    if (s > 0) {
      cache.append_kv(0, from_ptr(s * batch, c.d_model, k), from_ptr(s * batch, c.d_model, v));
    }
    cache.offload_prefill_v(0);
    cache.begin_decode();
    const Matrix qm = from_ptr(batch, c.d_model, q);
    TopNResult r = decode_attention_topn(qm, cache, 0, top_n, renormalize != 0, ordered != 0);
    std::memcpy(out, r.out.data.data(), r.out.data.size() * sizeof(float));
    std::size_t off = 0;
    for (std::size_t slot = 0; slot < r.selection.indices.size(); ++slot) {
      const auto& ix = r.selection.indices[slot];
      const auto& wx = r.selection.weights[slot];
      std::memcpy(idx + off, ix.data(), ix.size() * sizeof(uint32_t));
      std::memcpy(w + off, wx.data(), wx.size() * sizeof(float));
      dropped[slot] = r.selection.dropped_mass[slot];
      off += ix.size();
    }
    *h2d = r.h2d_bytes;
    *ledger_h2d_total = cache.h2d_bytes_total();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int kcref_decode_full(std::size_t batch, std::size_t n_heads, std::size_t h, std::size_t s,
                      const float* q, const float* k, const float* v, int resident, float* out) {
  try {
    const ModelConfig c = make_config(1, n_heads, h, s > 0 ? s : 1);
    TieredKVCache cache(c, batch, TierPlacement::kcache(resident ? 1 : 0, 1));
    if (s > 0) {
      cache.append_kv(0, from_ptr(s * batch, c.d_model, k), from_ptr(s * batch, c.d_model, v));
    }
    cache.offload_prefill_v(0);
    cache.begin_decode();
    const Matrix r = decode_attention_full(from_ptr(batch, c.d_model, q), cache, 0);
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// prefill_attention (attention.cpp:31-62): one sequence, [s][n_heads*h].
int kcref_prefill(std::size_t s, std::size_t n_heads, std::size_t h, const float* q, const float* k,
                  const float* v, float* out) {
  try {
    const std::size_t d = n_heads * h;
    const Matrix r = prefill_attention(from_ptr(s, d, q), from_ptr(s, d, k), from_ptr(s, d, v), n_heads);
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// arg_topk (matrix.cpp:109-122). Returns the count, or -(error code).
long kcref_arg_topk(const float* values, std::size_t n, std::size_t k, uint32_t* out) {
  try {
    const auto r = arg_topk({values, n}, k);
    for (std::size_t i = 0; i < r.size(); ++i) out[i] = static_cast<uint32_t>(r[i]);
    return static_cast<long>(r.size());
  } catch (...) {
    return -map_exception();
  }
}

void kcref_softmax(float* row, std::size_t n) { softmax_inplace({row, n}); }

// The first n draws of SeededRng(seed).next_uniform(lo, hi) (rng.hpp:22-26):
// pins the counter-indexed generators of the oracle and the GPU.
void kcref_rng_uniform(uint64_t seed, std::size_t n, float lo, float hi, float* out) {
  SeededRng rng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_uniform(lo, hi);
}

// ---------------------------------------------------------------------------
// Timed CPU baseline: the reference decode_attention_topn over a sample of the
// bench workload, on all host threads. A shard is (batch row, head group):
// its own TieredKVCache(batch=1, one layer) because the cache is single-owner
// (SPEC.md:271). Inputs are the same SplitMix64 fp16-rounded synthetic
// tensors the GPU arm uses (K seed, V seed, q seed; element index
// (pos*B + b)*D + col like append_kv rows).
struct KcrefBench {
  std::vector<std::unique_ptr<TieredKVCache>> caches;
  std::vector<Matrix> qs;
  std::size_t top_n = 0;
  int renormalize = 0;
  unsigned threads = 1;
};

// n_layers q sets (seed_q + 100*layer, the GPU bench's q seeds) against one
// layer's cache: one run = decode_attention_topn of every layer for every
// (row, head-group) shard -- a whole decode step's work, timed as such.
void* kcref_bench_create(std::size_t s, std::size_t batch, std::size_t n_heads, std::size_t h,
                         std::size_t heads_per_shard, std::size_t top_n, int renormalize,
                         unsigned threads, uint64_t seed_q, uint64_t seed_k, uint64_t seed_v,
                         std::size_t n_layers) {
  try {
    if (heads_per_shard == 0 || n_heads % heads_per_shard != 0) {
      throw ShapeError("heads_per_shard must divide n_heads");
    }
    auto* bench = new KcrefBench;
    bench->top_n = top_n;
    bench->renormalize = renormalize;
    bench->threads = threads ? threads : 1;
    const std::size_t D = n_heads * h;
    const std::size_t groups = n_heads / heads_per_shard;
    const std::size_t n_shards = batch * groups;
    const ModelConfig c = make_config(1, heads_per_shard, h, s);
    bench->caches.resize(n_shards);
    const std::size_t n_sets = n_layers ? n_layers : 1;
    bench->qs.resize(n_sets * n_shards);
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < bench->threads; ++t) {
      pool.emplace_back([&] {
        for (std::size_t sh = next++; sh < n_shards; sh = next++) {
          const std::size_t b = sh / groups, grp = sh % groups;
          const std::size_t col0 = grp * heads_per_shard * h;
          Matrix km(s, c.d_model), vm(s, c.d_model);
          for (std::size_t pos = 0; pos < s; ++pos) {
            const uint64_t base = (pos * batch + b) * D + col0;
            for (std::size_t col = 0; col < c.d_model; ++col) {
              km.data[pos * c.d_model + col] = synth_f16(seed_k, base + col, -1.0f, 1.0f);
              vm.data[pos * c.d_model + col] = synth_f16(seed_v, base + col, -1.0f, 1.0f);
            }
          }
          for (std::size_t l = 0; l < n_sets; ++l) {
            Matrix ql(1, c.d_model);
            for (std::size_t col = 0; col < c.d_model; ++col) {
              ql.data[col] = synth_f16(seed_q + 100 * l, b * D + col0 + col, -1.0f, 1.0f);
            }
            bench->qs[l * n_shards + sh] = std::move(ql);
          }
          auto cache = std::make_unique<TieredKVCache>(c, 1, TierPlacement::kcache(0, 1));
          cache->append_kv(0, km, vm);
          cache->offload_prefill_v(0);
          cache->begin_decode();
          bench->caches[sh] = std::move(cache);
        }
      });
    }
    for (auto& th : pool) th.join();
    return bench;
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

// One pass over every (q set, shard); returns wall seconds of the decode
// calls only.
double kcref_bench_run(void* handle, double* checksum) {
  auto* bench = static_cast<KcrefBench*>(handle);
  const std::size_t n = bench->qs.size();
  const std::size_t n_shards = bench->caches.size();
  std::vector<double> sums(n, 0.0);
  std::atomic<std::size_t> next{0};
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < bench->threads; ++t) {
    pool.emplace_back([&] {
      for (std::size_t sh = next++; sh < n; sh = next++) {
        TopNResult r = decode_attention_topn(bench->qs[sh], *bench->caches[sh % n_shards], 0, bench->top_n,
                                             bench->renormalize != 0);
        double acc = 0.0;
        for (float x : r.out.data) acc += x;
        sums[sh] = acc;
      }
    });
  }
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  double total = 0.0;
  for (double x : sums) total += x;
  if (checksum) *checksum = total;
  return std::chrono::duration<double>(t1 - t0).count();
}

void kcref_bench_destroy(void* handle) { delete static_cast<KcrefBench*>(handle); }

}  // extern "C"

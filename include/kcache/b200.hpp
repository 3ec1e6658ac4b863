// b200.hpp -- B200-only additions to the C++ operator API. Nothing here is
// part of the reference's surface, so the reference's own headers
// (engine.hpp's StepStats, ...) never collide with it.
//
// Engine::forward_decode (proj/core/src/engine.cpp:124-165) does, per layer:
// append this step's K/V rows, TopN (offloaded layers) or full attention, and
// the StepStats bookkeeping of engine.cpp:146-159. decode_step_attention is
// that block as one library call; its statistics accumulate on the device and
// are read once per step with read_step_stats.
#pragma once

#include <array>
#include <cstdint>

#include "kcache/attention.hpp"
#include "kcache/kv_cache.hpp"
#include "kcache/matrix.hpp"

namespace kcache::b200 {

inline constexpr std::size_t kHistogramBins = 8;  // engine.hpp:35

// Same fields and meaning as the reference's StepStats (engine.hpp:37-45).
struct DeviceStepStats {
  std::uint64_t h2d_bytes = 0;
  std::uint64_t d2h_bytes = 0;
  double mean_dropped_mass = 0.0;
  std::array<std::uint64_t, kHistogramBins> position_histogram{};
};

// k_rows / v_rows: batch x (kv_heads * head_dim), q: batch x d_model.
Matrix decode_step_attention(const Matrix& q, const Matrix& k_rows, const Matrix& v_rows,
                             TieredKVCache& cache, std::size_t layer, bool use_topn,
                             std::size_t top_n, bool renormalize);

// Statistics of the decode_step_attention calls since the previous read.
DeviceStepStats read_step_stats(TieredKVCache& cache);

}  // namespace kcache::b200

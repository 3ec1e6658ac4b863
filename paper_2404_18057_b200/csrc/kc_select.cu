// kc_select.cu -- per-(batch, kv-head) top-N selection (sm_100a).
//
// Replaces the softmax normalisation (proj/core/src/matrix.cpp:45-61),
// arg_topk (proj/core/src/matrix.cpp:109-122) and the TopNSelection fill
// loop (proj/core/src/attention.cpp:126-154).
//
// One 1024-thread CTA per (batch, kv head):
//   1. global softmax stats per q head from the scoring kernel's per-split
//      (max, sum exp): M = max m_i, Z = sum_i l_i exp(m_i - M) (ascending i);
//   2. key_j = fp32 bits of p_j = exp(s_j - M) / Z -- the reference ranks the
//      fp32 PROBABILITIES (attention.cpp:140), so equal probabilities tie even
//      when logits differ; for GQA key_j = sum_g p_g[j]. p >= 0,
//      so the raw bits order like the values;
//   3. MSB-first radix select (11/11/10-bit digits, shared-memory histograms
//      with warp-aggregated atomics) finds the N-th largest key T and how many
//      of the keys equal to T to keep;
//   4. ordered compaction (per-warp contiguous segments, ballot ranks) keeps
//      every key > T and the LOWEST-index keys == T -- exactly
//      stable_sort(desc) + resize(N) -- and emits the survivors already in
//      ascending position order (the reference's final std::sort);
//   5. weights p_g[idx], dropped = 1 - sum double(p) (ascending order, as
//      attention.cpp:146-152) and the fp32 renormaliser 1/sum p
//      (attention.cpp:167-174), each summed sequentially like the reference.
#include "kc_device.cuh"
#include "kc_kernels.cuh"

namespace kc {

namespace {

constexpr int kT = 1024;
constexpr int kNW = kT / 32;
constexpr int kBins = 2048;
constexpr int kMaxG = 32;

struct SelShared {
  uint32_t hist[kBins];
  uint32_t wa[kNW], wb[kNW], wc[kNW], wd[kNW];
  float M[kMaxG], Z[kMaxG];
  uint32_t bin, need;
};

__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool active, int lane) {
  const uint32_t key = active ? bin : 0xffffffffu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int leader = __ffs(peers) - 1;
  if (active && lane == leader) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

// Among the bins, find B with (count above B) < need <= (count at or above B).
// Leaves S.bin = B and S.need = need - (count above B).
__device__ void find_bin(SelShared& S, uint32_t need) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t h0 = S.hist[2 * t], h1 = S.hist[2 * t + 1];
  const uint32_t local = h0 + h1;
  uint32_t v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v += n;
  }
  if (lane == 0) S.wa[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const uint32_t own = S.wa[lane];
    uint32_t x = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_down_sync(0xffffffffu, x, o);
      if (lane + o < 32) x += n;
    }
    S.wb[lane] = x - own;  // sum over later warps
  }
  __syncthreads();
  const uint32_t above = S.wb[warp] + (v - local);  // bins of later threads
  if (above < need && above + h1 >= need) {
    S.bin = 2 * t + 1;
    S.need = need - above;
  } else if (above + h1 < need && above + h1 + h0 >= need) {
    S.bin = 2 * t;
    S.need = need - (above + h1);
  }
  __syncthreads();
}

__device__ __forceinline__ void clear_hist(SelShared& S) {
  for (int i = threadIdx.x; i < kBins; i += kT) S.hist[i] = 0;
  __syncthreads();
}

// keys[0..s) (already written, visible to the block) -> idx[0..nc) ascending.
__device__ void radix_compact(SelShared& S, const uint32_t* keys, int s, int nc, uint32_t* idx) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t T = 0, k_eq = (uint32_t)nc;
  if (nc < s) {
    // digit 0: bits 31..21
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      const bool act = j < s;
      const uint32_t k = act ? keys[j] : 0u;
      hist_add(S.hist, k >> 21, act, lane);
    }
    __syncthreads();
    find_bin(S, (uint32_t)nc);
    const uint32_t b0 = S.bin;
    uint32_t need = S.need;
    // digit 1: bits 20..10
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < s ? keys[j] : 0u;
      const bool act = j < s && (k >> 21) == b0;
      hist_add(S.hist, (k >> 10) & 0x7ffu, act, lane);
    }
    __syncthreads();
    find_bin(S, need);
    const uint32_t p01 = (b0 << 11) | S.bin;
    need = S.need;
    // digit 2: bits 9..0
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < s ? keys[j] : 0u;
      const bool act = j < s && (k >> 10) == p01;
      hist_add(S.hist, k & 0x3ffu, act, lane);
    }
    __syncthreads();
    find_bin(S, need);
    T = (p01 << 10) | S.bin;
    k_eq = S.need;
  }

  // ordered compaction: keys > T, plus the first k_eq keys == T by position
  const int seg = (((s + kNW - 1) / kNW) + 31) & ~31;
  const int w0 = warp * seg;
  const int w1 = min(s, w0 + seg);
  uint32_t cgt = 0, ceq = 0;
  for (int j0 = w0; j0 < w1; j0 += 32) {
    const int j = j0 + lane;
    const bool act = j < w1;
    const uint32_t k = act ? keys[j] : 0u;
    cgt += __popc(__ballot_sync(0xffffffffu, act && k > T));
    ceq += __popc(__ballot_sync(0xffffffffu, act && k == T));
  }
  if (lane == 0) {
    S.wa[warp] = cgt;
    S.wb[warp] = ceq;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t gt = S.wa[lane], eq = S.wb[lane];
    uint32_t x = eq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += n;
    }
    const uint32_t eq_excl = x - eq;
    const uint32_t take = eq_excl >= k_eq ? 0u : min(eq, k_eq - eq_excl);
    const uint32_t sel = gt + take;
    uint32_t y = sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += n;
    }
    S.wc[lane] = eq_excl;
    S.wd[lane] = y - sel;
  }
  __syncthreads();
  uint32_t run_eq = S.wc[warp], run_sel = S.wd[warp];
  const uint32_t lt = lanemask_lt();
  for (int j0 = w0; j0 < w1; j0 += 32) {
    const int j = j0 + lane;
    const bool act = j < w1;
    const uint32_t k = act ? keys[j] : 0u;
    const bool is_eq = act && k == T;
    const uint32_t beq = __ballot_sync(0xffffffffu, is_eq);
    const uint32_t eqr = run_eq + __popc(beq & lt);
    const bool sel = (act && k > T) || (is_eq && eqr < k_eq);
    const uint32_t bsel = __ballot_sync(0xffffffffu, sel);
    if (sel) idx[run_sel + __popc(bsel & lt)] = (uint32_t)j;
    run_eq += __popc(beq);
    run_sel += __popc(bsel);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kT) select_kernel(const SelectParams p) {
  __shared__ SelShared S;
  const int row = blockIdx.x;
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int G = p.G;
  const int n_q = p.n_kv * G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* lbase = p.logits + ((size_t)b * n_q + kvh * G) * p.lstride;
  uint32_t* keys = p.keys + (size_t)row * p.kstride;
  uint32_t* idx = p.idx + (size_t)row * p.nc;

  // 1. global softmax stats per q head of the group
  for (int g = warp; g < G; g += kNW) {
    const float2* part = p.partials + ((size_t)b * n_q + kvh * G + g) * p.max_splits;
    float m = -INFINITY;
    for (int i = lane; i < p.n_splits; i += 32) m = fmaxf(m, part[i].x);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      float z = 0.0f;
      for (int i = 0; i < p.n_splits; ++i) {
        const float2 ml = part[i];
        if (ml.y > 0.0f) z += ml.y * expf(ml.x - m);
      }
      S.M[g] = m;
      S.Z[g] = z;
    }
  }
  __syncthreads();

  // 2. keys
  for (int j = tid; j < p.s; j += kT) {
    float acc = 0.0f;
    for (int g = 0; g < G; ++g) {
      const float pg = expf(lbase[(size_t)g * p.lstride + j] - S.M[g]) / S.Z[g];
      acc = (g == 0) ? pg : acc + pg;
    }
    keys[j] = __float_as_uint(acc);
  }
  __syncthreads();

  // 3-4. select
  radix_compact(S, keys, p.s, p.nc, idx);

  // 5. weights, dropped mass, renormaliser
  for (int r = tid; r < p.nc; r += kT) {
    const uint32_t j = idx[r];
    for (int g = 0; g < G; ++g) {
      const float pg = expf(lbase[(size_t)g * p.lstride + j] - S.M[g]) / S.Z[g];
      p.w[((size_t)b * n_q + kvh * G + g) * p.nc + r] = pg;
    }
  }
  __syncthreads();
  for (int g = tid; g < G; g += kT) {
    const size_t slot = (size_t)b * n_q + kvh * G + g;
    const float* wg = p.w + slot * p.nc;
    double mass = 0.0;
    float sum = 0.0f;
    for (int r = 0; r < p.nc; ++r) {
      const float x = wg[r];
      mass += (double)x;
      sum += x;
    }
    p.dropped[slot] = 1.0 - mass;
    p.norm[slot] = sum > 0.0f ? 1.0f / sum : 1.0f;
  }
}

__global__ void __launch_bounds__(kT)
    arg_topk_kernel(const float* values, int n, int nc, uint32_t* keys, uint32_t* out) {
  __shared__ SelShared S;
  for (int j = threadIdx.x; j < n; j += kT) {
    const uint32_t u = __float_as_uint(values[j]);
    keys[j] = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  }
  __syncthreads();
  radix_compact(S, keys, n, nc, out);
}

__global__ void __launch_bounds__(256) probs_kernel(const SelectParams p, float* probs) {
  __shared__ float sMZ[2];
  const int slot = blockIdx.x;  // b*n_q + head
  const int lane = threadIdx.x & 31;
  const float2* part = p.partials + (size_t)slot * p.max_splits;
  if (threadIdx.x < 32) {
    float m = -INFINITY;
    for (int i = lane; i < p.n_splits; i += 32) m = fmaxf(m, part[i].x);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      float z = 0.0f;
      for (int i = 0; i < p.n_splits; ++i) {
        const float2 ml = part[i];
        if (ml.y > 0.0f) z += ml.y * expf(ml.x - m);
      }
      sMZ[0] = m;
      sMZ[1] = z;
    }
  }
  __syncthreads();
  const float* lrow = p.logits + (size_t)slot * p.lstride;
  for (int j = threadIdx.x; j < p.s; j += blockDim.x)
    probs[(size_t)slot * p.s + j] = expf(lrow[j] - sMZ[0]) / sMZ[1];
}

}  // namespace

void probs_launch(const SelectParams& p, float* probs, cudaStream_t st) {
  probs_kernel<<<p.rows * p.G, 256, 0, st>>>(p, probs);
}

void select_launch(const SelectParams& p, cudaStream_t st) {
  select_kernel<<<p.rows, kT, 0, st>>>(p);
}

void arg_topk_launch(const float* values, int n, int k, uint32_t* keys_scratch, uint32_t* out,
                     cudaStream_t st) {
  const int nc = k < n ? k : n;
  arg_topk_kernel<<<1, kT, 0, st>>>(values, n, nc, keys_scratch, out);
}

}  // namespace kc

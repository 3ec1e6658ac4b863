// kc_rowsel.cuh -- top-N selection of one MHA row by the 256 consumer threads
// of a scoring CTA (sm_100a), fused into score_fast_kernel.
//
// The reference ranks p = exp(s - M)/Z with a stable descending sort, keeps
// min(N, s) positions and returns them in ascending order with their raw p
// (proj/core/src/matrix.cpp:109-122, attention.cpp:126-154). select_reg_kernel
// (kc_select.cu) does that as a separate launch after the scoring; here the
// last CTA to finish a row's splits (a per-row completion counter) selects the
// row itself while the other CTAs keep streaming K, so the selection leaves
// the critical path. Outputs are bit-identical to select_reg_kernel's:
//   1. (M, Z) from the row's split partials (softmax_stats);
//   2. keys = order-preserving bits of the logit (p is monotone in s, so the
//      p-order and the s-order can only disagree inside a p-tie, which the
//      classification resolves with the exact p);
//   3. bound: tau = min over the 8 warps of each warp's ceil(N/8)-th largest
//      thread maximum (>= N keys are >= tau), lowered by the p-tie window;
//      the keys >= tau are compacted into shared memory in position order
//      (the scoring ring, free once the CTA's item is done). Too many, or
//      p(tau) not a normal float: every position is a candidate, read from L2;
//   4. MSB-first radix select (11/11/10-bit digits) of the N-th largest key T;
//   5. classification (p-exact inside T's tie window), three block scans,
//      ordered output: idx ascending, w = expf(s - M) / Z;
//   6. dropped = 1 - sum double(w) and 1/sum w with finish_group's reduction
//      tree (1024 virtual threads, xor butterflies), so the bits match.
// The logits row was written by other SMs during this kernel: it is read with
// ld.global.cg (L2), never through a possibly stale L1 line.
#pragma once

#include <cfloat>

#include "kc_device.cuh"

namespace kc {
namespace rowsel {

constexpr int kNT = 256;             // consumer threads
constexpr int kNW = kNT / 32;
constexpr int kBins = 2048;
constexpr int kBPT = kBins / kNT;    // histogram bins per thread
constexpr int kMaxNc = kNW * 32;     // the warp-local bound needs ceil(N/8) <= 32

struct Shared {
  uint32_t hist[kBins];
  uint32_t wa[kNW], wb[kNW], wc[kNW];
  double red_d[32];
  float red_f[32];
  float M, Z;
  uint32_t bin, need;
};
// candidates follow the Shared block in the ring
constexpr int kSharedBytes = (int)((sizeof(Shared) + 15) / 16 * 16);

__device__ __forceinline__ void bar() { asm volatile("bar.sync 1, %0;" ::"r"(kNT) : "memory"); }

// exclusive prefix sum over the 256 threads (thread order) + the total
__device__ __forceinline__ uint32_t excl_scan(uint32_t x, uint32_t* wt, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) wt[warp] = v;
  bar();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kNW; ++w) {
    const uint32_t c = wt[w];
    before += w < warp ? c : 0u;
    tot += c;
  }
  bar();
  total = tot;
  return before + v - x;
}

__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool active, int lane) {
  const uint32_t key = active ? bin : 0xffffffffu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int leader = 31 - __clz(peers);
  if (active && lane == leader) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

__device__ __forceinline__ void clear_hist(Shared& S) {
  for (int i = threadIdx.x; i < kBins; i += kNT) S.hist[i] = 0;
  bar();
}

// Among the bins, find B with (count above B) < need <= (count at or above B);
// leaves S.bin = B, S.need = need - (count above B).
__device__ __forceinline__ void find_bin(Shared& S, uint32_t need) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t h[kBPT], local = 0;
#pragma unroll
  for (int i = 0; i < kBPT; ++i) {
    h[i] = S.hist[t * kBPT + i];
    local += h[i];
  }
  uint32_t v = local;  // inclusive suffix sum over the warp's lanes
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v += n;
  }
  if (lane == 0) S.wa[warp] = v;
  bar();
  uint32_t acc = v - local;  // bins of later lanes of this warp
  for (int w = warp + 1; w < kNW; ++w) acc += S.wa[w];
#pragma unroll
  for (int i = kBPT - 1; i >= 0; --i) {
    if (acc < need && acc + h[i] >= need) {
      S.bin = (uint32_t)(t * kBPT + i);
      S.need = need - acc;
    }
    acc += h[i];
  }
  bar();
}

// The nc-th largest key over the items each(fn(key, pos, valid)) visits.
template <typename Each>
__device__ __forceinline__ uint32_t radix_T(Shared& S, Each&& each, uint32_t nc) {
  const int lane = threadIdx.x & 31;
  clear_hist(S);
  each([&](uint32_t k, uint32_t, bool v) { hist_add(S.hist, k >> 21, v, lane); });
  bar();
  find_bin(S, nc);
  const uint32_t b0 = S.bin;
  uint32_t need = S.need;
  clear_hist(S);
  each([&](uint32_t k, uint32_t, bool v) {
    const bool act = v && (k >> 21) == b0;
    if (__any_sync(0xffffffffu, act)) hist_add(S.hist, (k >> 10) & 0x7ffu, act, lane);
  });
  bar();
  find_bin(S, need);
  const uint32_t p01 = (b0 << 11) | S.bin;
  need = S.need;
  clear_hist(S);
  each([&](uint32_t k, uint32_t, bool v) {
    const bool act = v && (k >> 10) == p01;
    if (__any_sync(0xffffffffu, act)) hist_add(S.hist, k & 0x3ffu, act, lane);
  });
  bar();
  find_bin(S, need);
  return (p01 << 10) | S.bin;
}

// select_reg_kernel's MHA classification: 2 = ranked above the N-th p,
// 1 = in its tie class, 0 = out
struct Cls {
  float Ts, M, Z, pT, win;
  bool all, exact_all;
  __device__ __forceinline__ int operator()(uint32_t key) const {
    if (all) return 2;
    const float sj = from_ordered(key);
    if (sj > Ts + win) return 2;
    if (exact_all || sj >= Ts - win) {
      const float pj = expf(sj - M) / Z;
      return pj > pT ? 2 : (pj == pT ? 1 : 0);
    }
    return 0;
  }
};

// radix select + classification + ordered output over the items (visited in
// position order per thread, threads in position order)
template <typename Each>
__device__ void select_items(Shared& S, Each&& each, uint32_t n_valid, uint32_t nc, float M, float Z,
                             uint32_t* idx, float* w) {
  Cls cls{};
  cls.M = M;
  cls.Z = Z;
  cls.all = nc >= n_valid;
  if (!cls.all) {
    const uint32_t T = radix_T(S, each, nc);
    cls.Ts = from_ordered(T);
    cls.pT = expf(cls.Ts - M) / Z;
    cls.win = tie_window(cls.Ts, M);
    cls.exact_all = !(cls.pT >= FLT_MIN);  // p(T) subnormal or 0: ties are wide
  }
  uint32_t cgt = 0, ceq = 0;
  each([&](uint32_t k, uint32_t, bool v) {
    if (!v) return;
    const int r = cls(k);
    cgt += r == 2;
    ceq += r == 1;
  });
  uint32_t n_gt = 0, tot = 0;
  excl_scan(cgt, S.wa, n_gt);
  const uint32_t keq = nc - n_gt;
  const uint32_t eq_base = excl_scan(ceq, S.wb, tot);
  const uint32_t take = eq_base >= keq ? 0u : min(ceq, keq - eq_base);
  uint32_t o = excl_scan(cgt + take, S.wc, tot);
  uint32_t eqr = eq_base;
  each([&](uint32_t k, uint32_t pos, bool v) {
    if (!v) return;
    const int r = cls(k);
    bool sel = r == 2;
    if (r == 1) {
      sel = eqr < keq;
      ++eqr;
    }
    if (sel) {
      idx[o] = pos;
      w[o] = expf(from_ordered(k) - M) / Z;  // = expf(s - M)/Z (-0 -> +0 changes nothing)
      ++o;
    }
  });
}

// finish_group (kc_select.cu) for one q head, emulating its 1024-thread tree:
// virtual thread t sums w[t], w[t + 1024], ...; xor butterflies per virtual
// warp, then over the 32 warp totals.
__device__ __forceinline__ void finish(Shared& S, const float* wrow, uint32_t nc, double* dropped, float* norm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int vw = warp; vw < 32; vw += kNW) {
    double md = 0.0;
    float fs = 0.0f;
    for (uint32_t r = vw * 32 + lane; r < nc; r += 1024) {
      const float x = wrow[r];
      md += (double)x;
      fs += x;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      md += __shfl_xor_sync(0xffffffffu, md, o);
      fs += __shfl_xor_sync(0xffffffffu, fs, o);
    }
    if (lane == 0) {
      S.red_d[vw] = md;
      S.red_f[vw] = fs;
    }
  }
  bar();
  if (warp == 0) {
    double a = S.red_d[lane];
    float f = S.red_f[lane];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      f += __shfl_xor_sync(0xffffffffu, f, o);
    }
    if (lane == 0) {
      *dropped = 1.0 - a;
      *norm = f > 0.0f ? 1.0f / f : 1.0f;
    }
  }
}

struct RowOut {
  uint32_t* idx;   // [nc]
  float* w;        // [nc]
  double* dropped;
  float* norm;
};

// Select the row's top-nc (nc <= min(s, kMaxNc) not required: any nc >= 1).
// smem: >= kSharedBytes + 8 * cap bytes, 16-B aligned. Called by the 256
// consumer threads only (named barrier 1).
__device__ void select_row(uint8_t* smem, int cap, const float* lrow, const float2* part, int n_splits, int s,
                           int nc, const RowOut& out, bool keep_logits) {
  Shared& S = *reinterpret_cast<Shared*>(smem);
  uint32_t* ckey = reinterpret_cast<uint32_t*>(smem + kSharedBytes);
  uint32_t* cpos = ckey + cap;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (warp == 0) {
    float m, z;
    softmax_stats<true>(part, n_splits, lane, m, z);
    if (lane == 0) {
      S.M = m;
      S.Z = z;
    }
  }
  bar();
  const float M = S.M, Z = S.Z;
  // thread t owns positions [t*ppt, t*ppt + ppt) (float4 granules; rows are
  // padded to 32 floats, so a granule starting below s is in bounds)
  const int ppt = (((s + kNT - 1) / kNT) + 3) & ~3;
  const int j0 = t * ppt;
  // batches of 8 independent 16-B L2 loads in flight (a pass is a few L2
  // round trips, not ppt/4 of them); the trip count is warp-uniform
  constexpr int kB = 8;
  auto l2_each = [&](auto&& fn) {
    for (int jb = 0; jb < ppt; jb += 4 * kB) {
      float4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int j = j0 + jb + 4 * u;
        v[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (jb + 4 * u < ppt && j < s) v[u] = __ldcg(reinterpret_cast<const float4*>(lrow + j));
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (jb + 4 * u < ppt) {
          const int j = j0 + jb + 4 * u;
          fn(ordered_bits(v[u].x), (uint32_t)j, j < s);
          fn(ordered_bits(v[u].y), (uint32_t)j + 1, j + 1 < s);
          fn(ordered_bits(v[u].z), (uint32_t)j + 2, j + 2 < s);
          fn(ordered_bits(v[u].w), (uint32_t)j + 3, j + 3 < s);
        }
      }
    }
  };
  bool done = false;
  if (nc < s && nc <= kMaxNc) {
    uint32_t tmax = 0;
    l2_each([&](uint32_t k, uint32_t, bool v) {
      if (v) tmax = max(tmax, k);
    });
    const int kw = (nc + kNW - 1) / kNW;
    uint32_t v = tmax, kth = 0;
    for (int r = 0; r < kw; ++r) {
      kth = __reduce_max_sync(0xffffffffu, v);
      const uint32_t ball = __ballot_sync(0xffffffffu, v == kth);
      if (lane == __ffs(ball) - 1) v = 0u;
    }
    if (lane == 0) S.wa[warp] = kth;
    bar();
    uint32_t tau = S.wa[0];
#pragma unroll
    for (int w = 1; w < kNW; ++w) tau = min(tau, S.wa[w]);
    bar();
    // a score just below tau can still share the N-th score's p: lower the
    // bound by the tie window; p(tau) not a normal float: every position
    const float ts = from_ordered(tau);
    const bool fast = expf(ts - M) / Z >= FLT_MIN;
    if (ts > -INFINITY) tau = ordered_bits(ts - 2.0f * tie_window(ts, M));
    if (fast) {
      uint32_t cnt = 0, C = 0;
      l2_each([&](uint32_t k, uint32_t, bool vld) { cnt += (vld && k >= tau) ? 1u : 0u; });
      uint32_t base = excl_scan(cnt, S.wa, C);
      if (C <= (uint32_t)cap) {
        l2_each([&](uint32_t k, uint32_t pos, bool vld) {
          if (vld && k >= tau) {
            ckey[base] = k;
            cpos[base] = pos;
            ++base;
          }
        });
        bar();
        const int cpt = (int)((C + kNT - 1) / kNT);
        auto c_each = [&](auto&& fn) {
          for (int i = 0; i < cpt; ++i) {
            const int c = t * cpt + i;
            const bool vld = c < (int)C;
            fn(vld ? ckey[c] : 0u, vld ? cpos[c] : 0u, vld);
          }
        };
        select_items(S, c_each, C, (uint32_t)nc, M, Z, out.idx, out.w);
        done = true;
      }
    }
  }
  if (!done) select_items(S, l2_each, (uint32_t)s, (uint32_t)nc, M, Z, out.idx, out.w);
  bar();
  finish(S, out.w, (uint32_t)nc, out.dropped, out.norm);
  if (!keep_logits) {
    // the dead logits leave L2 without a write-back
    const int lines = (s * 4 + 127) / 128;
    for (int e = t; e < lines; e += kNT) discard_l2_line(reinterpret_cast<const char*>(lrow) + (size_t)e * 128);
  }
  bar();  // the ring is reused by nothing after this, but S must not be read late
}

}  // namespace rowsel
}  // namespace kc

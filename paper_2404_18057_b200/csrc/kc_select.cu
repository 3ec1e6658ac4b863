// kc_select.cu -- per-(batch, kv-head) top-N selection (sm_100a).
//
// Replaces the softmax normalisation (proj/core/src/matrix.cpp:45-61),
// arg_topk (proj/core/src/matrix.cpp:109-122) and the TopNSelection fill
// loop (proj/core/src/attention.cpp:126-154).
//
// The reference ranks the fp32 PROBABILITIES p_j = exp(s_j - M) / Z
// (attention.cpp:140) with a stable descending sort, so equal probabilities
// tie to the lowest position even when their logits differ, and returns the
// survivors in ascending position order. The GPU reproduces exactly that rule
// on its own p (for GQA the key is sum_g p_g[j]):
//   1. global (M, Z) per q head from the scoring kernel's per-split
//      (max, sum exp) (softmax_stats, kc_device.cuh);
//   2. keys. MHA: the order-preserving bits of the logit itself -- p is a
//      monotone non-decreasing function of s, so the p-order and the s-order
//      can only disagree inside a p-tie, which step 4 resolves exactly.
//      GQA: the fp32 bits of sum_g p_g (>= 0, so raw bits order like values);
//   3. MSB-first radix select (11/11/10-bit digits, shared-memory histograms
//      with warp-aggregated atomics) finds the N-th largest key T;
//   4. classification + ordered compaction: survivors are the keys ranked
//      above the N-th p plus the lowest-position members of its tie class;
//      two block scans give every thread its output offset, so indices come
//      out ascending (the reference's final std::sort) with no sort at all;
//   5. weights p[idx], dropped = 1 - sum double(p), renormaliser 1/sum p
//      (attention.cpp:146-152,167-174).
// s <= 32768: keys stay in registers (select_reg_kernel, thread t owns
// positions [t*KPT, t*KPT+KPT)); longer rows use a global-memory key scratch
// (select_kernel).
#include <cfloat>

#include "kc_device.cuh"
#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace kc {

namespace {

constexpr int kT = 1024;
constexpr int kNW = kT / 32;
constexpr int kBins = 2048;
constexpr int kMaxG = 32;
constexpr int kCandSmem = 4096;  // select_kernel fast path: candidates held in shared memory

struct SelShared {
  uint32_t hist[kBins];
  uint32_t wa[kNW], wb[kNW], wc[kNW], wd[kNW];
  float M[kMaxG], Z[kMaxG];
  uint32_t bin, need;
  float red_f[kNW];
  double red_d[kNW];
};

__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool active, int lane) {
  const uint32_t key = active ? bin : 0xffffffffu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int leader = 31 - __clz(peers);  // highest peer lane (FLO, no BREV)
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

// Block-wide exclusive prefix sum over the 1024 threads (thread order).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = warp_tot[lane];
    uint32_t u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += n;
    }
    warp_tot[lane] = u - t;
  }
  __syncthreads();
  const uint32_t r = warp_tot[warp] + v - x;
  __syncthreads();
  return r;
}

// Radix select over (key, valid) pairs given by get(i) for the items a thread
// owns; returns the N-th largest key T and how many keys equal to T survive.
template <int KPT, typename Get>
__device__ __forceinline__ void radix_threshold(SelShared& S, Get&& get, int nc, int n_valid,
                                                uint32_t& T, uint32_t& k_eq) {
  const int lane = threadIdx.x & 31;
  T = 0;
  k_eq = (uint32_t)nc;
  if (nc >= n_valid) return;  // everything survives
  clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    hist_add(S.hist, k >> 21, v, lane);
  }
  __syncthreads();
  find_bin(S, (uint32_t)nc);
  const uint32_t b0 = S.bin;
  uint32_t need = S.need;
  clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    const bool act = v && (k >> 21) == b0;
    if (__any_sync(0xffffffffu, act)) hist_add(S.hist, (k >> 10) & 0x7ffu, act, lane);
  }
  __syncthreads();
  find_bin(S, need);
  const uint32_t p01 = (b0 << 11) | S.bin;
  need = S.need;
  clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    const bool act = v && (k >> 10) == p01;
    if (__any_sync(0xffffffffu, act)) hist_add(S.hist, k & 0x3ffu, act, lane);
  }
  __syncthreads();
  find_bin(S, need);
  T = (p01 << 10) | S.bin;
  k_eq = S.need;
}

// Candidate-mode fallback: recompute one MHA row's scores into the dense
// logits row, bit-identical to score_fast_kernel<T, 1, 4, ...>: the same lane
// roles (4 lanes per position, 16-B chunk c = ((ci ^ (pos & 1)) << 2) | sub),
// the same fmaf sequence, the same xor-shuffle tree and the multiply by scale
// after the sum.
template <typename T>
__device__ void recompute_row_t(const SelectParams& p, int row) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = lane >> 2, sub = lane & 3;
  const int b = row / p.n_kv, kvh = row - b * p.n_kv;
  const float* qh = p.q + ((size_t)b * p.n_kv + kvh) * 128;
  float qf[4][8];
#pragma unroll
  for (int ci = 0; ci < 4; ++ci) {
    const int c = ((ci ^ (rl & 1)) << 2) | sub;
#pragma unroll
    for (int e = 0; e < 8; ++e) qf[ci][e] = qh[c * 8 + e];
  }
  const T* kslot = static_cast<const T*>(p.k) + (size_t)row * p.max_seq * 128;
  float* lrow = const_cast<float*>(p.logits) + ((size_t)b * p.n_kv + kvh) * p.lstride;
  for (int base = warp * 8; base < p.s; base += kNW * 8) {
    const int pos = base + rl;
    float acc = 0.0f;
    if (pos < p.s) {
      const uint4* krow = reinterpret_cast<const uint4*>(kslot + (size_t)pos * 128);
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) {
        const int c = ((ci ^ (rl & 1)) << 2) | sub;
        float kf[8];
        unpack8<T>(krow[c], kf);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(qf[ci][e], kf[e], acc);
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (pos < p.s && sub == 0) lrow[pos] = acc * p.scale;
  }
}

// Dense-redo prologue of the selection kernels (candidate-mode fallback):
// false when this row needs no redo.
__device__ __forceinline__ bool fallback_prologue(const SelectParams& p, int row) {
  if (!p.fb_flags) return true;
  if (p.fb_flags[row] == 0) return false;
  if (p.kdtype == KC_BF16) recompute_row_t<__nv_bfloat16>(p, row);
  else recompute_row_t<__half>(p, row);
  __syncthreads();
  return true;
}

__device__ __forceinline__ void load_stats(SelShared& S, const SelectParams& p, int b, int kvh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_q = p.n_kv * p.G;
  for (int g = warp; g < p.G; g += kNW) {
    float m, z;
    softmax_stats(p.partials + ((size_t)b * n_q + kvh * p.G + g) * p.max_splits, p.n_splits, lane, m, z);
    if (lane == 0) {
      S.M[g] = m;
      S.Z[g] = z;
    }
  }
  __syncthreads();
}

// dropped mass and renormaliser of every q head of the group from the weights
// just written (block-wide reductions; the weights are visible after the
// caller's __syncthreads).
// wsm: the same weights staged in shared memory ([G][nc], saves the global
// round trip), or null.
__device__ void finish_group(SelShared& S, const SelectParams& p, int b, int kvh, const float* wsm = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_q = p.n_kv * p.G;
  for (int g = 0; g < p.G; ++g) {
    const size_t slot = (size_t)b * n_q + kvh * p.G + g;
    const float* wg = wsm ? wsm + (size_t)g * p.nc : p.w + slot * p.nc;
    double md = 0.0;
    float fs = 0.0f;
    for (int r = tid; r < p.nc; r += kT) {
      const float x = wg[r];
      md += (double)x;
      fs += x;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      md += __shfl_xor_sync(0xffffffffu, md, o);
      fs += __shfl_xor_sync(0xffffffffu, fs, o);
    }
    if (lane == 0) {
      S.red_d[warp] = md;
      S.red_f[warp] = fs;
    }
    __syncthreads();
    if (warp == 0) {
      double a = S.red_d[lane];
      float f = S.red_f[lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        f += __shfl_xor_sync(0xffffffffu, f, o);
      }
      if (lane == 0) {
        p.dropped[slot] = 1.0 - a;
        p.norm[slot] = f > 0.0f ? 1.0f / f : 1.0f;
      }
    }
    __syncthreads();
  }
}

// Drop the row's dead logits (dirty scratch) from L2 without write-back: saves
// the HBM write and keeps L2 free for the V recall's host reads.
__device__ __forceinline__ void drop_rows(const float* base, int64_t stride, int nrows, int s) {
  const int lines = (s * 4 + 127) / 128;
  for (int e = threadIdx.x; e < nrows * lines; e += kT) {
    const int g = e / lines, l = e - g * lines;
    discard_l2_line(reinterpret_cast<const char*>(base + (size_t)g * stride) + (size_t)l * 128);
  }
}

template <int KPT>
__device__ __forceinline__ void select_reg_body(const SelectParams& p) {
  __shared__ SelShared S;
  const int row = p.row0 + blockIdx.x;
  if (!fallback_prologue(p, row)) return;
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int G = p.G;
  const int n_q = p.n_kv * G;
  const int tid = threadIdx.x;
  const float* lbase = p.logits + ((size_t)b * n_q + kvh * G) * p.lstride;
  uint32_t* idx = p.idx + (size_t)row * p.nc;
  const int s = p.s, nc = p.nc;
  const int j0 = tid * KPT;

  // keys: MHA -> ordered logit bits (loaded before the stats' barrier: the
  // two global round trips overlap); GQA -> bits of sum_g p_g (needs M, Z)
  uint32_t key[KPT];
  if (G == 1) {
    if (j0 + KPT <= s) {
#pragma unroll
      for (int i = 0; i < KPT; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(lbase + j0 + i);
        key[i] = ordered_bits(v.x);
        key[i + 1] = ordered_bits(v.y);
        key[i + 2] = ordered_bits(v.z);
        key[i + 3] = ordered_bits(v.w);
      }
    } else {
#pragma unroll
      for (int i = 0; i < KPT; ++i) key[i] = j0 + i < s ? ordered_bits(lbase[j0 + i]) : 0u;
    }
  }
  load_stats(S, p, b, kvh);
  if (G != 1) {
#pragma unroll
    for (int i = 0; i < KPT; ++i) key[i] = 0u;
    // GQA ranking key sum_g p_g: the fast exp and a reciprocal (ranking only;
    // the weights below use the exact expf(s - M) / Z)
    for (int g = 0; g < G; ++g) {
      const float* lr = lbase + (size_t)g * p.lstride;
      const float Mg = S.M[g], rZ = 1.0f / S.Z[g];
      if (j0 + KPT <= s) {
#pragma unroll
        for (int i = 0; i < KPT; i += 4) {
          const float4 v = *reinterpret_cast<const float4*>(lr + j0 + i);
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float pg = __expf(e[u] - Mg) * rZ;
            key[i + u] = (g == 0) ? __float_as_uint(pg) : __float_as_uint(__uint_as_float(key[i + u]) + pg);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
          if (j0 + i < s) {
            const float pg = __expf(lr[j0 + i] - Mg) * rZ;
            key[i] = (g == 0) ? __float_as_uint(pg) : __float_as_uint(__uint_as_float(key[i]) + pg);
          }
        }
      }
    }
  }

  // ---- fast path: threshold from thread maxima, exact select on candidates --
  // tau = the nc-th largest of the 1024 per-thread maxima is a lower bound of
  // the nc-th largest key (nc threads each hold a key >= tau), and for
  // unstructured rows only ~nc keys reach it. Those candidates (<= 1024, in
  // position order) get the exact treatment; anything else (ties flooding
  // the bound, nc > 1024) falls through to the full radix pass below.
  bool fast = nc < s && nc <= kT;
  uint32_t tau = 0;
  if (fast) {
    uint32_t tmax = 0;
#pragma unroll
    for (int i = 0; i < KPT; ++i)
      if (j0 + i < s) tmax = max(tmax, key[i]);
    // tau = min over warps of the warp's kw-th largest thread maximum
    // (kw = ceil(nc / 32)): every warp holds >= kw maxima >= tau, so >= nc
    // keys are >= tau. Warp-local (REDUX + BALLOT), one block barrier --
    // ~2.3x more candidates than the exact nc-th maximum, far fewer barriers.
    {
      const int lane = tid & 31, warp = tid >> 5;
      const int kw = (nc + 31) / 32;
      uint32_t v = tmax, kth = 0;
      for (int r = 0; r < kw; ++r) {
        kth = __reduce_max_sync(0xffffffffu, v);
        const uint32_t ball = __ballot_sync(0xffffffffu, v == kth);
        if (lane == __ffs(ball) - 1) v = 0u;
      }
      if (lane == 0) S.wa[warp] = kth;
      __syncthreads();
      tau = S.wa[0];
#pragma unroll 8
      for (int w = 1; w < kNW; ++w) tau = min(tau, S.wa[w]);
      __syncthreads();  // S.wa is reused by the scans below
    }
    if (G == 1) {
      // a score just below tau can still share the N-th score's p (p-tie):
      // lower the bound by the tie window (keys are ordered logit bits).
      // When p(tau) is not a normal float the ties below tau are unbounded
      // (p underflows): take the full pass instead.
      const float ts = from_ordered(tau);
      fast = expf(ts - S.M[0]) / S.Z[0] >= FLT_MIN;
      if (ts > -INFINITY) tau = ordered_bits(ts - 2.0f * tie_window(ts, S.M[0]));
    }
  }
  if (fast) {
    uint32_t ccount = 0;
#pragma unroll
    for (int i = 0; i < KPT; ++i) ccount += (j0 + i < s && key[i] >= tau) ? 1u : 0u;
    uint32_t cbase = block_excl_scan(ccount, S.wa);
    if (tid == kT - 1) S.need = cbase + ccount;
    __syncthreads();
    const uint32_t C = S.need;
    if (C <= (uint32_t)kT) {
      // candidates -> shared memory (reuse the histogram space), position order
      uint32_t* ckey = S.hist;
      uint32_t* cpos = S.hist + kT;
#pragma unroll
      for (int i = 0; i < KPT; ++i) {
        if (j0 + i < s && key[i] >= tau) {
          ckey[cbase] = key[i];
          cpos[cbase] = (uint32_t)(j0 + i);
          ++cbase;
        }
      }
      __syncthreads();
      const bool have = (uint32_t)tid < C;
      const uint32_t ck = have ? ckey[tid] : 0u;
      const uint32_t cp = have ? cpos[tid] : 0u;
      __syncthreads();  // the histogram space is reused by the radix below
      uint32_t T, k_eq;
      radix_threshold<1>(S, [&](int, bool& v) { v = have; return ck; }, nc, (int)C, T, k_eq);
      uint32_t gt = 0, eq = 0;
      if ((uint32_t)nc >= C) {
        gt = have ? 1u : 0u;  // exactly nc candidates: all of them survive
      } else if (have) {
        if (G == 1) {
          const float Ts = from_ordered(T);
          const float M = S.M[0], Z = S.Z[0];
          const float pT = expf(Ts - M) / Z;
          const float win = tie_window(Ts, M);
          const bool exact_all = !(pT >= FLT_MIN);  // p(T) subnormal or 0: ties are wide
          const float sj = from_ordered(ck);
          if (sj > Ts + win) {
            gt = 1;
          } else if (exact_all || sj >= Ts - win) {
            const float pj = expf(sj - M) / Z;
            gt = pj > pT;
            eq = pj == pT;
          }
        } else {
          gt = ck > T;
          eq = ck == T;
        }
      }
      const uint32_t gbase = block_excl_scan(gt, S.wc);
      if (tid == kT - 1) S.need = gbase + gt;
      __syncthreads();
      const uint32_t keq = (uint32_t)nc - S.need;
      const uint32_t ebase = block_excl_scan(eq, S.wa);
      const bool sel = gt || (eq && ebase < keq);
      const uint32_t o = block_excl_scan(sel ? 1u : 0u, S.wb);
      // the weights also go to shared memory (the histogram space is free
      // now) so finish_group reduces them without a global round trip
      float* wsm = G * nc <= kBins ? reinterpret_cast<float*>(S.hist) : nullptr;
      if (sel) {
        idx[o] = cp;
        for (int g = 0; g < G; ++g) {
          // MHA: the candidate's logit is from_ordered(ck) (-0 -> +0 changes
          // nothing in expf(s - M)); GQA reloads each head's logit
          const float sg = G == 1 ? from_ordered(ck) : lbase[(size_t)g * p.lstride + cp];
          const float wv = expf(sg - S.M[g]) / S.Z[g];
          p.w[((size_t)b * n_q + kvh * G + g) * nc + o] = wv;
          if (wsm) wsm[(size_t)g * nc + o] = wv;
        }
      }
      __syncthreads();
      if (!p.keep_logits) drop_rows(lbase, p.lstride, G, s);
      finish_group(S, p, b, kvh, wsm);
      return;
    }
  }

  uint32_t T, k_eq;
  radix_threshold<KPT>(S, [&](int i, bool& v) { v = j0 + i < s; return key[i]; }, nc,
                       min(s, kT * KPT), T, k_eq);

  // classification: 2 = ranked above the N-th p, 1 = in its tie class
  uint32_t cls_gt = 0, cls_eq = 0;  // bit i set for item i
  if (G == 1 && nc < s) {
    // p is monotone in s: only logits close to T_s can share T's probability.
    // Inside the window compare exact p (the same expression the weights use).
    const float Ts = from_ordered(T);
    const float M = S.M[0], Z = S.Z[0];
    const float pT = expf(Ts - M) / Z;
    const float win = tie_window(Ts, M);
    const bool exact_all = !(pT >= FLT_MIN);  // p(T) subnormal or 0: ties are wide
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      if (j0 + i >= s) continue;
      const float sj = from_ordered(key[i]);
      if (sj > Ts + win) {
        cls_gt |= 1u << i;
      } else if (exact_all || sj >= Ts - win) {
        const float pj = expf(sj - M) / Z;
        if (pj > pT) cls_gt |= 1u << i;
        else if (pj == pT) cls_eq |= 1u << i;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      if (j0 + i >= s) continue;
      if (key[i] > T) cls_gt |= 1u << i;
      else if (key[i] == T) cls_eq |= 1u << i;
    }
  }
  // ties take the remaining places, lowest positions first
  const uint32_t n_gt_local = __popc(cls_gt);
  uint32_t n_gt_total;
  {
    const uint32_t base = block_excl_scan(n_gt_local, S.wc);
    if (tid == kT - 1) S.need = base + n_gt_local;
    __syncthreads();
    n_gt_total = S.need;
    __syncthreads();
  }
  k_eq = (uint32_t)nc - n_gt_total;
  const uint32_t ceq = __popc(cls_eq);
  const uint32_t eq_base = block_excl_scan(ceq, S.wa);
  const uint32_t take = eq_base >= k_eq ? 0u : min(ceq, k_eq - eq_base);
  uint32_t o = block_excl_scan(n_gt_local + take, S.wb);
  uint32_t eqr = eq_base;
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool sel = (cls_gt >> i) & 1u;
    if ((cls_eq >> i) & 1u) {
      sel = eqr < k_eq;
      ++eqr;
    }
    if (sel) {
      const int j = j0 + i;
      idx[o] = (uint32_t)j;
      for (int g = 0; g < G; ++g)
        p.w[((size_t)b * n_q + kvh * G + g) * nc + o] =
            expf(lbase[(size_t)g * p.lstride + j] - S.M[g]) / S.Z[g];
      ++o;
    }
  }
  __syncthreads();
  if (!p.keep_logits) drop_rows(lbase, p.lstride, G, s);
  finish_group(S, p, b, kvh);
}

template <int KPT>
__global__ void __launch_bounds__(kT, 1) select_reg_kernel(const SelectParams p) {
  select_reg_body<KPT>(p);
}

// Any length: keys in a global scratch row (L2-resident), same rule.
__global__ void __launch_bounds__(kT) select_kernel(const SelectParams p) {
  __shared__ SelShared S;
  const int row = p.row0 + blockIdx.x;
  if (!fallback_prologue(p, row)) return;
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int G = p.G;
  const int n_q = p.n_kv * G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* lbase = p.logits + ((size_t)b * n_q + kvh * G) * p.lstride;
  uint32_t* keys = p.keys + (size_t)row * p.kstride;
  uint32_t* idx = p.idx + (size_t)row * p.nc;
  const int s = p.s, nc = p.nc;
  load_stats(S, p, b, kvh);

  // keys: MHA the exact p (its bits order like p, ties exact); GQA the
  // ranking key sum_g p_g with the fast exp and a reciprocal (ranking only --
  // the weights below are recomputed exactly), four positions per thread step
  uint32_t tmax = 0;
  if (G == 1) {
    for (int j = tid; j < s; j += kT) {
      const uint32_t k = __float_as_uint(expf(lbase[j] - S.M[0]) / S.Z[0]);
      keys[j] = k;
      tmax = max(tmax, k);
    }
  } else {
    for (int j4 = tid * 4; j4 < s; j4 += kT * 4) {
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int g = 0; g < G; ++g) {
        const float* lr = lbase + (size_t)g * p.lstride;
        const float Mg = S.M[g], rZ = 1.0f / S.Z[g];
        float e[4];
        if (j4 + 4 <= s) {
          const float4 v = *reinterpret_cast<const float4*>(lr + j4);
          e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) e[u] = j4 + u < s ? lr[j4 + u] : -INFINITY;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += __expf(e[u] - Mg) * rZ;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j4 + u < s) {
          const uint32_t k = __float_as_uint(acc[u]);
          keys[j4 + u] = k;
          tmax = max(tmax, k);
        }
      }
    }
  }
  __syncthreads();

  // ---- fast path: bound from the thread maxima, exact select on the few
  // candidates (keys are bits of p: exact order, no tie window needed) ----
  if (nc < s && nc <= kT) {
    __shared__ uint32_t ckey[kCandSmem], cpos[kCandSmem];
    const int kw = (nc + 31) / 32;
    uint32_t v = tmax, kth = 0;
    for (int r = 0; r < kw; ++r) {
      kth = __reduce_max_sync(0xffffffffu, v);
      const uint32_t ball = __ballot_sync(0xffffffffu, v == kth);
      if (lane == __ffs(ball) - 1) v = 0u;
    }
    if (lane == 0) S.wa[warp] = kth;
    __syncthreads();
    uint32_t tau = S.wa[0];
    for (int w = 1; w < kNW; ++w) tau = min(tau, S.wa[w]);
    __syncthreads();
    // candidates >= tau, compacted in position order (warp segments)
    const int seg = (((s + kNW - 1) / kNW) + 31) & ~31;
    const int w0 = warp * seg, w1 = min(s, w0 + seg);
    uint32_t cnt = 0;
    for (int j0 = w0; j0 < w1; j0 += 32) {
      const int j = j0 + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, j < w1 && keys[j] >= tau));
    }
    if (lane == 0) S.wb[warp] = cnt;
    __syncthreads();
    uint32_t base = 0, C = 0;
    for (int w = 0; w < kNW; ++w) {
      const uint32_t c = S.wb[w];
      base += (w < warp) ? c : 0u;
      C += c;
    }
    if (C <= (uint32_t)kCandSmem) {
      const uint32_t lt = lanemask_lt();
      for (int j0 = w0; j0 < w1; j0 += 32) {
        const int j = j0 + lane;
        const uint32_t k = j < w1 ? keys[j] : 0u;
        const bool take = j < w1 && k >= tau;
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        if (take) {
          const uint32_t o = base + __popc(bal & lt);
          ckey[o] = k;
          cpos[o] = (uint32_t)j;
        }
        base += __popc(bal);
      }
      __syncthreads();
      constexpr int CK = kCandSmem / kT;
      const int c0 = tid * CK;
      uint32_t key[CK];
#pragma unroll
      for (int i = 0; i < CK; ++i) key[i] = c0 + i < (int)C ? ckey[c0 + i] : 0u;
      uint32_t T2 = 0, k_eq2 = (uint32_t)nc;
      radix_threshold<CK>(S, [&](int i, bool& vld) { vld = c0 + i < (int)C; return key[i]; }, nc, (int)C, T2, k_eq2);
      uint32_t cls_gt = 0, cls_eq = 0;
#pragma unroll
      for (int i = 0; i < CK; ++i) {
        if (c0 + i >= (int)C) continue;
        if ((uint32_t)nc >= C || key[i] > T2) cls_gt |= 1u << i;
        else if (key[i] == T2) cls_eq |= 1u << i;
      }
      const uint32_t n_gt_local = __popc(cls_gt);
      uint32_t n_gt_total;
      {
        const uint32_t b0 = block_excl_scan(n_gt_local, S.wc);
        if (tid == kT - 1) S.need = b0 + n_gt_local;
        __syncthreads();
        n_gt_total = S.need;
        __syncthreads();
      }
      const uint32_t keq = (uint32_t)nc - n_gt_total;
      const uint32_t ceq = __popc(cls_eq);
      const uint32_t eq_base = block_excl_scan(ceq, S.wa);
      const uint32_t takeq = eq_base >= keq ? 0u : min(ceq, keq - eq_base);
      uint32_t o = block_excl_scan(n_gt_local + takeq, S.wb);
      uint32_t eqr = eq_base;
#pragma unroll
      for (int i = 0; i < CK; ++i) {
        bool sel = (cls_gt >> i) & 1u;
        if ((cls_eq >> i) & 1u) {
          sel = eqr < keq;
          ++eqr;
        }
        if (sel) {
          const uint32_t j = cpos[c0 + i];
          idx[o] = j;
          for (int g = 0; g < G; ++g)
            p.w[((size_t)b * n_q + kvh * G + g) * nc + o] =
                expf(lbase[(size_t)g * p.lstride + j] - S.M[g]) / S.Z[g];
          ++o;
        }
      }
      __syncthreads();
      if (!p.keep_logits) drop_rows(lbase, p.lstride, G, s);
      drop_rows(reinterpret_cast<const float*>(keys), 0, 1, s);
      finish_group(S, p, b, kvh);
      return;
    }
  }

  // strided radix passes over the scratch row
  uint32_t T = 0, k_eq = (uint32_t)nc;
  if (nc < s) {
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      hist_add(S.hist, (j < s ? keys[j] : 0u) >> 21, j < s, lane);
    }
    __syncthreads();
    find_bin(S, (uint32_t)nc);
    const uint32_t b0 = S.bin;
    uint32_t need = S.need;
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < s ? keys[j] : 0u;
      const bool act = j < s && (k >> 21) == b0;
      if (__any_sync(0xffffffffu, act)) hist_add(S.hist, (k >> 10) & 0x7ffu, act, lane);
    }
    __syncthreads();
    find_bin(S, need);
    const uint32_t p01 = (b0 << 11) | S.bin;
    need = S.need;
    clear_hist(S);
    for (int base = 0; base < s; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < s ? keys[j] : 0u;
      const bool act = j < s && (k >> 10) == p01;
      if (__any_sync(0xffffffffu, act)) hist_add(S.hist, k & 0x3ffu, act, lane);
    }
    __syncthreads();
    find_bin(S, need);
    T = (p01 << 10) | S.bin;
    k_eq = S.need;
  }

  // ordered compaction over per-warp contiguous segments
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
    if (sel) {
      const uint32_t o = run_sel + __popc(bsel & lt);
      idx[o] = (uint32_t)j;
      for (int g = 0; g < G; ++g)
        p.w[((size_t)b * n_q + kvh * G + g) * nc + o] =
            expf(lbase[(size_t)g * p.lstride + j] - S.M[g]) / S.Z[g];
    }
    run_eq += __popc(beq);
    run_sel += __popc(bsel);
  }
  __syncthreads();
  if (!p.keep_logits) drop_rows(lbase, p.lstride, G, s);
  drop_rows(reinterpret_cast<const float*>(keys), 0, 1, s);
  finish_group(S, p, b, kvh);
}

// Candidate mode (MHA): the scoring kernel left, per split, the positions
// that can still be in the row's top-N (kc_score.cu emit_candidates) in
// position order; concatenated over splits they stay in position order, so
// the dense kernel's rule applies unchanged to the (score, position) list:
// radix select of the N-th largest score T, p-exact tie classification,
// ordered compaction. The row is complete -- no excluded position could rank
// above or tie with p(T) -- iff every split's exclusion bound lies below T's
// tie window and p(T) is a normal float; otherwise the row is flagged for the
// dense redo (select_fallback).
constexpr int kCandKPT = 16;  // up to 16384 candidates per row

__global__ void __launch_bounds__(kT, 1) select_cand_kernel(const SelectParams p) {
  __shared__ SelShared S;
  extern __shared__ uint2 csm[];  // [kT * kCandKPT] candidates, then prefix[n_splits + 1]
  uint32_t* pre = reinterpret_cast<uint32_t*>(csm + kT * kCandKPT);
  const int row = p.row0 + blockIdx.x;
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nc = p.nc;
  uint32_t* idx = p.idx + (size_t)row * nc;
  load_stats(S, p, b, kvh);

  if (warp == 0) {
    const uint2* meta = p.cand_meta + (size_t)row * p.max_splits;
    uint32_t run = 0;
    float bmax = -INFINITY;
    for (int s0 = 0; s0 < p.n_splits; s0 += 32) {
      const int sp = s0 + lane;
      const uint2 m = sp < p.n_splits ? meta[sp] : make_uint2(0u, __float_as_uint(-INFINITY));
      bmax = fmaxf(bmax, __uint_as_float(m.y));
      uint32_t v = m.x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
      }
      if (sp < p.n_splits) pre[sp] = run + v - m.x;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    if (lane == 0) {
      pre[p.n_splits] = run;
      S.need = run;
      S.red_f[0] = bmax;
    }
  }
  __syncthreads();
  const uint32_t C = S.need;
  const float bmax = S.red_f[0];
  __syncthreads();  // S.need / S.red_f are reused below
  if (C > (uint32_t)(kT * kCandKPT) || C < (uint32_t)nc || p.force_fallback) {
    if (tid == 0) p.fb_flags[row] = 1u;
    return;
  }
  for (int sp = warp; sp < p.n_splits; sp += kNW) {
    const uint32_t o = pre[sp], n = pre[sp + 1] - o;
    const uint2* src = p.cand + (size_t)row * p.lstride + (size_t)sp * p.chunk;
    for (uint32_t i = lane; i < n; i += 32) csm[o + i] = src[i];
  }
  __syncthreads();

  const int j0 = tid * kCandKPT;
  uint32_t key[kCandKPT];
#pragma unroll
  for (int i = 0; i < kCandKPT; ++i) key[i] = j0 + i < (int)C ? ordered_bits(__uint_as_float(csm[j0 + i].x)) : 0u;

  uint32_t T, k_eq;
  if ((uint32_t)nc < C) {
    radix_threshold<kCandKPT>(S, [&](int i, bool& v) { v = j0 + i < (int)C; return key[i]; }, nc, (int)C, T, k_eq);
  } else {
    // every candidate survives: T = the smallest key
    uint32_t mn = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < kCandKPT; ++i)
      if (j0 + i < (int)C) mn = min(mn, key[i]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) S.wa[warp] = mn;
    __syncthreads();
    if (warp == 0) {
      uint32_t x = S.wa[lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) S.bin = x;
    }
    __syncthreads();
    T = S.bin;
    __syncthreads();
  }
  const float Ts = from_ordered(T);
  const float M = S.M[0], Z = S.Z[0];
  const float pT = expf(Ts - M) / Z;
  const float win = tie_window(Ts, M);
  const bool exact_all = !(pT >= FLT_MIN);
  if (bmax > -INFINITY && (bmax > Ts - win || exact_all)) {
    if (tid == 0) p.fb_flags[row] = 1u;  // an excluded position might rank or tie: redo densely
    return;
  }

  uint32_t cls_gt = 0, cls_eq = 0;
#pragma unroll
  for (int i = 0; i < kCandKPT; ++i) {
    if (j0 + i >= (int)C) continue;
    const float sj = from_ordered(key[i]);
    if (sj > Ts + win) {
      cls_gt |= 1u << i;
    } else if (exact_all || sj >= Ts - win) {
      const float pj = expf(sj - M) / Z;
      if (pj > pT) cls_gt |= 1u << i;
      else if (pj == pT) cls_eq |= 1u << i;
    }
  }
  const uint32_t n_gt_local = __popc(cls_gt);
  uint32_t n_gt_total;
  {
    const uint32_t base = block_excl_scan(n_gt_local, S.wc);
    if (tid == kT - 1) S.need = base + n_gt_local;
    __syncthreads();
    n_gt_total = S.need;
    __syncthreads();
  }
  k_eq = (uint32_t)nc - n_gt_total;
  const uint32_t ceq = __popc(cls_eq);
  const uint32_t eq_base = block_excl_scan(ceq, S.wa);
  const uint32_t take = eq_base >= k_eq ? 0u : min(ceq, k_eq - eq_base);
  uint32_t o = block_excl_scan(n_gt_local + take, S.wb);
  uint32_t eqr = eq_base;
  float* wrow = p.w + ((size_t)b * p.n_kv + kvh) * nc;
#pragma unroll
  for (int i = 0; i < kCandKPT; ++i) {
    bool sel = (cls_gt >> i) & 1u;
    if ((cls_eq >> i) & 1u) {
      sel = eqr < k_eq;
      ++eqr;
    }
    if (sel) {
      idx[o] = csm[j0 + i].y;
      wrow[o] = expf(from_ordered(key[i]) - M) / Z;
      ++o;
    }
  }
  if (tid == 0) p.fb_flags[row] = 0u;
  __syncthreads();
  finish_group(S, p, b, kvh);
}

// arg_topk over raw floats: ordered-float keys, lowest index wins ties.
__global__ void __launch_bounds__(kT)
    arg_topk_kernel(const float* values, int n, int nc, uint32_t* keys, uint32_t* out) {
  __shared__ SelShared S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < n; j += kT) keys[j] = ordered_bits(values[j]);
  __syncthreads();
  uint32_t T = 0, k_eq = (uint32_t)nc;
  if (nc < n) {
    clear_hist(S);
    for (int base = 0; base < n; base += kT) {
      const int j = base + tid;
      hist_add(S.hist, (j < n ? keys[j] : 0u) >> 21, j < n, lane);
    }
    __syncthreads();
    find_bin(S, (uint32_t)nc);
    const uint32_t b0 = S.bin;
    uint32_t need = S.need;
    clear_hist(S);
    for (int base = 0; base < n; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < n ? keys[j] : 0u;
      hist_add(S.hist, (k >> 10) & 0x7ffu, j < n && (k >> 21) == b0, lane);
    }
    __syncthreads();
    find_bin(S, need);
    const uint32_t p01 = (b0 << 11) | S.bin;
    need = S.need;
    clear_hist(S);
    for (int base = 0; base < n; base += kT) {
      const int j = base + tid;
      const uint32_t k = j < n ? keys[j] : 0u;
      hist_add(S.hist, k & 0x3ffu, j < n && (k >> 10) == p01, lane);
    }
    __syncthreads();
    find_bin(S, need);
    T = (p01 << 10) | S.bin;
    k_eq = S.need;
  }
  const int seg = (((n + kNW - 1) / kNW) + 31) & ~31;
  const int w0 = warp * seg;
  const int w1 = min(n, w0 + seg);
  uint32_t cgt = 0, ceq = 0;
  for (int j0 = w0; j0 < w1; j0 += 32) {
    const int j = j0 + lane;
    const bool act = j < w1;
    const uint32_t k = act ? keys[j] : 0u;
    cgt += __popc(__ballot_sync(0xffffffffu, act && k > T));
    ceq += __popc(__ballot_sync(0xffffffffu, act && k == T));
  }
  const uint32_t eq_base = block_excl_scan(lane == 0 ? ceq : 0u, S.wa);
  const uint32_t take = eq_base >= k_eq ? 0u : min(ceq, k_eq - eq_base);
  uint32_t run_sel = block_excl_scan(lane == 0 ? cgt + take : 0u, S.wb);
  run_sel = __shfl_sync(0xffffffffu, run_sel, 0);
  uint32_t run_eq = __shfl_sync(0xffffffffu, eq_base, 0);
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
    if (sel) out[run_sel + __popc(bsel & lt)] = (uint32_t)j;
    run_eq += __popc(beq);
    run_sel += __popc(bsel);
  }
}

__global__ void __launch_bounds__(256) probs_kernel(const SelectParams p, float* probs) {
  __shared__ float sMZ[2];
  const int slot = blockIdx.x;  // b*n_q + head
  if (threadIdx.x < 32) {
    float m, z;
    softmax_stats(p.partials + (size_t)slot * p.max_splits, p.n_splits, threadIdx.x, m, z);
    if (threadIdx.x == 0) {
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

void select_launch(const SelectParams& p, cudaStream_t st) {
  // register-resident keys up to 32 per thread (s <= 32768); the lstride
  // padding (multiple of 32 floats) keeps the float4 loads in bounds.
  if (!p.force_global && p.G <= kMaxG) {
    if (p.s <= 4 * kT) { select_reg_kernel<4><<<p.rows, kT, 0, st>>>(p); return; }
    if (p.s <= 8 * kT) { select_reg_kernel<8><<<p.rows, kT, 0, st>>>(p); return; }
    if (p.s <= 16 * kT) { select_reg_kernel<16><<<p.rows, kT, 0, st>>>(p); return; }
    if (p.s <= 32 * kT) { select_reg_kernel<32><<<p.rows, kT, 0, st>>>(p); return; }
  }
  select_kernel<<<p.rows, kT, 0, st>>>(p);
}

bool select_cand_launch(const SelectParams& p, cudaStream_t st) {
  if (p.G != 1 || !p.cand || !p.fb_flags) return false;
  const size_t smem = (size_t)kT * kCandKPT * sizeof(uint2) + ((size_t)p.n_splits + 1) * 4;
  if (smem > 200 * 1024) return false;
  static unsigned long long configured = 0;  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(select_cand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured |= 1ull << (dev & 63);
  }
  select_cand_kernel<<<p.rows, kT, smem, st>>>(p);
  // dense redo of the flagged rows (CTAs of unflagged rows exit at once)
  SelectParams f = p;
  f.force_global = 0;
  select_launch(f, st);
  return true;
}

void probs_launch(const SelectParams& p, float* probs, cudaStream_t st) {
  probs_kernel<<<p.rows * p.G, 256, 0, st>>>(p, probs);
}

void arg_topk_launch(const float* values, int n, int k, uint32_t* keys_scratch, uint32_t* out,
                     cudaStream_t st) {
  const int nc = k < n ? k : n;
  arg_topk_kernel<<<1, kT, 0, st>>>(values, n, nc, keys_scratch, out);
}

}  // namespace kc

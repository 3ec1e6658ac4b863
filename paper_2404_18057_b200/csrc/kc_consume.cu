// kc_consume.cu -- dataflow consumer: per-row top-N selection + V recall +
// P.V, overlapped with the scoring kernel that produces the rows (sm_100a).
//
// Replaces, in one kernel, softmax normalisation (proj/core/src/matrix.cpp:45-61),
// arg_topk (matrix.cpp:109-122), the TopNSelection fill (attention.cpp:126-154),
// gather_v (kv_cache.cpp:150-187) and the P.V loop + add_scaled
// (attention.cpp:159-188, :23-27) -- with the exact rule of select_reg_kernel
// and recall_pv_kernel (kc_select.cu, kc_recall.cu), bit for bit: same keys,
// same threshold, same p-tie classification, same weights, the same reduction
// tree for dropped mass / renormaliser, the same P.V operation order.
//
// Why a consumer: the scoring kernel (HBM-bound, all SMs) finishes its
// (batch, kv-head) rows in order; each scoring CTA bumps its row's completion
// counter (release) after its logits and split statistics are written. A small
// persistent grid of these CTAs, launched on another stream, waits for a row's
// counter to reach n_splits (acquire) and then selects (and, for single-layer
// calls, recalls + reduces) that row while the scoring streams the later rows'
// K. The selection leaves the scoring stream's critical path (previously:
// score -> select in stream order, a full-GPU barrier-bound launch per layer).
// Multi-layer calls leave the recall to recall_pv_kernel on a side stream
// under the next layer's scoring: a consumer that also recalls slows the
// scoring it runs beside.
//
// Selection per row with 256 threads, keys streamed from L2 (no register-
// resident key array, so a consumer CTA fits beside two scoring CTAs):
//   1. global (M, Z) per q head from the split statistics (softmax_stats);
//   2. pass 1: each warp streams a contiguous segment of the row (coalesced
//      float4), lane (l, i mod 4) keeps a group maximum; tau = min over warps of
//      each warp's ceil(nc/8)-th largest group maximum is a lower bound of the
//      nc-th largest key (MHA: lowered by the p-tie window, as select_reg);
//   3. pass 2: keys >= tau are compacted per warp in position order (ballot
//      scan) into shared memory -- typically ~1.5 nc of them;
//   4. exact radix select on the candidates, p-exact tie classification, block
//      scans for position-ordered output (select_reg's fast path);
//   anything the fast path cannot prove (nc > 1024, > 1024 candidates or > 128
//   in one warp's segment, p(tau) not a normal float, nc >= s) takes the
//   streamed exact path: 3 radix passes over all keys + two ordered
//   classification passes.
// select_rows_cached_kernel runs the same row selection stream-ordered for GQA
// (one row per CTA, the selection values cached in shared memory).
#include <cfloat>

#include "kc_device.cuh"
#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace kc {

namespace {

constexpr int kCT = 256;                 // consumer threads
constexpr int kCW = kCT / 32;            // consumer warps
constexpr int kCandCap = 1024;           // candidates held in shared memory
constexpr int kWarpCap = kCandCap / kCW; // per-warp candidate region
constexpr int kCPT = kCandCap / kCT;     // candidates per thread (max)
constexpr int kCBins = 2048;
constexpr int kUnionBytes = 32 * 1024;   // candidate arrays / staged V rows
constexpr int kWsm = 2048;               // weights staged in smem when G*nc fits
constexpr int kFastMaxNc = 1024;         // 8 warps x 128 group maxima
constexpr int kMaxGq = 32;               // q heads per kv head (G*h <= 1024)
constexpr int kRedG = 8;                 // heads reduced per finish round
constexpr size_t kCachedSmemMax = 112 * 1024;  // select_rows_cached: two CTAs per SM

struct CShared {
  union {
    struct {
      uint32_t rkey[kCandCap];  // per-warp regions [kCW][kWarpCap]
      uint32_t rpos[kCandCap];
      uint32_t ckey[kCandCap];  // compacted, position order
      uint32_t cpos[kCandCap];
    } sel;
    uint32_t hist[kCBins];      // aliases rkey / rpos (dead once compacted)
    uint8_t vbuf[kUnionBytes];  // recall: staged V rows
  } u;
  float wsm[kWsm];              // [G][nc] weights
  float M[kMaxGq], Z[kMaxGq], rZ[kMaxGq], nrm[kMaxGq];
  uint32_t wa[kCW], wb[kCW], wc[kCW], wd[kCW];
  uint32_t bin, need, tot;
  float red_f[kRedG][32];
  double red_d[kRedG][32];
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// phase timestamps of one row (ConsumeParams::dbg, development probe)
#define KC_STAMP(k)                                                        \
  do {                                                                     \
    if (p.dbg && threadIdx.x == 0) p.dbg[(size_t)r.row * 8 + (k)] = globaltimer_ns(); \
  } while (0)

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Block-wide exclusive prefix sum over the 256 threads (thread order); the
// block total lands in *tot (read it before the next scan).
__device__ __forceinline__ uint32_t c_excl_scan(uint32_t x, uint32_t* wt, uint32_t* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) wt[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < kCW ? wt[lane] : 0u;
    uint32_t u = t;
#pragma unroll
    for (int o = 1; o < kCW; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += n;
    }
    if (lane < kCW) wt[lane] = u - t;
    if (lane == kCW - 1) *tot = u;
  }
  __syncthreads();
  const uint32_t r = wt[warp] + v - x;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void c_hist_add(uint32_t* hist, uint32_t bin, bool active, int lane) {
  const uint32_t key = active ? bin : 0xffffffffu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int leader = 31 - __clz(peers);
  if (active && lane == leader) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

__device__ __forceinline__ void c_clear_hist(CShared& S) {
  for (int i = threadIdx.x; i < kCBins; i += kCT) S.u.hist[i] = 0;
  __syncthreads();
}

// Among the bins, B with (count above B) < need <= (count at or above B):
// S.bin = B, S.need = need - (count above B). Thread t owns bins 8t..8t+7.
__device__ void c_find_bin(CShared& S, uint32_t need) {
  const int t = threadIdx.x;
  uint32_t h[8];
  uint32_t local = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    h[k] = S.u.hist[8 * t + k];
    local += h[k];
  }
  const uint32_t before = c_excl_scan(local, S.wa, &S.tot);
  uint32_t above = S.tot - before - local;
#pragma unroll
  for (int k = 7; k >= 0; --k) {
    if (above < need && above + h[k] >= need) {
      S.bin = 8 * t + k;
      S.need = need - above;
    }
    above += h[k];
  }
  __syncthreads();
}

// MSB-first radix select (11/11/10-bit digits) over items a thread owns:
// T = the nc-th largest key, k_eq = how many keys equal to T survive.
template <int KPT, typename Get>
__device__ __forceinline__ void c_radix_threshold(CShared& S, Get&& get, int nc, int n_valid, uint32_t& T,
                                                  uint32_t& k_eq) {
  const int lane = threadIdx.x & 31;
  T = 0;
  k_eq = (uint32_t)nc;
  if (nc >= n_valid) return;
  c_clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    if (__any_sync(0xffffffffu, v)) c_hist_add(S.u.hist, k >> 21, v, lane);
  }
  __syncthreads();
  c_find_bin(S, (uint32_t)nc);
  const uint32_t b0 = S.bin;
  uint32_t need = S.need;
  c_clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    const bool act = v && (k >> 21) == b0;
    if (__any_sync(0xffffffffu, act)) c_hist_add(S.u.hist, (k >> 10) & 0x7ffu, act, lane);
  }
  __syncthreads();
  c_find_bin(S, need);
  const uint32_t p01 = (b0 << 11) | S.bin;
  need = S.need;
  c_clear_hist(S);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool v;
    const uint32_t k = get(i, v);
    const bool act = v && (k >> 10) == p01;
    if (__any_sync(0xffffffffu, act)) c_hist_add(S.u.hist, k & 0x3ffu, act, lane);
  }
  __syncthreads();
  c_find_bin(S, need);
  T = (p01 << 10) | S.bin;
  k_eq = S.need;
}

// Selection key of position j (select_reg_kernel's keys, bit for bit):
// MHA the ordered logit bits, GQA the fp32 bits of sum_g p_g with the fast exp.
// GQ: the group size at compile time (1, 2, 4, 8), 0 = runtime G.
template <int GQ, int UB = 0>
struct RowKeys {
  static constexpr int kGQ = GQ;
  const float* lbase;  // the row's first q head's logits
  int64_t lstride;
  int G;
  const float* M;      // shared
  const float* rZ;
  float* kcache = nullptr;  // shared-memory copy of the row's values (pass 1 -> pass 2), or null
  static constexpr int kR = GQ > 0 ? GQ : 1;  // raw float4 per position quad
  // loads in flight per lane in a streaming pass: U position quads
  // loads in flight per lane in a streaming pass: U position quads (UB > 0:
  // set by the caller -- more registers, fewer round trips)
  static constexpr int U = UB > 0 ? UB : (GQ == 1 ? 8 : (GQ == 2 ? 4 : (GQ == 4 ? 2 : 1)));

  __device__ __forceinline__ int g_n() const { return GQ > 0 ? GQ : G; }

  __device__ __forceinline__ uint32_t key1(int j) const {
    if (g_n() == 1) return ordered_bits(__ldcg(lbase + j));
    float acc = 0.0f;
    for (int g = 0; g < g_n(); ++g) {
      const float pg = __expf(__ldcg(lbase + (size_t)g * lstride + j) - M[g]) * rZ[g];
      acc = (g == 0) ? pg : acc + pg;
    }
    return __float_as_uint(acc);
  }
  // raw logits of positions j..j+3 (16-B aligned) below `end` (GQ > 0 only)
  __device__ __forceinline__ void load(int j, int end, float4 (&x)[kR]) const {
    if (j + 3 < end) {
#pragma unroll
      for (int g = 0; g < kR; ++g) x[g] = __ldcg(reinterpret_cast<const float4*>(lbase + (size_t)g * lstride + j));
    } else {
#pragma unroll
      for (int g = 0; g < kR; ++g) {
        const float* l = lbase + (size_t)g * lstride + j;
        x[g].x = j < end ? __ldcg(l) : 0.0f;
        x[g].y = j + 1 < end ? __ldcg(l + 1) : 0.0f;
        x[g].z = j + 2 < end ? __ldcg(l + 2) : 0.0f;
        x[g].w = j + 3 < end ? __ldcg(l + 3) : 0.0f;
      }
    }
  }
  // Comparable values of a quad: MHA the logit (float order = key order),
  // GQA sum_g p_g (>= 0, float order = bit order); invalid positions get
  // kInvalid, below every threshold.
  static constexpr float kInvalid = GQ == 1 ? -INFINITY : -1.0f;
  __device__ __forceinline__ void vals(const float4 (&x)[kR], int j, int end, float (&f)[4]) const {
    if (GQ == 1) {
      f[0] = x[0].x;
      f[1] = x[0].y;
      f[2] = x[0].z;
      f[3] = x[0].w;
    } else {
#pragma unroll
      for (int g = 0; g < kR; ++g) {
        const float e[4] = {x[g].x, x[g].y, x[g].z, x[g].w};
        const float Mg = M[g], rz = rZ[g];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float pg = __expf(e[u] - Mg) * rz;
          f[u] = (g == 0) ? pg : f[u] + pg;
        }
      }
    }
    if (j + 3 >= end) {
#pragma unroll
      for (int u = 0; u < 4; ++u) f[u] = j + u < end ? f[u] : kInvalid;
    }
  }
  __device__ __forceinline__ float val1(int j) const {
    if (g_n() == 1) return __ldcg(lbase + j);
    return __uint_as_float(key1(j));
  }
  // key bits of a comparable value, and back
  __device__ __forceinline__ uint32_t key_of(float f) const {
    return g_n() == 1 ? ordered_bits(f) : __float_as_uint(f);
  }
  __device__ __forceinline__ float val_of(uint32_t k) const {
    return g_n() == 1 ? from_ordered(k) : __uint_as_float(k);
  }
  // U quads: it0.. of a warp segment starting at w0, lane offset 4*lane
  __device__ __forceinline__ void batch(int w0, int w1, int it0, int n_it, int lane, float (&f)[U][4]) const {
    if constexpr (GQ > 0) {
      float4 x[U][kR];
#pragma unroll
      for (int u = 0; u < U; ++u) load(w0 + (it0 + u) * 128 + 4 * lane, it0 + u < n_it ? w1 : 0, x[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) vals(x[u], w0 + (it0 + u) * 128 + 4 * lane, it0 + u < n_it ? w1 : 0, f[u]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = w0 + (it0 + u) * 128 + 4 * lane, end = it0 + u < n_it ? w1 : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) f[u][q] = j + q < end ? val1(j + q) : kInvalid;
      }
    }
  }
};

// p-exact classification of an MHA key against the threshold T (select_reg).
struct MhaClass {
  float Ts, M, Z, pT, win;
  bool exact_all;
  __device__ __forceinline__ void init(uint32_t T, float M_, float Z_) {
    Ts = from_ordered(T);
    M = M_;
    Z = Z_;
    pT = expf(Ts - M) / Z;
    win = tie_window(Ts, M);
    exact_all = !(pT >= FLT_MIN);
  }
  __device__ __forceinline__ void cls(uint32_t key, bool& gt, bool& eq) const {
    gt = eq = false;
    const float sj = from_ordered(key);
    if (sj > Ts + win) {
      gt = true;
    } else if (exact_all || sj >= Ts - win) {
      const float pj = expf(sj - M) / Z;
      gt = pj > pT;
      eq = pj == pT;
    }
  }
};

struct RowCtx {
  int b, kvh, row, G, n_q, nc, s;
  bool wsm_ok;
};

// weights of selected position `pos` (key `key`) at output slot o
template <class RK>
__device__ __forceinline__ void write_sel(const ConsumeParams& p, CShared& S, const RowCtx& r,
                                          const RK& rk, int o, uint32_t pos, uint32_t key) {
  p.idx[(size_t)r.row * r.nc + o] = pos;
  for (int g = 0; g < r.G; ++g) {
    const float sg = r.G == 1 ? from_ordered(key) : __ldcg(rk.lbase + (size_t)g * rk.lstride + pos);
    const float wv = expf(sg - S.M[g]) / S.Z[g];
    p.w[((size_t)r.b * r.n_q + r.kvh * r.G + g) * r.nc + o] = wv;
    if (r.wsm_ok) S.wsm[g * r.nc + o] = wv;
  }
}

// tau = min over warps of each warp's ceil(nc/8)-th largest of its lanes'
// four group maxima (keys): >= nc distinct positions hold keys >= tau. MHA:
// lowered by the p-tie window. Returns tau as a comparable value, or NaN when
// p(tau) is not a normal float (ties unbounded: exact path). Uniform.
template <class RK>
__device__ float bound_from_groups(const ConsumeParams& p, CShared& S, const RowCtx& r, const RK& rk,
                                   uint32_t (&gm)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kw = (r.nc + kCW - 1) / kCW;
  uint32_t kth = 0u;
  for (int rr = 0; rr < kw; ++rr) {
    const uint32_t m = max(max(gm[0], gm[1]), max(gm[2], gm[3]));
    kth = __reduce_max_sync(0xffffffffu, m);
    const uint32_t ball = __ballot_sync(0xffffffffu, m == kth);
    if (lane == __ffs(ball) - 1) {
      if (gm[0] == kth) gm[0] = 0u;
      else if (gm[1] == kth) gm[1] = 0u;
      else if (gm[2] == kth) gm[2] = 0u;
      else gm[3] = 0u;
    }
  }
  if (lane == 0) S.wd[warp] = kth;
  __syncthreads();
  uint32_t tau = S.wd[0];
#pragma unroll
  for (int w = 1; w < kCW; ++w) tau = min(tau, S.wd[w]);
  float tau_f = rk.val_of(tau);
  if (r.G == 1) {
    // a score just below tau can share the N-th score's p: lower the bound by
    // the tie window; p(tau) not a normal float -> unbounded ties, exact path
    const float ts = tau_f;
    if (!(expf(ts - S.M[0]) / S.Z[0] >= FLT_MIN)) return NAN;
    if (ts > -INFINITY) tau_f = from_ordered(ordered_bits(ts - 2.0f * tie_window(ts, S.M[0])));
  }
  (void)p;
  return tau_f;
}

// Candidates by two streaming passes over the row's logits (group maxima,
// then keys >= tau, compacted per warp in position order). Leaves them in
// ckey/cpos in position order; returns their count, or -1 (exact path).
template <class RK>
__device__ int cands_passes(const ConsumeParams& p, CShared& S, const RowCtx& r, const RK& rk) {
  constexpr int U = RK::U;
  constexpr int GQ = RK::kGQ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = r.s, nc = r.nc;
  (void)tid;
  (void)nc;
  const int seg = ((s + kCW * 128 - 1) / (kCW * 128)) * 128;
  const int w0 = warp * seg, w1 = min(s, w0 + seg);
  const int n_it = w1 > w0 ? (w1 - w0 + 127) / 128 : 0;

  // ---- pass 1: group maxima -> tau ----
  float gmf[4] = {RK::kInvalid, RK::kInvalid, RK::kInvalid, RK::kInvalid};
  for (int it0 = 0; it0 < n_it; it0 += U) {
    float f[U][4];
    rk.batch(w0, w1, it0, n_it, lane, f);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gmf[(it0 + u) & 3] = fmaxf(gmf[(it0 + u) & 3], fmaxf(fmaxf(f[u][0], f[u][1]), fmaxf(f[u][2], f[u][3])));
      if (rk.kcache && it0 + u < n_it)
        *reinterpret_cast<float4*>(rk.kcache + w0 + (it0 + u) * 128 + 4 * lane) =
            make_float4(f[u][0], f[u][1], f[u][2], f[u][3]);
    }
  }
  KC_STAMP(2);
  uint32_t gm[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) gm[i] = rk.key_of(GQ == 1 ? gmf[i] : fmaxf(gmf[i], 0.0f));
  const float tau_f = bound_from_groups(p, S, r, rk, gm);
  if (tau_f != tau_f) return -1;  // uniform

  // ---- pass 2: candidates (value >= tau), per-warp regions in position
  // order: position = w0 + 128 it + 4 lane + q, so (lane, q) order within a
  // quad row is position order -- ballot per q, prefix by popcounts ----
  uint32_t wcount = 0;
  const uint32_t lt = lanemask_lt();
  for (int it0 = 0; it0 < n_it; it0 += U) {
    float f[U][4];
    if (rk.kcache) {  // the values pass 1 kept (the same bits; invalid positions stayed kInvalid)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float4 x = it0 + u < n_it ? *reinterpret_cast<const float4*>(rk.kcache + w0 + (it0 + u) * 128 + 4 * lane)
                                        : make_float4(RK::kInvalid, RK::kInvalid,
                                                      RK::kInvalid, RK::kInvalid);
        f[u][0] = x.x;
        f[u][1] = x.y;
        f[u][2] = x.z;
        f[u][3] = x.w;
      }
    } else {
      rk.batch(w0, w1, it0, n_it, lane, f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool c0 = f[u][0] >= tau_f, c1 = f[u][1] >= tau_f, c2 = f[u][2] >= tau_f, c3 = f[u][3] >= tau_f;
      const uint32_t b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
      const uint32_t b2 = __ballot_sync(0xffffffffu, c2), b3 = __ballot_sync(0xffffffffu, c3);
      if ((b0 | b1 | b2 | b3) == 0u) continue;  // warp-uniform
      const int j = w0 + (it0 + u) * 128 + 4 * lane;
      uint32_t o = wcount + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
      const bool cc[4] = {c0, c1, c2, c3};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cc[q]) {
          if (o < (uint32_t)kWarpCap) {
            S.u.sel.rkey[warp * kWarpCap + o] = rk.key_of(f[u][q]);
            S.u.sel.rpos[warp * kWarpCap + o] = (uint32_t)(j + q);
          }
          ++o;
        }
      }
      wcount += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
    }
  }
  if (lane == 0) S.wc[warp] = wcount;
  __syncthreads();
  uint32_t C = 0, base = 0;
  bool over = false;
#pragma unroll
  for (int w = 0; w < kCW; ++w) {
    const uint32_t cw = S.wc[w];
    over |= cw > (uint32_t)kWarpCap;
    if (w < warp) base += cw;
    C += cw;
  }
  KC_STAMP(3);
  if (over) return -1;  // uniform
  for (uint32_t e = lane; e < S.wc[warp]; e += 32) {
    S.u.sel.ckey[base + e] = S.u.sel.rkey[warp * kWarpCap + e];
    S.u.sel.cpos[base + e] = S.u.sel.rpos[warp * kWarpCap + e];
  }
  __syncthreads();
  return (int)C;
}

// Fast path: bound -> candidates -> exact select. false: take the exact path
// (nothing written).
template <class RK>
__device__ bool select_fast(const ConsumeParams& p, CShared& S, const RowCtx& r, const RK& rk) {
  const int tid = threadIdx.x;
  const int s = r.s, nc = r.nc;
  if (nc >= s || nc > kFastMaxNc) return false;
  const int Ci = cands_passes(p, S, r, rk);
  if (Ci < 0) return false;
  const uint32_t C = (uint32_t)Ci;

  // ---- exact selection among the C candidates (thread t: [t*cpt, t*cpt+cpt)) ----
  const int cpt = (int)((C + kCT - 1) / kCT);
  uint32_t ck[kCPT], cp[kCPT];
  bool have[kCPT];
#pragma unroll
  for (int k = 0; k < kCPT; ++k) {
    const int e = tid * cpt + k;
    have[k] = k < cpt && e < (int)C;
    ck[k] = have[k] ? S.u.sel.ckey[e] : 0u;
    cp[k] = have[k] ? S.u.sel.cpos[e] : 0u;
  }
  uint32_t T, k_eq;
  c_radix_threshold<kCPT>(S, [&](int i, bool& v) { v = have[i]; return ck[i]; }, nc, (int)C, T, k_eq);
  bool gt[kCPT], eq[kCPT];
  if ((uint32_t)nc >= C) {
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
      gt[k] = have[k];
      eq[k] = false;
    }
  } else if (r.G == 1) {
    MhaClass mc;
    mc.init(T, S.M[0], S.Z[0]);
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
      gt[k] = eq[k] = false;
      if (have[k]) mc.cls(ck[k], gt[k], eq[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
      gt[k] = have[k] && ck[k] > T;
      eq[k] = have[k] && ck[k] == T;
    }
  }
  uint32_t ngt = 0, neq = 0;
#pragma unroll
  for (int k = 0; k < kCPT; ++k) {
    ngt += gt[k] ? 1u : 0u;
    neq += eq[k] ? 1u : 0u;
  }
  c_excl_scan(ngt, S.wc, &S.tot);
  const uint32_t keq = (uint32_t)nc - S.tot;
  uint32_t eqr = c_excl_scan(neq, S.wa, &S.tot);
  bool sel[kCPT];
  uint32_t nsel = 0;
#pragma unroll
  for (int k = 0; k < kCPT; ++k) {
    sel[k] = gt[k];
    if (eq[k]) {
      sel[k] = eqr < keq;
      ++eqr;
    }
    nsel += sel[k] ? 1u : 0u;
  }
  uint32_t o = c_excl_scan(nsel, S.wb, &S.tot);
#pragma unroll
  for (int k = 0; k < kCPT; ++k) {
    if (sel[k]) {
      write_sel(p, S, r, rk, (int)o, cp[k], ck[k]);
      ++o;
    }
  }
  return true;
}

// Exact path for any row: streamed radix threshold over every key, then two
// ordered classification passes (per-warp contiguous segments).
template <class RK>
__device__ void select_exact(const ConsumeParams& p, CShared& S, const RowCtx& r, const RK& rk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = r.s, nc = r.nc;
  const bool all = nc >= s;
  uint32_t T = 0;
  if (!all) {
    // radix digits over streamed keys (every lane runs every iteration)
    uint32_t prefix = 0, need = (uint32_t)nc;
    for (int d = 0; d < 3; ++d) {
      // digit d: key bits [21,32) / [10,21) / [0,10); keys must match the
      // digits found so far
      const int shift = d == 0 ? 21 : (d == 1 ? 10 : 0);
      const uint32_t dmask = d == 2 ? 0x3ffu : 0x7ffu;
      c_clear_hist(S);
      for (int j0 = 0; j0 < s; j0 += kCT) {
        const int j = j0 + tid;
        const bool valid = j < s;
        const uint32_t key = valid ? rk.key1(j) : 0u;
        const bool act = valid && (d == 0 || (key >> (d == 1 ? 21 : 10)) == prefix);
        if (__any_sync(0xffffffffu, act)) c_hist_add(S.u.hist, (key >> shift) & dmask, act, lane);
      }
      __syncthreads();
      c_find_bin(S, need);
      prefix = d == 0 ? S.bin : ((prefix << (d == 1 ? 11 : 10)) | S.bin);
      need = S.need;
    }
    T = prefix;
  }
  MhaClass mc;
  if (!all && r.G == 1) mc.init(T, S.M[0], S.Z[0]);
  auto classify = [&](int j, bool valid, bool& gt, bool& eq) {
    gt = eq = false;
    if (!valid) return;
    if (all) {
      gt = true;
      return;
    }
    const uint32_t key = rk.key1(j);
    if (r.G == 1) {
      mc.cls(key, gt, eq);
    } else {
      gt = key > T;
      eq = key == T;
    }
  };
  const int seg = ((s + kCW * 32 - 1) / (kCW * 32)) * 32;
  const int w0 = warp * seg, w1 = min(s, w0 + seg);
  const int n_it = w1 > w0 ? (w1 - w0 + 31) / 32 : 0;
  uint32_t ngt = 0, neq = 0;
  for (int it = 0; it < n_it; ++it) {
    const int j = w0 + it * 32 + lane;
    bool gt, eq;
    classify(j, j < w1, gt, eq);
    ngt += __popc(__ballot_sync(0xffffffffu, gt));
    neq += __popc(__ballot_sync(0xffffffffu, eq));
  }
  if (lane == 0) {
    S.wa[warp] = ngt;
    S.wb[warp] = neq;
  }
  __syncthreads();
  uint32_t gbase = 0, ebase = 0, n_gt = 0;
#pragma unroll
  for (int w = 0; w < kCW; ++w) {
    if (w < warp) {
      gbase += S.wa[w];
      ebase += S.wb[w];
    }
    n_gt += S.wa[w];
  }
  const uint32_t keq = (uint32_t)nc - n_gt;
  const uint32_t lt = lanemask_lt();
  for (int it = 0; it < n_it; ++it) {
    const int j = w0 + it * 32 + lane;
    bool gt, eq;
    classify(j, j < w1, gt, eq);
    const uint32_t bg = __ballot_sync(0xffffffffu, gt), be = __ballot_sync(0xffffffffu, eq);
    const uint32_t gb = gbase + __popc(bg & lt), eb = ebase + __popc(be & lt);
    if (gt || (eq && eb < keq)) write_sel(p, S, r, rk, (int)(gb + min(eb, keq)), (uint32_t)j, rk.key1(j));
    gbase += __popc(bg);
    ebase += __popc(be);
  }
}

// dropped mass and renormaliser per q head: select_reg's 1024-thread reduction
// tree emulated (virtual warp vw = elements 32vw..32vw+31 (+1024k), xor
// butterflies, then a butterfly over the 32 warp partials), bit for bit.
__device__ void finish_rows(const ConsumeParams& p, CShared& S, const RowCtx& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nc = r.nc;
  for (int g0 = 0; g0 < r.G; g0 += kRedG) {
    const int ng = min(kRedG, r.G - g0);
    for (int item = warp; item < ng * 32; item += kCW) {
      const int gl = item >> 5, vw = item & 31, g = g0 + gl;
      if (vw * 32 >= nc) {  // no weights: exact zeros (x + 0 == x keeps the tree's result)
        if (lane == 0) {
          S.red_d[gl][vw] = 0.0;
          S.red_f[gl][vw] = 0.0f;
        }
        continue;
      }
      const size_t slot = (size_t)r.b * r.n_q + r.kvh * r.G + g;
      const float* wg = r.wsm_ok ? S.wsm + g * nc : p.w + slot * nc;
      double md = 0.0;
      float fs = 0.0f;
      for (int e = vw * 32 + lane; e < nc; e += 1024) {
        const float x = r.wsm_ok ? wg[e] : __ldcg(wg + e);
        md += (double)x;
        fs += x;
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        md += __shfl_xor_sync(0xffffffffu, md, o);
        fs += __shfl_xor_sync(0xffffffffu, fs, o);
      }
      if (lane == 0) {
        S.red_d[gl][vw] = md;
        S.red_f[gl][vw] = fs;
      }
    }
    __syncthreads();
    if (warp < ng) {
      const int g = g0 + warp;
      double a = S.red_d[warp][lane];
      float f = S.red_f[warp][lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        f += __shfl_xor_sync(0xffffffffu, f, o);
      }
      if (lane == 0) {
        const size_t slot = (size_t)r.b * r.n_q + r.kvh * r.G + g;
        const float nr = f > 0.0f ? 1.0f / f : 1.0f;
        p.dropped[slot] = 1.0 - a;
        p.norm[slot] = nr;
        S.nrm[g] = nr;
      }
    }
    __syncthreads();
  }
}

// V recall of the row's selected positions + P.V (recall_pv_kernel's order).
template <typename T>
__device__ void recall_row(const ConsumeParams& p, CShared& S, const RowCtx& r) {
  const int tid = threadIdx.x;
  const int h = p.h, G = r.G, nc = r.nc;
  const int rowb = h * (int)sizeof(T);
  const int rc_max = kUnionBytes / rowb;
  const T* vslot = static_cast<const T*>(p.v) + (size_t)r.row * p.max_seq * h;
  const uint32_t* idx = p.idx + (size_t)r.row * nc;
  T* vbuf = reinterpret_cast<T*>(S.u.vbuf);
  const int n_out = G * h;
  constexpr int kMaxOut = 4;  // G*h <= 1024
  float acc[kMaxOut];
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) acc[i] = 0.0f;
  const uint64_t pol = l2_evict_first_policy();
  const int n_chunks = (nc + rc_max - 1) / rc_max;
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int chunk = p.reverse ? (n_chunks - 1 - ci) : ci;
    const int c0 = chunk * rc_max;
    const int rc = min(rc_max, nc - c0);
    if ((rowb & 15) == 0) {
      const int vpr = rowb >> 4;
      const int total = rc * vpr;
      uint4* dst = reinterpret_cast<uint4*>(vbuf);
      constexpr int kBatch = 8;
      for (int v0 = tid; v0 < total; v0 += kCT * kBatch) {
        uint4 tmp[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int v = v0 + u * kCT;
          if (v < total) {
            const int rr = v / vpr, part = v - rr * vpr;
            tmp[u] = ld_stream16(reinterpret_cast<const uint4*>(vslot + (size_t)__ldcg(idx + c0 + rr) * h) + part, pol);
          }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int v = v0 + u * kCT;
          if (v < total) dst[v] = tmp[u];
        }
      }
    } else {
      for (int e = tid; e < rc * h; e += kCT) {
        const int rr = e / h, c = e - rr * h;
        vbuf[e] = vslot[(size_t)__ldcg(idx + c0 + rr) * h + c];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kMaxOut; ++i) {
      const int o = tid + i * kCT;
      if (o < n_out) {
        const int g = o / h, c = o - g * h;
        const size_t slot = (size_t)r.b * r.n_q + r.kvh * G + g;
        // weights: staged in shared memory, or this kernel's global writes (L2)
        const float* wg = r.wsm_ok ? S.wsm + g * nc + c0 : p.w + slot * nc + c0;
        const float nr = S.nrm[g];
        auto wat = [&](int rr) { return r.wsm_ok ? wg[rr] : __ldcg(wg + rr); };
        float a = acc[i];
        if (!p.reverse) {
          for (int rr = 0; rr < rc; ++rr) {
            const float w = p.renormalize ? __fmul_rn(wat(rr), nr) : wat(rr);
            a = __fadd_rn(a, __fmul_rn(w, to_f32<T>(vbuf[rr * h + c])));
          }
        } else {
          for (int rr = rc - 1; rr >= 0; --rr) {
            const float w = p.renormalize ? __fmul_rn(wat(rr), nr) : wat(rr);
            a = __fadd_rn(a, __fmul_rn(w, to_f32<T>(vbuf[rr * h + c])));
          }
        }
        acc[i] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) {
    const int o = tid + i * kCT;
    if (o < n_out) {
      const int g = o / h, c = o - g * h;
      p.out[((size_t)r.b * r.n_q + r.kvh * G + g) * h + c] = acc[i];
    }
  }
}

// Wait until every split of `row` is scored (counter == n_splits), then reset
// the counter for the next use of this buffer slot. A row that never completes
// (a scheduling bug) traps after ~4 s instead of hanging the GPU.
__device__ __forceinline__ void wait_row(const ConsumeParams& p, int row) {
  if (threadIdx.x == 0 && p.row_done) {
    // one 128-B line per row: the polls of different rows hit different L2
    // slices; relaxed polls with back-off (long while the row has not
    // started), one acquire fence once it is complete
    uint32_t* ctr = p.row_done + (size_t)row * kRowDoneStride;
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0, v;
    while ((v = ld_relaxed_u32(ctr)) < (uint32_t)p.n_splits) {
      __nanosleep(v == 0 ? 1000 : 200);
      if ((++spins & 255u) == 0 && globaltimer_ns() - t0 > 4000000000ull) {
        if (p.err) atomicExch(p.err, 1u);
        __trap();
      }
    }
    __threadfence();
    *ctr = 0u;
  }
  __syncthreads();
}

// One row's selection (stats, bound, candidates, exact select, dropped mass /
// renormaliser, dead-logit discard): shared by the consumer and the
// stream-ordered cached row selection. kcache: shared memory for the row's
// selection values (pass 1 -> pass 2), or null.
template <int GQ, int UB = 0>
__device__ __forceinline__ void select_row(const ConsumeParams& p, CShared& S, const RowCtx& r,
                                           float* kcache = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = r.G, n_q = r.n_q;
  for (int g = warp; g < G; g += kCW) {
    float m, z;
    softmax_stats<true>(p.partials + ((size_t)r.b * n_q + r.kvh * G + g) * p.max_splits, p.n_splits, lane, m, z);
    if (lane == 0) {
      S.M[g] = m;
      S.Z[g] = z;
      S.rZ[g] = 1.0f / z;
    }
  }
  __syncthreads();
  KC_STAMP(1);
  RowKeys<GQ, UB> rk;
  rk.lbase = p.logits + ((size_t)r.b * n_q + r.kvh * G) * p.lstride;
  rk.lstride = p.lstride;
  rk.G = G;
  rk.M = S.M;
  rk.rZ = S.rZ;
  rk.kcache = kcache;
  if (!select_fast(p, S, r, rk)) {
    __syncthreads();
    select_exact(p, S, r, rk);
  }
  __syncthreads();
  KC_STAMP(4);
  finish_rows(p, S, r);
  KC_STAMP(5);
  if (!p.keep_logits) {
    // the row's logits are dead: drop them from L2 without write-back
    const int lines = (p.s * 4 + 127) / 128;
    for (int e = threadIdx.x; e < G * lines; e += kCT) {
      const int g = e / lines, l = e - g * lines;
      discard_l2_line(reinterpret_cast<const char*>(rk.lbase + (size_t)g * p.lstride) + (size_t)l * 128);
    }
  }
}

__device__ __forceinline__ RowCtx row_ctx(const ConsumeParams& p, int row) {
  RowCtx r;
  r.row = row;
  r.b = row / p.n_kv;
  r.kvh = row - r.b * p.n_kv;
  r.G = p.G;
  r.n_q = p.n_kv * p.G;
  r.nc = p.nc;
  r.s = p.s;
  r.wsm_ok = p.G * p.nc <= kWsm;
  return r;
}

template <typename T, int GQ, int UB>
__device__ __forceinline__ void consume_rows(const ConsumeParams& p, CShared& S) {
  for (int row = p.row0 + blockIdx.x; row < p.row0 + p.rows; row += gridDim.x) {
    RowCtx r = row_ctx(p, row);
    KC_STAMP(7);
    wait_row(p, row);
    KC_STAMP(0);
    select_row<GQ, UB>(p, S, r);
    if (p.v) recall_row<T>(p, S, r);  // null: selection only
    KC_STAMP(6);
  }
}

template <typename T, int GQ>
__global__ void __maxnreg__(88) consume_kernel(const ConsumeParams p) {
  __shared__ CShared S;
  consume_rows<T, GQ, 0>(p, S);
}


// Stream-ordered GQA selection: one row per CTA, the row's selection values
// (sum_g p_g, G exp per position) computed once in pass 1 and kept in shared
// memory for pass 2; two CTAs per SM hold all 256 rows of C3 in one wave
// (select_reg_kernel: one 1024-thread CTA per SM, 1.73 waves).
// quads in flight per lane in the cached kernel's pass 1 (up to 128 registers)
template <int GQ>
constexpr int kCachedU = GQ <= 2 ? 8 : (GQ == 4 ? 4 : 2);

template <int GQ>
__global__ void __launch_bounds__(kCT, 2) select_rows_cached_kernel(const ConsumeParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CShared& S = *reinterpret_cast<CShared*>(smem_raw);
  float* kc = reinterpret_cast<float*>(smem_raw + ((sizeof(CShared) + 15) & ~size_t(15)));
  for (int row = p.row0 + blockIdx.x; row < p.row0 + p.rows; row += gridDim.x) {
    const RowCtx r = row_ctx(p, row);
    KC_STAMP(7);
    KC_STAMP(0);
    select_row<GQ, kCachedU<GQ>>(p, S, r, kc);
    KC_STAMP(6);
  }
}

template <int GQ>
bool launch_cached(const ConsumeParams& p, size_t smem, cudaStream_t st) {
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured[dev & 63] < (int)smem) {
    if (cudaFuncSetAttribute(select_rows_cached_kernel<GQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    configured[dev & 63] = (int)smem;
  }
  select_rows_cached_kernel<GQ><<<p.rows, kCT, smem, st>>>(p);
  return true;
}

template <typename T>
void launch_g(const ConsumeParams& p, int grid, cudaStream_t st) {
  switch (p.G) {
    case 1: consume_kernel<T, 1><<<grid, kCT, 0, st>>>(p); break;
    case 2: consume_kernel<T, 2><<<grid, kCT, 0, st>>>(p); break;
    case 4: consume_kernel<T, 4><<<grid, kCT, 0, st>>>(p); break;
    case 8: consume_kernel<T, 8><<<grid, kCT, 0, st>>>(p); break;
    default: consume_kernel<T, 0><<<grid, kCT, 0, st>>>(p); break;
  }
}

}  // namespace

bool select_rows_cached_launch(const ConsumeParams& p, cudaStream_t st) {
  // the cache covers every position a warp segment can touch (s + 127)
  const size_t smem = ((sizeof(CShared) + 15) & ~size_t(15)) + ((size_t)p.s + 128) * sizeof(float);
  if (smem > kCachedSmemMax) return false;
  switch (p.G) {
    case 2: return launch_cached<2>(p, smem, st);
    case 4: return launch_cached<4>(p, smem, st);
    case 8: return launch_cached<8>(p, smem, st);
    default: return false;
  }
}

bool consume_supported(int G, int h) { return G >= 1 && G <= kMaxGq && G * h <= 1024 && h >= 1; }

void consume_launch(const ConsumeParams& p, int vdtype, int grid, cudaStream_t st) {
  grid = grid > 0 ? std::min(grid, p.rows) : p.rows;
  if (grid < 1) grid = 1;
  switch (vdtype) {
    case KC_F16: launch_g<__half>(p, grid, st); break;
    case KC_BF16: launch_g<__nv_bfloat16>(p, grid, st); break;
    default: launch_g<float>(p, grid, st); break;
  }
}

}  // namespace kc

// kc_score.cu -- split-sequence q.K^T scoring kernel (sm_100a).
//
// Replaces head_weights + dot_scaled (proj/core/src/attention.cpp:15-21,66-78)
// and the max/sum half of softmax_inplace (proj/core/src/matrix.cpp:45-61).
//
// Work items are (row, split): row = b*n_kv + kv_head, split = a chunk of
// positions. A row's K for one split is one contiguous run of chunk*h
// elements in the [b][kv][pos][h] arena; one CTA per item (the hardware block
// scheduler balances the items against the recall kernel that runs
// concurrently on the side stream -- a persistent grid measured 20-25 %
// slower). In each CTA one elected producer lane streams K stages (64 positions = 16 KB)
// into a STAGES-deep shared-memory ring with 1-D TMA bulk copies
// (cp.async.bulk, L2 evict-first) on mbarriers; eight consumer warps score
// them against every q head of the GQA group held in registers (the K tile is
// read from HBM once per kv head, not once per q head). Each lane owns 128/LPR
// elements of a row (LPR lanes per row, 16-B chunks rotated per row so a
// quarter-warp's 16-B shared loads hit eight distinct bank groups), FMA in
// fp32, log2(LPR) xor-shuffles per row. Writes fp32 logits (score * scale, the
// multiply after the sum like dot_scaled) and a per-split online (max, sum
// exp) per q head; softmax_stats combines the splits into the global softmax.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kc_device.cuh"
#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace kc {

namespace {

constexpr int kRows = 64;     // positions per pipeline stage
constexpr int kCWarps = 8;    // consumer warps
constexpr int kH = 128;       // head_dim of the fast path
constexpr int kMaxCandChunk = 2048;  // candidate mode: positions per split held in smem
// MHA scoring: 3 CTAs / SM (<= 72 registers, no spills). Without the bound
// ptxas takes 82 and the SM holds only two: C2 330 -> 310 us per layer
// scoring inside the pipelined step, candidate mode 40k 463 -> 418 us.
#ifndef KC_MHA_MINB
#define KC_MHA_MINB 3
#endif

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Dataflow signal (kc_consume.cu): after the barrier that follows the item's
// last logits / statistics write, one thread publishes the split at GPU scope
// (fence + relaxed add = release; the consumer's acquire load pairs with it).
__device__ __forceinline__ void signal_row(const ScoreParams& p, int row) {
  if (p.row_done && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p.row_done + (size_t)row * kRowDoneStride, 1u);
  }
}

template <int LPR>
__device__ __forceinline__ int chunk_of(int ci, int rl, int sub) {
  if constexpr (LPR == 4) {
    return ((ci ^ (rl & 1)) << 2) | sub;
  } else {
    return ci * LPR + sub;
  }
}

// ---- the K stream shared by the scoring kernels ----------------------------
// Producer warp: lane 0 streams the items' K runs (one contiguous run of
// chunk*h elements per (row, split) in the [b][kv][pos][h] arena) into a
// STAGES-deep ring of 64-position stages with 1-D TMA bulk copies
// (cp.async.bulk) on mbarriers, under an L2 evict-first policy: a decode step
// streams the whole K cache exactly once, so its lines should be the first
// to leave L2 (they are never dropped without write-back -- the cache data
// stays defined whatever the L2 state).
template <typename T, int STAGES>
__device__ __forceinline__ void produce_k(const ScoreParams& p, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                          int lane, int n_items) {
  constexpr int ROWB = kH * (int)sizeof(T);
  const uint64_t pol = l2_policy(p.k_policy);
  uint32_t g = 0;  // global stage counter across items
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int row = p.row0 + item / p.n_splits;
    const int split = item - (row - p.row0) * p.n_splits;
    const int pos0 = split * p.chunk;
    const int npos = min(p.chunk, p.s - pos0);
    const int n_it = (npos + kRows - 1) / kRows;
    const T* kslot = static_cast<const T*>(p.k) + (size_t)row * p.max_seq * kH;
    if (p.tlb_ahead > 0 && lane == 0) {
      // warm the address translation of a row the CTAs launched ~3 waves
      // later will stream (one touch per 2 MB page of its K run): their
      // first TMA then does not queue behind the recall's page walks
      const int r2 = row + p.tlb_ahead;
      const size_t row_bytes = (size_t)p.s * ROWB;
      const size_t off = (size_t)split << 21;
      if (r2 < p.row0 + p.rows && off < row_bytes) {
        const char* a = reinterpret_cast<const char*>(static_cast<const T*>(p.k) + (size_t)r2 * p.max_seq * kH) + off;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
    if (lane == 0) {
      for (int it = 0; it < n_it; ++it, ++g) {
        const int st = (int)(g % STAGES);
        if (g >= (uint32_t)STAGES) mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
        const int pstart = pos0 + it * kRows;
        const int rows = min(kRows, npos - it * kRows);
        const uint32_t bytes = (uint32_t)(rows * ROWB);
        mbar_arrive_expect_tx(&full[st], bytes);
        tma_bulk_g2s(ring + st * kRows * ROWB, kslot + (size_t)pstart * kH, bytes, &full[st], pol);
      }
    }
  }
}

// Candidate epilogue of one split (MHA): scb[0..npos) holds the split's
// scores. tau = the minimum over the 8 consumer warps of each warp's
// ceil(nc/8)-th largest thread maximum is a lower bound of the split's nc-th
// largest score (>= nc threads each hold a score >= tau; the exact nc-th
// largest of the 256 maxima cost an all-pairs scan, +20 % instructions per
// split), so every position below tau has >= nc positions of this
// split strictly above it in p (p = exp(s - M)/Z is monotone in s) and can
// never be selected -- except through a p-tie, which needs |s - tau| within a
// few ulps: the bound keeps a window of 2^-9 (1 + |tau| + |max|) below tau.
// The selection kernel re-checks that window against the row's actual N-th
// score and recomputes the row densely if it is ever too narrow.
__device__ __forceinline__ void emit_candidates(const float* scb, float* mx, uint32_t* wcnt, int npos,
                                                int nc, int pos0, uint2* cand, uint2* meta) {
  constexpr int NT = kCWarps * 32;
  const int ct = threadIdx.x;  // 0..255 (consumer warps)
  const int lane = ct & 31, warp = ct >> 5;
  float* mred = mx;            // [kCWarps] per-warp bound
  float* mtop = mx + kCWarps;  // [kCWarps] per-warp maximum
  // thread ct owns the contiguous positions [a, e) of the split
  const int ppt = (npos + NT - 1) / NT;
  const int a = min(npos, ct * ppt), e = min(npos, a + ppt);
  float bound = -INFINITY;
  if (npos > nc) {
    float m = -INFINITY;
    for (int j = a; j < e; ++j) m = fmaxf(m, scb[j]);
    // tau = min over warps of the warp's kw-th largest thread maximum
    // (kw = ceil(nc / 8)): every warp holds >= kw maxima >= tau, so >= nc
    // positions of the split score >= tau. Warp-local (REDUX + BALLOT on
    // order-preserving bits), one barrier.
    const int kw = (nc + kCWarps - 1) / kCWarps;
    const uint32_t um = __float_as_uint(m);
    uint32_t v = (um & 0x80000000u) ? ~um : (um | 0x80000000u), kth = 0, top = 0;
    for (int r = 0; r < kw; ++r) {
      kth = __reduce_max_sync(0xffffffffu, v);
      top = r == 0 ? kth : top;
      const uint32_t ball = __ballot_sync(0xffffffffu, v == kth);
      if (lane == __ffs(ball) - 1) v = 0u;
    }
    auto unord = [](uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); };
    if (lane == 0) {
      mred[warp] = unord(kth);
      mtop[warp] = unord(top);
    }
    named_sync(1, NT);
    float tau = mred[0], smax = mtop[0];
#pragma unroll
    for (int w = 1; w < kCWarps; ++w) {
      tau = fminf(tau, mred[w]);
      smax = fmaxf(smax, mtop[w]);
    }
    if (tau > -INFINITY) bound = tau - 0x1p-9f * (1.0f + fabsf(tau) + fabsf(smax));
  }
  // ordered compaction: count, block exclusive scan, write in position order
  uint32_t cnt = 0;
  for (int j = a; j < e; ++j) cnt += scb[j] >= bound ? 1u : 0u;
  uint32_t v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) wcnt[warp] = v;
  named_sync(1, NT);
  uint32_t off = v - cnt, tot = 0;
#pragma unroll
  for (int w = 0; w < kCWarps; ++w) {
    const uint32_t c = wcnt[w];
    off += (w < warp) ? c : 0u;
    tot += c;
  }
  for (int j = a; j < e; ++j) {
    const float x = scb[j];
    if (x >= bound) cand[off++] = make_uint2(__float_as_uint(x), (uint32_t)(pos0 + j));
  }
  if (ct == 0) *meta = make_uint2(tot, __float_as_uint(bound));
}

template <typename T, int G, int LPR, int STAGES, bool CAND>
__global__ void __launch_bounds__((kCWarps + 1) * 32, (G >= 2 ? 2 : KC_MHA_MINB))
    score_fast_kernel(const ScoreParams p) {
  constexpr int CPL = 16 / LPR;            // 16-B chunks per lane per row
  constexpr int RPP = 32 / LPR;            // rows per warp pass
  constexpr int PASSES = (kRows / kCWarps) / RPP;
  constexpr int ROWB = kH * (int)sizeof(T);  // 256 B
  static_assert(G <= LPR, "one writer lane per q head");

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kRows * ROWB);
  uint64_t* empty = full + STAGES;
  float2* red = reinterpret_cast<float2*>(empty + STAGES);  // [kCWarps][G]
  // candidate mode: the split's scores, block maxima, warp counts
  float* scb = reinterpret_cast<float*>(red + kCWarps * G);  // [chunk]
  float* mx = scb + (CAND ? p.chunk : 0);                     // [2 * kCWarps]
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(mx + 2 * kCWarps);
  static_assert(!CAND || G == 1, "candidate mode ranks raw scores: MHA only");

  const int n_items = p.rows * p.n_splits;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kCWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kCWarps) {
    produce_k<T, STAGES>(p, ring, full, empty, lane, n_items);
    return;
  }

  // ---------------- consumers ----------------
  const int sub = lane % LPR;
  const int rl = lane / LPR;
  const int n_q = p.n_kv * G;
  uint32_t g = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int row = p.row0 + item / p.n_splits;
    const int split = item - (row - p.row0) * p.n_splits;
    const int b = row / p.n_kv;
    const int kvh = row - b * p.n_kv;
    const int pos0 = split * p.chunk;
    const int npos = min(p.chunk, p.s - pos0);
    const int n_it = (npos + kRows - 1) / kRows;
    float qf[G][CPL][8];
#pragma unroll
    for (int gh = 0; gh < G; ++gh) {
      const float* qh = p.q + ((size_t)b * n_q + kvh * G + gh) * kH;
#pragma unroll
      for (int ci = 0; ci < CPL; ++ci) {
        const int c = chunk_of<LPR>(ci, rl, sub);
        const float4 a = *reinterpret_cast<const float4*>(qh + c * 8);
        const float4 bq = *reinterpret_cast<const float4*>(qh + c * 8 + 4);
        qf[gh][ci][0] = a.x; qf[gh][ci][1] = a.y; qf[gh][ci][2] = a.z; qf[gh][ci][3] = a.w;
        qf[gh][ci][4] = bq.x; qf[gh][ci][5] = bq.y; qf[gh][ci][6] = bq.z; qf[gh][ci][7] = bq.w;
      }
    }
    float m_run = -INFINITY, l_run = 0.0f;
    float* lrow = p.logits + ((size_t)b * n_q + kvh * G + (sub < G ? sub : 0)) * p.lstride + pos0;

    for (int it = 0; it < n_it; ++it, ++g) {
      const int st = (int)(g % STAGES);
      mbar_wait(&full[st], (g / STAGES) & 1);
      const uint8_t* sb = ring + st * kRows * ROWB;
#pragma unroll
      for (int pass = 0; pass < PASSES; ++pass) {
        const int r = warp * (kRows / kCWarps) + pass * RPP + rl;
        const int pl = it * kRows + r;
        const uint4* srow = reinterpret_cast<const uint4*>(sb + r * ROWB);
        float acc[G];
        if constexpr (G == 1) {
          // MHA: one fmaf chain in element order (the candidate-mode dense
          // redo in kc_select.cu reproduces this exact sequence)
          acc[0] = 0.0f;
#pragma unroll
          for (int ci = 0; ci < CPL; ++ci) {
            const uint4 raw = srow[chunk_of<LPR>(ci, rl, sub)];
            float kf[8];
            unpack8<T>(raw, kf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[0] = fmaf(qf[0][ci][e], kf[e], acc[0]);
          }
        } else {
          // GQA is issue-bound (G dot products per K element): packed FFMA2
          // over even/odd element pairs, the two chains summed at the end
          float2 acc2[G];
#pragma unroll
          for (int gh = 0; gh < G; ++gh) acc2[gh] = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int ci = 0; ci < CPL; ++ci) {
            const uint4 raw = srow[chunk_of<LPR>(ci, rl, sub)];
            float kf[8];
            unpack8<T>(raw, kf);
#pragma unroll
            for (int gh = 0; gh < G; ++gh) {
#pragma unroll
              for (int e = 0; e < 8; e += 2)
                acc2[gh] = ffma2(qf[gh][ci][e], qf[gh][ci][e + 1], kf[e], kf[e + 1], acc2[gh]);
            }
          }
#pragma unroll
          for (int gh = 0; gh < G; ++gh) acc[gh] = acc2[gh].x + acc2[gh].y;
        }
#pragma unroll
        for (int o = LPR / 2; o >= 1; o >>= 1) {
#pragma unroll
          for (int gh = 0; gh < G; ++gh) acc[gh] += __shfl_xor_sync(0xffffffffu, acc[gh], o);
        }
        float mine = acc[0];
#pragma unroll
        for (int gh = 1; gh < G; ++gh) mine = (sub == gh) ? acc[gh] : mine;
        const float sc = mine * p.scale;
        if (pl < npos && sub < G) {
          if constexpr (CAND) {
            scb[pl] = sc;
          } else {
            lrow[pl] = sc;
          }
          if (sc > m_run) {
            l_run = l_run * expf(m_run - sc) + 1.0f;
            m_run = sc;
          } else {
            l_run += expf(sc - m_run);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }

    // per-split (max, sum exp) per q head: lanes with equal `sub`, then warps
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m_run, o);
      const float l2 = __shfl_xor_sync(0xffffffffu, l_run, o);
      ml_combine(m_run, l_run, m2, l2);
    }
    if (lane < G) red[warp * G + lane] = make_float2(m_run, l_run);
    named_sync(1, kCWarps * 32);
    if (threadIdx.x < G) {
      const int gh = threadIdx.x;
      float m = -INFINITY, l = 0.0f;
      for (int w = 0; w < kCWarps; ++w) ml_combine(m, l, red[w * G + gh].x, red[w * G + gh].y);
      p.partials[((size_t)b * n_q + kvh * G + gh) * p.max_splits + split] = make_float2(m, l);
    }
    if constexpr (CAND)
      emit_candidates(scb, mx, wcnt, npos, p.cand_nc, pos0, p.cand + (size_t)row * p.lstride + pos0,
                      p.cand_meta + (size_t)row * p.max_splits + split);
    named_sync(1, kCWarps * 32);  // red / scb are reused by the next item
    signal_row(p, row);
  }
}

// ---- GQA scoring on the tensor cores ---------------------------------------
// For G q heads per kv head the scoring is a [G x 128] x [128 x positions]
// product per (row, split); on CUDA cores it is issue-bound (G FMAs per K
// element). Here each consumer warp computes its 8 positions of a stage with
// mma.sync m16n8k16 (fp32 accumulation): A = the group's q (heads as rows,
// padded to 16), B = K^T straight from shared memory (8 positions as
// columns, no conversion). K is exact in the MMA's input type; q carries
// fp32 precision as a sum of parts: fp16 K -> q*2^e = hi + lo in fp16 (e puts
// the head's max |q| at 2^14, so both parts are normal and hi+lo keeps ~22
// significand bits of every element relative to the largest), bf16 K ->
// q = p1 + p2 + p3 in bf16 (24 bits). One MMA per part and k-step.
// The k dimension is permuted so a lane's operands are contiguous: lane
// (gid, tig) loads 16-B chunks tig, tig+4, tig+8, tig+12 of position gid's
// row; k-step j uses 4 dims of chunk tig+4(j/2) at offset 4(j%2): b0 = dims
// +0,+1 (k = 2tig, 2tig+1), b1 = dims +2,+3 (k = 2tig+8, +9). Two positions
// per quarter-warp share banks pairwise (2-way conflict). q is permuted the
// same way.
template <typename T>
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1);
template <>
__device__ __forceinline__ void mma_16816<__half>(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                                  uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma_16816<__nv_bfloat16>(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// NCW consumer warps: 8 = two halves alternating stages (one CTA per SM at
// 140 registers), 4 = every warp on every stage (two CTAs per SM)
template <typename T, int STAGES, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) score_mma_kernel(const ScoreParams p) {
  using QS = QSplit<T>;
  constexpr int NP = QS::NP;
  constexpr int ROWB = kH * (int)sizeof(T);
  constexpr int kMaxG = 8;
  constexpr int kHalf = 4;            // warps per stage (16 positions each)
  constexpr int kHalves = NCW / kHalf;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kRows * ROWB);
  uint64_t* empty = full + STAGES;
  float2* red = reinterpret_cast<float2*>(empty + STAGES);  // [NCW][kMaxG]

  const int n_items = p.rows * p.n_splits;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kHalf);  // each stage is consumed by one half of the warps
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NCW) {
    produce_k<T, STAGES>(p, ring, full, empty, lane, n_items);
    return;
  }

  const int G = p.G, n_q = p.n_kv * G;
  const int gid = lane >> 2, tig = lane & 3;
  const bool hv = gid < G;     // this lane's A row is a real head
  const int half = warp / kHalf;  // stages with (global index % kHalves) == half
  const int wq = warp % kHalf;    // positions 16wq .. 16wq+15 of those stages
  uint32_t g = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int row = p.row0 + item / p.n_splits;
    const int split = item - (row - p.row0) * p.n_splits;
    const int b = row / p.n_kv;
    const int kvh = row - b * p.n_kv;
    const int pos0 = split * p.chunk;
    const int npos = min(p.chunk, p.s - pos0);
    const int n_it = (npos + kRows - 1) / kRows;
    // A fragments of head gid: k-step j -> a0 = dims c*8 + 4(j&1) + {0,1},
    // a2 = + {2,3}, c = tig + 4(j>>1)
    const float* qh = p.q + ((size_t)b * n_q + kvh * G + (hv ? gid : 0)) * kH;
    float qv[32];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = tig + 4 * i;
      const float4 x0 = *reinterpret_cast<const float4*>(qh + c * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(qh + c * 8 + 4);
      qv[8 * i + 0] = x0.x; qv[8 * i + 1] = x0.y; qv[8 * i + 2] = x0.z; qv[8 * i + 3] = x0.w;
      qv[8 * i + 4] = x1.x; qv[8 * i + 5] = x1.y; qv[8 * i + 6] = x1.z; qv[8 * i + 7] = x1.w;
    }
    float amax = 0.0f;
#pragma unroll
    for (int e = 0; e < 32; ++e) amax = fmaxf(amax, fabsf(qv[e]));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
    const float pre = QS::prescale(amax);
    const float post = 1.0f / pre;  // exact: a power of two
    uint32_t af[NP][8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e0 = 8 * (j >> 1) + 4 * (j & 1) + 2 * u;
        float x = hv ? qv[e0] * pre : 0.0f, y = hv ? qv[e0 + 1] * pre : 0.0f;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const uint32_t w = QS::pack(x, y);
          af[k][j][u] = w;
          const float2 back = QS::unpack(w);
          x -= back.x;
          y -= back.y;
        }
      }
    }
    float m_run = -INFINITY, l_run = 0.0f;
    float* lrow = p.logits + ((size_t)b * n_q + kvh * G + (hv ? gid : 0)) * p.lstride + pos0;
    for (int it = 0; it < n_it; ++it, ++g) {
      if ((int)(g % kHalves) != half) continue;
      const int st = (int)(g % STAGES);
      mbar_wait(&full[st], (g / STAGES) & 1);
      const uint8_t* sb = ring + st * kRows * ROWB;
      // two n-tiles: positions 16wq + gid and 16wq + 8 + gid
      uint4 kc[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          kc[t][i] = *reinterpret_cast<const uint4*>(sb + (16 * wq + 8 * t + gid) * ROWB + 16 * (tig + 4 * i));
      float dd[2][NP][4];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int k = 0; k < NP; ++k)
#pragma unroll
          for (int e = 0; e < 4; ++e) dd[t][k][e] = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const uint4 c = kc[t][j >> 1];
          const uint32_t b0 = (j & 1) ? c.z : c.x;
          const uint32_t b1 = (j & 1) ? c.w : c.y;
#pragma unroll
          for (int k = 0; k < NP; ++k) mma_16816<T>(dd[t][k], af[k][j][0], af[k][j][1], b0, b1);
        }
      }
      // free the stage only once every lane's shared-memory loads have
      // returned: ptxas schedules the arrive right behind the first MMAs
      // (it does not depend on the loaded registers) and an arrive does not
      // wait for loads still in flight, so the producer's next TMA fill of
      // the stage could land under them (observed: an 8-position n-tile of
      // wrong logits every few C3 layers while a recall ran beside the
      // scoring). The CTA-scope fence waits for this lane's loads.
      // (An arrive whose count depends on both n-tiles' last MMA outputs
      // measured the same.)
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      // dd[t][.][0..1] = head gid at the stage's positions 16wq + 8t + 2tig, +1
      if (hv) {
        float sc[4];
        float smax = -INFINITY;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int pl = it * kRows + 16 * wq + 8 * t + 2 * tig;
          float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
          for (int k = NP - 1; k >= 0; --k) {  // small parts first
            a0 += dd[t][k][0];
            a1 += dd[t][k][1];
          }
          sc[2 * t] = pl < npos ? (a0 * post) * p.scale : -INFINITY;
          sc[2 * t + 1] = pl + 1 < npos ? (a1 * post) * p.scale : -INFINITY;
          if (pl + 1 < npos) {
            *reinterpret_cast<float2*>(lrow + pl) = make_float2(sc[2 * t], sc[2 * t + 1]);
          } else if (pl < npos) {
            lrow[pl] = sc[2 * t];
          }
          smax = fmaxf(smax, fmaxf(sc[2 * t], sc[2 * t + 1]));
        }
        // one rescale per stage; the sum-exp terms use the fast exp (the
        // split's l only normalises -- p itself is recomputed exactly)
        if (smax > -INFINITY) {
          const float mn = fmaxf(m_run, smax);
          float acc = (m_run == -INFINITY) ? 0.0f : l_run * __expf(m_run - mn);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc += (sc[e] == -INFINITY) ? 0.0f : __expf(sc[e] - mn);
          m_run = mn;
          l_run = acc;
        }
      }
    }
    // per-split (max, sum exp) per head: the 4 lanes of a head, then warps
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m_run, o);
      const float l2 = __shfl_xor_sync(0xffffffffu, l_run, o);
      ml_combine(m_run, l_run, m2, l2);
    }
    if (tig == 0 && hv) red[warp * kMaxG + gid] = make_float2(m_run, l_run);
    named_sync(1, NCW * 32);
    if (threadIdx.x < G) {
      const int gh = threadIdx.x;
      float m = -INFINITY, l = 0.0f;
      for (int w = 0; w < NCW; ++w) ml_combine(m, l, red[w * kMaxG + gh].x, red[w * kMaxG + gh].y);
      p.partials[((size_t)b * n_q + kvh * G + gh) * p.max_splits + split] = make_float2(m, l);
    }
    named_sync(1, NCW * 32);  // red is reused by the next item
    signal_row(p, row);
  }
}

// Any dtype / head_dim / group size: one warp per position, lane-strided dot.
template <typename T>
__global__ void __launch_bounds__(256) score_generic_kernel(const ScoreParams p) {
  extern __shared__ float2 wstat[];  // [8][G]
  const int split = blockIdx.x;
  const int row = p.row0 + blockIdx.y;
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int G = p.G, h = p.h, n_q = p.n_kv * G;
  const int pos0 = split * p.chunk;
  const int npos = min(p.chunk, p.s - pos0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* kslot = static_cast<const T*>(p.k) + (size_t)row * p.max_seq * h;
  for (int g = lane; g < G; g += 32) wstat[warp * G + g] = make_float2(-INFINITY, 0.0f);
  __syncwarp();
  for (int pl = warp; pl < npos; pl += 8) {
    const T* krow = kslot + (size_t)(pos0 + pl) * h;
    for (int g = 0; g < G; ++g) {
      const float* qh = p.q + ((size_t)b * n_q + kvh * G + g) * h;
      float acc = 0.0f;
      for (int c = lane; c < h; c += 32) acc = fmaf(qh[c], to_f32<T>(krow[c]), acc);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const float sc = acc * p.scale;
        p.logits[((size_t)b * n_q + kvh * G + g) * p.lstride + pos0 + pl] = sc;
        float2 ml = wstat[warp * G + g];
        ml_combine(ml.x, ml.y, sc, 1.0f);
        wstat[warp * G + g] = ml;
      }
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    float m = -INFINITY, l = 0.0f;
    for (int w = 0; w < 8; ++w) ml_combine(m, l, wstat[w * G + g].x, wstat[w * G + g].y);
    p.partials[((size_t)b * n_q + kvh * G + g) * p.max_splits + split] = make_float2(m, l);
  }
  __syncthreads();
  signal_row(p, row);
}

// ---- decode_attention_full, fused (attention.cpp:91-114) -------------------
// CTA = (row, split). The producer lane streams the split's K stages and then
// its V stages through one STAGES-deep TMA ring (both 64 positions x 256 B);
// consumers score K exactly like score_fast_kernel into shared memory, take
// the split max m and p_j = exp(s_j - m), l = sum p_j, then accumulate
// sum_j p_j V_j: thread (pg, ch) owns the 16-B column chunk ch of positions
// pg, pg+16, pg+32, pg+48 of each V stage (a half-warp reads one 256-B row:
// conflict-free). Partials are reduced across position groups in a fixed
// order; full_combine_kernel rescales the splits by exp(m_i - M).
template <typename T, int G, int LPR, int STAGES>
__global__ void __launch_bounds__((kCWarps + 1) * 32)
    full_fast_kernel(const FullParams p) {
  constexpr int CPL = 16 / LPR;
  constexpr int RPP = 32 / LPR;
  constexpr int PASSES = (kRows / kCWarps) / RPP;
  constexpr int ROWB = kH * (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kRows * ROWB);
  uint64_t* empty = full + STAGES;
  float* mls = reinterpret_cast<float*>(empty + STAGES);  // [G] m, [G] l
  float* sc = mls + 2 * G;                                // [G][chunk] scores -> p
  float* red = reinterpret_cast<float*>(ring);            // [kCWarps][G][kH], after the last stage

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x / p.n_splits;
  const int split = blockIdx.x - row * p.n_splits;
  const int b = row / p.n_kv, kvh = row - b * p.n_kv;
  const int n_q = p.n_kv * G;
  const int pos0 = split * p.chunk;
  const int npos = min(p.chunk, p.s - pos0);
  const int n_it = (npos + kRows - 1) / kRows;  // stages per tensor
  const size_t slot_off = (size_t)row * p.max_seq * kH;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kCWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kCWarps) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      const uint32_t total = 2u * (uint32_t)n_it;
      for (uint32_t g = 0; g < total; ++g) {
        const int st = (int)(g % STAGES);
        if (g >= (uint32_t)STAGES) mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
        const int it = (int)(g % (uint32_t)n_it);
        const T* base = static_cast<const T*>(g < (uint32_t)n_it ? p.k : p.v) + slot_off;
        const int pstart = pos0 + it * kRows;
        const int rows = min(kRows, npos - it * kRows);
        const uint32_t bytes = (uint32_t)(rows * ROWB);
        mbar_arrive_expect_tx(&full[st], bytes);
        tma_bulk_g2s(ring + st * kRows * ROWB, base + (size_t)pstart * kH, bytes, &full[st], pol);
      }
    }
    return;
  }

  // ---- phase 1: scores of the split's positions -> sc ----
  const int sub = lane % LPR, rl = lane / LPR;
  float qf[G][CPL][8];
#pragma unroll
  for (int gh = 0; gh < G; ++gh) {
    const float* qh = p.q + ((size_t)b * n_q + kvh * G + gh) * kH;
#pragma unroll
    for (int ci = 0; ci < CPL; ++ci) {
      const int c = chunk_of<LPR>(ci, rl, sub);
      const float4 a = *reinterpret_cast<const float4*>(qh + c * 8);
      const float4 bq = *reinterpret_cast<const float4*>(qh + c * 8 + 4);
      qf[gh][ci][0] = a.x; qf[gh][ci][1] = a.y; qf[gh][ci][2] = a.z; qf[gh][ci][3] = a.w;
      qf[gh][ci][4] = bq.x; qf[gh][ci][5] = bq.y; qf[gh][ci][6] = bq.z; qf[gh][ci][7] = bq.w;
    }
  }
  uint32_t g = 0;
  for (int it = 0; it < n_it; ++it, ++g) {
    const int st = (int)(g % STAGES);
    mbar_wait(&full[st], (g / STAGES) & 1);
    const uint8_t* sb = ring + st * kRows * ROWB;
#pragma unroll
    for (int pass = 0; pass < PASSES; ++pass) {
      const int r = warp * (kRows / kCWarps) + pass * RPP + rl;
      const int pl = it * kRows + r;
      const uint4* srow = reinterpret_cast<const uint4*>(sb + r * ROWB);
      float acc[G];
#pragma unroll
      for (int gh = 0; gh < G; ++gh) acc[gh] = 0.0f;
#pragma unroll
      for (int ci = 0; ci < CPL; ++ci) {
        const uint4 raw = srow[chunk_of<LPR>(ci, rl, sub)];
        float kf[8];
        unpack8<T>(raw, kf);
#pragma unroll
        for (int gh = 0; gh < G; ++gh) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[gh] = fmaf(qf[gh][ci][e], kf[e], acc[gh]);
        }
      }
#pragma unroll
      for (int o = LPR / 2; o >= 1; o >>= 1) {
#pragma unroll
        for (int gh = 0; gh < G; ++gh) acc[gh] += __shfl_xor_sync(0xffffffffu, acc[gh], o);
      }
      float mine = acc[0];
#pragma unroll
      for (int gh = 1; gh < G; ++gh) mine = (sub == gh) ? acc[gh] : mine;
      if (pl < npos && sub < G) sc[sub * p.chunk + pl] = mine * p.scale;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  named_sync(1, kCWarps * 32);
  // ---- split softmax: m, p_j = exp(s_j - m), l = sum p_j (warp per head) ----
  for (int gh = warp; gh < G; gh += kCWarps) {
    float* sg = sc + gh * p.chunk;
    float m = -INFINITY;
    for (int j = lane; j < npos; j += 32) m = fmaxf(m, sg[j]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.0f;
    for (int j = lane; j < npos; j += 32) {
      const float e = expf(sg[j] - m);
      sg[j] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      mls[gh] = m;
      mls[G + gh] = l;
    }
  }
  named_sync(1, kCWarps * 32);
  // ---- phase 2: sum_j p_j V_j ----
  const int ct = threadIdx.x;
  const int ch = ct & 15, pg = ct >> 4;
  float acc[G][8];
#pragma unroll
  for (int gh = 0; gh < G; ++gh)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[gh][e] = 0.0f;
  for (int it = 0; it < n_it; ++it, ++g) {
    const int st = (int)(g % STAGES);
    mbar_wait(&full[st], (g / STAGES) & 1);
    const uint8_t* sb = ring + st * kRows * ROWB;
#pragma unroll
    for (int k4 = 0; k4 < kRows / 16; ++k4) {
      const int j = pg + 16 * k4;
      const int pl = it * kRows + j;
      if (pl < npos) {
        float vf[8];
        unpack8<T>(reinterpret_cast<const uint4*>(sb + j * ROWB)[ch], vf);
#pragma unroll
        for (int gh = 0; gh < G; ++gh) {
          const float w = sc[gh * p.chunk + pl];
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[gh][e] = fmaf(w, vf[e], acc[gh][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  // position groups pg and pg^1 share a warp (lanes ch, ch + 16)
#pragma unroll
  for (int gh = 0; gh < G; ++gh)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[gh][e] += __shfl_xor_sync(0xffffffffu, acc[gh][e], 16);
  // the ring is free once every stage is consumed and every TMA has landed
  named_sync(1, kCWarps * 32);
  if (lane < 16) {
#pragma unroll
    for (int gh = 0; gh < G; ++gh)
#pragma unroll
      for (int e = 0; e < 8; ++e) red[(warp * G + gh) * kH + ch * 8 + e] = acc[gh][e];
  }
  named_sync(1, kCWarps * 32);
  for (int o = ct; o < G * kH; o += kCWarps * 32) {
    const int gh = o / kH, c = o - gh * kH;
    float a = 0.0f;
#pragma unroll
    for (int w = 0; w < kCWarps; ++w) a += red[(w * G + gh) * kH + c];
    const size_t slot = (size_t)b * n_q + kvh * G + gh;
    p.part_out[(slot * p.max_splits + split) * kH + c] = a;
    if (c == 0) p.part_ml[slot * p.max_splits + split] = make_float2(mls[gh], mls[G + gh]);
  }
}

// out = sum_i exp(m_i - M) acc_i / sum_i exp(m_i - M) l_i, splits in order
__global__ void full_combine_kernel(const FullParams p) {
  const int slot = blockIdx.x;
  const int c = threadIdx.x;  // kH threads
  const float2* ml = p.part_ml + (size_t)slot * p.max_splits;
  float M = -INFINITY;
  for (int i = 0; i < p.n_splits; ++i) M = fmaxf(M, ml[i].x);
  float num = 0.0f, den = 0.0f;
  for (int i = 0; i < p.n_splits; ++i) {
    const float f = expf(ml[i].x - M);
    num = fmaf(f, p.part_out[((size_t)slot * p.max_splits + i) * kH + c], num);
    den = fmaf(f, ml[i].y, den);
  }
  p.out[(size_t)slot * kH + c] = num / den;
}

template <typename T, int G, int LPR>
void launch_full(const FullParams& p, cudaStream_t st) {
  constexpr int STAGES = 4;
  constexpr int ROWB = kH * (int)sizeof(T);
  const size_t smem = STAGES * kRows * ROWB + 2 * STAGES * sizeof(uint64_t) +
                      (2 * G + (size_t)G * p.chunk) * sizeof(float);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(full_fast_kernel<T, G, LPR, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    configured |= 1ull << (dev & 63);
  }
  full_fast_kernel<T, G, LPR, STAGES><<<p.rows * p.n_splits, (kCWarps + 1) * 32, smem, st>>>(p);
  full_combine_kernel<<<(p.rows / p.n_kv) * p.n_kv * G, kH, 0, st>>>(p);
}

template <typename T>
bool try_full(const FullParams& p, cudaStream_t st) {
  // red ([8][G][128] floats) aliases the ring; sc must fit beside it
  if ((p.chunk % kRows) != 0 || (size_t)p.G * p.chunk * 4 > 96 * 1024) return false;
  switch (p.G) {
    case 1: launch_full<T, 1, 4>(p, st); return true;
    case 2: launch_full<T, 2, 4>(p, st); return true;
    case 4: launch_full<T, 4, 8>(p, st); return true;
    case 8: launch_full<T, 8, 16>(p, st); return true;
    default: return false;
  }
}

int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 63]) cudaDeviceGetAttribute(&n[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  return n[dev & 63] > 0 ? n[dev & 63] : 148;
}

template <typename T, int G, int LPR, int STAGES, bool CAND>
void launch_fast_s(const ScoreParams& p, cudaStream_t st) {
  constexpr int ROWB = kH * (int)sizeof(T);
  const size_t smem = STAGES * kRows * ROWB + 2 * STAGES * sizeof(uint64_t) +
                      kCWarps * G * sizeof(float2) +
                      (CAND ? (size_t)kMaxCandChunk * 4 + 3 * kCWarps * 4 : 0);
  static int configured[64] = {0};  // dynamic smem opted in, per device (grows with the split length)
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured[dev & 63] < (int)smem) {
    cudaFuncSetAttribute(score_fast_kernel<T, G, LPR, STAGES, CAND>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[dev & 63] = (int)smem;
  }
  const int n_items = p.rows * p.n_splits;
  score_fast_kernel<T, G, LPR, STAGES, CAND><<<n_items, (kCWarps + 1) * 32, smem, st>>>(p);
}

template <typename T, int G, int LPR, bool CAND>
void launch_fast(const ScoreParams& p, cudaStream_t st) {
  switch (p.stages) {
    case 2: launch_fast_s<T, G, LPR, 2, CAND>(p, st); break;
    case 3: launch_fast_s<T, G, LPR, 3, CAND>(p, st); break;
    case 6: launch_fast_s<T, G, LPR, 6, CAND>(p, st); break;
    case 8: launch_fast_s<T, G, LPR, 8, CAND>(p, st); break;
    default: launch_fast_s<T, G, LPR, 4, CAND>(p, st); break;
  }
}

template <typename T, int STAGES, int NCW>
void launch_mma_s(const ScoreParams& p, cudaStream_t st) {
  constexpr int ROWB = kH * (int)sizeof(T);
  const size_t smem = STAGES * kRows * ROWB + 2 * STAGES * sizeof(uint64_t) + NCW * 8 * sizeof(float2);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(score_mma_kernel<T, STAGES, NCW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured |= 1ull << (dev & 63);
  }
  const int n_items = p.rows * p.n_splits;
  score_mma_kernel<T, STAGES, NCW><<<n_items, (NCW + 1) * 32, smem, st>>>(p);
}

template <typename T>
bool try_fast(const ScoreParams& p, cudaStream_t st) {
  if (p.h != kH || (p.chunk % kRows) != 0) return false;
  if (p.G >= 2 && p.G <= 8 && p.cand_nc == 0 && p.use_mma) {
    if (p.use_mma == 2) {  // 8 consumer warps, one CTA per SM
      switch (p.stages) {
        case 8: launch_mma_s<T, 8, 8>(p, st); break;
        default: launch_mma_s<T, 4, 8>(p, st); break;
      }
    } else {  // 4 consumer warps, two CTAs per SM
      switch (p.stages) {
        case 8: launch_mma_s<T, 8, 4>(p, st); break;
        default: launch_mma_s<T, 4, 4>(p, st); break;
      }
    }
    return true;
  }
  if (p.cand_nc > 0) {
    if (p.G != 1 || p.chunk > kMaxCandChunk || p.cand_nc > kCWarps * 16) return false;
    launch_fast<T, 1, 4, true>(p, st);
    return true;
  }
  switch (p.G) {
    case 1: launch_fast<T, 1, 4, false>(p, st); return true;
    case 2: launch_fast<T, 2, 4, false>(p, st); return true;
    case 4: launch_fast<T, 4, 8, false>(p, st); return true;
    case 8: launch_fast<T, 8, 16, false>(p, st); return true;
    default: return false;
  }
}

}  // namespace

int score_pick_chunk(int s, int rows, int override_chunk, int G) {
  if (override_chunk > 0) return ((override_chunk + kRows - 1) / kRows) * kRows;
  const long long work = (long long)s * rows;
  long long c, hi;
  if (G >= 2) {
    // GQA (score_mma_kernel, 3 CTAs / SM): ~28 items per SM, 1024..8192
    // positions (r02, C3: 1024 vs 2048 positions 233 vs 238 us per layer
    // pipelined, 332 vs 346 in the engine step; 64 k x 64 rows and
    // 8 k x 512 rows also best at 1024)
    hi = 8192;
    c = (work + 148LL * 28 - 1) / (148LL * 28);
    c = std::max<long long>(1024, std::min<long long>(hi, c));
  } else {
    // MHA: ~48 items per SM (3 CTAs / SM; small items balance best against
    // the concurrent recall), 1024..2048 positions each (shorter items pay
    // their ramp-up: 4k context 70 -> 54 us per layer at 1024)
    hi = 2048;
    c = (work + 148LL * 48 - 1) / (148LL * 48);
    c = std::max<long long>(1024, std::min<long long>(hi, c));
  }
  // equal splits: floor(s / c) of them (at most `hi` positions each), so a
  // row a few positions past a multiple of c -- the decode phase after a
  // 16 k prefill -- does not get an extra split (an extra item per row) of a
  // handful of positions (tests/test_capi_cpu.py)
  long long n = std::max<long long>(1, s / c);
  if ((s + n - 1) / n > hi) n = (s + hi - 1) / hi;
  c = (s + n - 1) / n;
  c = ((c + kRows - 1) / kRows) * kRows;
  return (int)c;
}

int sm_count() { return num_sms(); }

bool full_fast_launch(const FullParams& p, int dtype, cudaStream_t st) {
  if (dtype == KC_F16) return try_full<__half>(p, st);
  if (dtype == KC_BF16) return try_full<__nv_bfloat16>(p, st);
  return false;
}


bool score_cand_supported(int dtype, int h, int G, int chunk, int nc) {
  // nc <= 128: the bound is the nc-th largest of the 256 consumer threads'
  // block maxima; with nc close to 256 it keeps nearly every position
  return (dtype == KC_F16 || dtype == KC_BF16) && h == kH && G == 1 && chunk % kRows == 0 &&
         chunk <= kMaxCandChunk && nc >= 1 && nc <= kCWarps * 16;
}

void score_launch(const ScoreParams& p, int dtype, cudaStream_t st) {
  // GQA on tcgen05 (kc_score_tc.cu) when the caller passed the layer's map
  if (p.use_mma == 3 && p.cand_nc == 0 && score_tc_launch(p, dtype, st)) return;
  if (dtype == KC_F16 && try_fast<__half>(p, st)) return;
  if (dtype == KC_BF16 && try_fast<__nv_bfloat16>(p, st)) return;
  if (p.cand_nc > 0) {  // the caller checked score_cand_supported: never silently dense
    fprintf(stderr, "kcache: candidate-mode scoring requested for an unsupported shape\n");
    abort();
  }
  dim3 grid(p.n_splits, p.rows);
  const size_t smem = 8 * (size_t)p.G * sizeof(float2);
  switch (dtype) {
    case KC_F16: score_generic_kernel<__half><<<grid, 256, smem, st>>>(p); break;
    case KC_BF16: score_generic_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(p); break;
    default: score_generic_kernel<float><<<grid, 256, smem, st>>>(p); break;
  }
}

}  // namespace kc

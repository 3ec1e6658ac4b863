// kc_recall.cu -- V recall + P.V, the full-attention comparator's P.V, and
// the store's append/convert kernels (sm_100a).
//
// recall_pv_kernel replaces gather_v (proj/core/src/kv_cache.cpp:150-187) and
// the P.V loop + add_scaled (proj/core/src/attention.cpp:159-188, :23-27).
// One CTA per (batch, kv head): the N selected V rows (256 B each at h=128,
// fp16) are pulled from the layer's V storage -- pinned, device-mapped host
// memory for offloaded layers (zero-copy PCIe reads, 16 B per lane, a whole
// chunk of rows in flight per CTA) or HBM for resident layers -- into shared
// memory, then every (q head, column) thread accumulates sum_r w_r * v_r[c]
// in ascending position order with separately rounded multiply and add
// (__fmul_rn/__fadd_rn), i.e. the same operation sequence as the reference's
// `acc[c] += w * v[c]` compiled with -ffp-contract=off. `reverse` is the
// reference's ordered_accumulation=false fault hook.
#include <algorithm>

#include "kc_device.cuh"
#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace kc {

namespace {

constexpr int kRecallThreads = 256;
constexpr int kRecallSmem = 40 * 1024;
constexpr int kH = 128;
constexpr int kMaxGroup = 8;

template <typename T>
__global__ void __launch_bounds__(kRecallThreads) recall_pv_kernel(const RecallParams p, int rc_max) {
  extern __shared__ __align__(16) uint8_t smem[];
  // grid <= rows: each CTA walks rows blockIdx.x, +gridDim.x, ... so a small
  // grid leaves SM room for the concurrently running scoring kernel
  for (int row = p.row_offset + blockIdx.x; row < p.row_offset + p.rows; row += gridDim.x) {
  const int b = row / p.n_kv;
  const int kvh = row - b * p.n_kv;
  const int G = p.G, h = p.h, n_q = p.n_kv * G, nc = p.nc;
  const int tid = threadIdx.x;
  const size_t rowb = (size_t)h * sizeof(T);
  T* vbuf = reinterpret_cast<T*>(smem);
  float* wbuf = reinterpret_cast<float*>(smem + (((size_t)rc_max * rowb + 15) & ~size_t(15)));
  // staged: rows already compacted to [rows][nc][h] (host gather + DMA)
  const T* vslot = static_cast<const T*>(p.v) + (size_t)row * (p.staged ? (size_t)nc : (size_t)p.max_seq) * h;
  const uint32_t* idx = p.idx + (size_t)row * nc;
  const int n_out = G * h;
  constexpr int kMaxOut = 4;  // G*h <= 1024
  float acc[kMaxOut];
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) acc[i] = 0.0f;

  const int n_chunks = (nc + rc_max - 1) / rc_max;
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int chunk = p.reverse ? (n_chunks - 1 - ci) : ci;
    const int c0 = chunk * rc_max;
    const int rc = min(rc_max, nc - c0);
    // ---- recall: selected rows -> shared memory ----
    if ((rowb & 15) == 0) {
      const int vpr = (int)(rowb >> 4);
      const int total = rc * vpr;
      uint4* dst = reinterpret_cast<uint4*>(vbuf);
      const uint64_t pol = l2_evict_first_policy();
      constexpr int kBatch = 8;
      for (int v0 = tid; v0 < total; v0 += kRecallThreads * kBatch) {
        uint4 tmp[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int v = v0 + u * kRecallThreads;
          if (v < total) {
            const int r = v / vpr, part = v - r * vpr;
            const size_t pos = p.staged ? (size_t)(c0 + r) : (size_t)idx[c0 + r];
            tmp[u] = ld_stream16(reinterpret_cast<const uint4*>(vslot + pos * h) + part, pol);
          }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int v = v0 + u * kRecallThreads;
          if (v < total) dst[v] = tmp[u];
        }
      }
    } else {
      for (int e = tid; e < rc * h; e += kRecallThreads) {
        const int r = e / h, c = e - r * h;
        const size_t pos = p.staged ? (size_t)(c0 + r) : (size_t)idx[c0 + r];
        vbuf[e] = vslot[pos * h + c];
      }
    }
    // ---- weights (raw p, or p * (1/sum p) when renormalising) ----
    for (int e = tid; e < G * rc; e += kRecallThreads) {
      const int g = e / rc, r = e - g * rc;
      const size_t slot = (size_t)b * n_q + kvh * G + g;
      float w = p.w[slot * nc + c0 + r];
      if (p.renormalize) w = __fmul_rn(w, p.norm[slot]);
      wbuf[g * rc_max + r] = w;
    }
    __syncthreads();
    // ---- P.V, fixed position order per output element ----
#pragma unroll
    for (int i = 0; i < kMaxOut; ++i) {
      const int o = tid + i * kRecallThreads;
      if (o < n_out) {
        const int g = o / h, c = o - g * h;
        const float* wg = wbuf + g * rc_max;
        float a = acc[i];
        if (!p.reverse) {
          for (int r = 0; r < rc; ++r) a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vbuf[r * h + c])));
        } else {
          for (int r = rc - 1; r >= 0; --r)
            a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vbuf[r * h + c])));
        }
        acc[i] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) {
    const int o = tid + i * kRecallThreads;
    if (o < n_out) {
      const int g = o / h, c = o - g * h;
      p.out[((size_t)b * n_q + kvh * G + g) * h + c] = acc[i];
    }
  }
  }  // row loop
}

// Software-pipelined variant for the common shape (h = 128 16-bit rows,
// nc <= 128): while the CTA reduces row r from one shared-memory buffer, the
// 16-B zero-copy loads of its next row are already in flight into registers,
// so a small grid keeps the PCIe read queue full without leaving the SMs to
// wait on host latency between rows. Same operation order as
// recall_pv_kernel.
constexpr int kPipeMaxNc = 128;

template <typename T>
__device__ __forceinline__ void recall_pipe_body(const RecallParams& p) {
  constexpr int kVpr = 16;  // 16-B chunks per 256-B row
  constexpr int kLoads = kPipeMaxNc * kVpr / kRecallThreads;  // 8
  extern __shared__ __align__(16) uint8_t smem[];
  uint4* vb = reinterpret_cast<uint4*>(smem);                       // [2][nc][16]
  float* wb = reinterpret_cast<float*>(smem + 2 * kPipeMaxNc * 256);  // [2][G][nc]
  const int G = p.G, n_q = p.n_kv * G, nc = p.nc;
  const int tid = threadIdx.x;
  const int total = nc * kVpr;
  const int end = p.row_offset + p.rows;
  uint4 tmp[kLoads];
  auto vslot_of = [&](int row) {
    return reinterpret_cast<const uint4*>(static_cast<const T*>(p.v) +
                                          (size_t)row * (p.staged ? (size_t)nc : (size_t)p.max_seq) * kH);
  };
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int row) {
    const uint4* vs = vslot_of(row);
    const uint32_t* idx = p.idx + (size_t)row * nc;
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int v = tid + u * kRecallThreads;
      if (v < total) {
        const int r = v >> 4, part = v & 15;
        const size_t pos = p.staged ? (size_t)r : (size_t)idx[r];
        tmp[u] = p.dbg ? make_uint4((uint32_t)pos, 0u, 0u, 0u) : ld_stream16(vs + pos * kVpr + part, pol);
      }
    }
  };
  int row = p.row_offset + blockIdx.x;
  if (p.dbg == 2) return;
  if (row < end) issue(row);
  int buf = 0;
  while (row < end) {
    const int b = row / p.n_kv;
    const int kvh = row - b * p.n_kv;
    // land: the rows this thread loaded -> shared memory; the weights of the
    // row's q heads
    {
      uint4* dst = vb + buf * kPipeMaxNc * kVpr;
#pragma unroll
      for (int u = 0; u < kLoads; ++u) {
        const int v = tid + u * kRecallThreads;
        if (v < total) dst[v] = tmp[u];
      }
      float* wd = wb + buf * kMaxGroup * kPipeMaxNc;
      for (int e = tid; e < G * nc; e += kRecallThreads) {
        const int g = e / nc, r = e - g * nc;
        const size_t slot = (size_t)b * n_q + kvh * G + g;
        float w = p.w[slot * nc + r];
        if (p.renormalize) w = __fmul_rn(w, p.norm[slot]);
        wd[g * kPipeMaxNc + r] = w;
      }
    }
    __syncthreads();
    const int next = row + gridDim.x;
    if (next < end) issue(next);  // in flight during the reduction below
    const T* vt = reinterpret_cast<const T*>(vb + buf * kPipeMaxNc * kVpr);
    const float* wd = wb + buf * kMaxGroup * kPipeMaxNc;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // G*h <= 1024 outputs
      const int o = tid + i * kRecallThreads;
      if (o < G * kH) {
        const int g = o / kH, c = o - g * kH;
        const float* wg = wd + g * kPipeMaxNc;
        float a = 0.0f;
        if (!p.reverse) {
          for (int r = 0; r < nc; ++r) a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vt[r * kH + c])));
        } else {
          for (int r = nc - 1; r >= 0; --r) a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vt[r * kH + c])));
        }
        p.out[((size_t)b * n_q + kvh * G + g) * kH + c] = a;
      }
    }
    row = next;
    buf ^= 1;
  }
}

template <typename T>
__global__ void __launch_bounds__(kRecallThreads) recall_pv_pipe_kernel(const RecallParams p) {
  recall_pipe_body<T>(p);
}

// the same at <= 72 registers: 256 x 72 fits beside two GQA scoring CTAs
template <typename T>
__global__ void __maxnreg__(72) recall_pv_pipe_lean_kernel(const RecallParams p) {
  recall_pipe_body<T>(p);
}

// The same operation with the V rows moved by the TMA unit: warp 0 issues one
// 256-B cp.async.bulk per selected row (global or host-resident arena ->
// shared memory, completion as transaction bytes on the buffer's mbarrier)
// for the CTA's next row while all threads reduce the current one. No
// registers or LSU slots hold the in-flight PCIe reads. Same operation order
// as recall_pv_kernel. h = 128 16-bit rows, nc <= 128, G <= 8.
template <typename T>
__global__ void __launch_bounds__(kRecallThreads) recall_tma_kernel(const RecallParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  T* vb = reinterpret_cast<T*>(smem);                                 // [2][kPipeMaxNc][kH]
  float* wb = reinterpret_cast<float*>(smem + 2 * kPipeMaxNc * 256);  // [2][kMaxGroup][kPipeMaxNc]
  __shared__ __align__(8) uint64_t full[2];
  const int G = p.G, n_q = p.n_kv * G, nc = p.nc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int end = p.row_offset + p.rows;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int row, int buf) {  // warp 0
    const T* vs = static_cast<const T*>(p.v) + (size_t)row * (p.staged ? (size_t)nc : (size_t)p.max_seq) * kH;
    const uint32_t* idx = p.idx + (size_t)row * nc;
    if (lane == 0) mbar_arrive_expect_tx(&full[buf], (uint32_t)nc * (uint32_t)(kH * sizeof(T)));
    __syncwarp();
    T* dst = vb + (size_t)buf * kPipeMaxNc * kH;
    for (int r = lane; r < nc; r += 32) {
      const size_t pos = p.staged ? (size_t)r : (size_t)__ldcg(idx + r);
      tma_bulk_g2s(dst + r * kH, vs + pos * kH, (uint32_t)(kH * sizeof(T)), &full[buf], pol);
    }
  };
  int row = p.row_offset + blockIdx.x;
  if (row < end && warp == 0) issue(row, 0);
  for (int it = 0; row < end; ++it) {
    const int buf = it & 1;
    const int b = row / p.n_kv;
    const int kvh = row - b * p.n_kv;
    float* wd = wb + buf * kMaxGroup * kPipeMaxNc;
    for (int e = tid; e < G * nc; e += kRecallThreads) {
      const int g = e / nc, r = e - g * nc;
      const size_t slot = (size_t)b * n_q + kvh * G + g;
      float w = p.w[slot * nc + r];
      if (p.renormalize) w = __fmul_rn(w, p.norm[slot]);
      wd[g * kPipeMaxNc + r] = w;
    }
    mbar_wait(&full[buf], (uint32_t)(it >> 1) & 1u);
    // weights visible; every thread is past the previous row's reduction, so
    // the other buffer is free for the next row's copies
    __syncthreads();
    const int next = row + gridDim.x;
    if (next < end && warp == 0) issue(next, buf ^ 1);
    const T* vt = vb + (size_t)buf * kPipeMaxNc * kH;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // G*h <= 1024 outputs
      const int o = tid + i * kRecallThreads;
      if (o < G * kH) {
        const int g = o / kH, c = o - g * kH;
        const float* wg = wd + g * kPipeMaxNc;
        float a = 0.0f;
        if (!p.reverse) {
          for (int r = 0; r < nc; ++r) a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vt[r * kH + c])));
        } else {
          for (int r = nc - 1; r >= 0; --r) a = __fadd_rn(a, __fmul_rn(wg[r], to_f32<T>(vt[r * kH + c])));
        }
        p.out[((size_t)b * n_q + kvh * G + g) * kH + c] = a;
      }
    }
    row = next;
  }
}

// decode_attention_full P.V: CTA (split, row) accumulates its positions in
// order with the global softmax weights; pv_reduce sums splits in order.
template <typename T>
__global__ void __launch_bounds__(256) pv_full_kernel(const PvFullParams p) {
  extern __shared__ float sh[];  // M[G], Z[G], w[G][chunk]
  const int split = blockIdx.x, row = blockIdx.y;
  const int b = row / p.n_kv, kvh = row - b * p.n_kv;
  const int G = p.G, h = p.h, n_q = p.n_kv * G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* sM = sh;
  float* sZ = sh + G;
  float* wb = sh + 2 * G;
  for (int g = warp; g < G; g += 8) {
    float m, z;
    softmax_stats(p.partials + ((size_t)b * n_q + kvh * G + g) * p.max_splits, p.n_splits, lane, m, z);
    if (lane == 0) {
      sM[g] = m;
      sZ[g] = z;
    }
  }
  __syncthreads();
  const int pos0 = split * p.chunk;
  const int npos = min(p.chunk, p.s - pos0);
  constexpr int kTile = 256;
  const T* vslot = static_cast<const T*>(p.v) + ((size_t)row * p.max_seq + pos0) * h;
  constexpr int kMaxOut = 4;  // G*h <= 1024
  float acc[kMaxOut];
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) acc[i] = 0.0f;
  for (int t0 = 0; t0 < npos; t0 += kTile) {
    const int nt = min(kTile, npos - t0);
    for (int e = tid; e < G * nt; e += 256) {
      const int g = e / nt, j = e - g * nt;
      const float* lrow = p.logits + ((size_t)b * n_q + kvh * G + g) * p.lstride;
      wb[g * kTile + j] = expf(lrow[pos0 + t0 + j] - sM[g]) / sZ[g];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kMaxOut; ++i) {
      const int o = tid + i * 256;
      if (o < G * h) {
        const int g = o / h, c = o - g * h;
        float a = acc[i];
        for (int j = 0; j < nt; ++j)
          a = __fadd_rn(a, __fmul_rn(wb[g * kTile + j], to_f32<T>(vslot[(size_t)(t0 + j) * h + c])));
        acc[i] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i) {
    const int o = tid + i * 256;
    if (o < G * h) {
      const int g = o / h, c = o - g * h;
      p.part_out[(((size_t)b * n_q + kvh * G + g) * p.n_splits + split) * h + c] = acc[i];
    }
  }
}

__global__ void pv_reduce_kernel(const float* part, float* out, int slots, int n_splits, int h) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)slots * h) return;
  const int64_t slot = e / h, c = e - slot * h;
  float a = 0.0f;
  for (int i = 0; i < n_splits; ++i) a += part[(slot * n_splits + i) * h + c];
  out[slot * h + c] = a;
}

// ---- append: position-major rows -> [b][kv][pos][h] storage ----
template <typename Ti, typename To>
__global__ void append_kernel(const AppendParams p) {
  const int64_t width = (int64_t)p.n_kv * p.h;
  const int64_t n = p.n_rows * width;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / width, col = e - r * width;
    const int64_t pos = p.pos0 + r / p.batch, bi = r % p.batch;
    const int64_t kvh = col / p.h, c = col - kvh * p.h;
    const float x = to_f32<Ti>(static_cast<const Ti*>(p.src)[e]);
    static_cast<To*>(p.dst)[((bi * p.n_kv + kvh) * p.max_seq + pos) * p.h + c] = from_f32<To>(x);
  }
}

// 8 consecutive elements of one head per thread (h % 8 == 0): 16-B stores.
template <typename Ti, typename To>
__global__ void append_vec8_kernel(const AppendParams p) {
  const int64_t width = (int64_t)p.n_kv * p.h;
  const int64_t n8 = p.n_rows * width / 8;
  for (int64_t e8 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e8 < n8;
       e8 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e8 * 8;
    const int64_t r = e / width, col = e - r * width;
    const int64_t pos = p.pos0 + r / p.batch, bi = r % p.batch;
    const int64_t kvh = col / p.h, c = col - kvh * p.h;
    const Ti* s = static_cast<const Ti*>(p.src) + e;
    To o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = from_f32<To>(to_f32<Ti>(s[i]));
    To* d = static_cast<To*>(p.dst) + ((bi * p.n_kv + kvh) * p.max_seq + pos) * p.h + c;
    if constexpr (sizeof(To) == 2) {
      *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(o);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = o[i];
    }
  }
}

template <typename Ti, typename To>
void append_typed(const AppendParams& p, cudaStream_t st) {
  const int64_t n = p.n_rows * (int64_t)p.n_kv * p.h;
  if (p.h % 8 == 0) {
    const int64_t n8 = n / 8;
    const int blocks = (int)std::min<int64_t>((n8 + 255) / 256, 148 * 16);
    append_vec8_kernel<Ti, To><<<std::max(blocks, 1), 256, 0, st>>>(p);
  } else {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    append_kernel<Ti, To><<<std::max(blocks, 1), 256, 0, st>>>(p);
  }
}

template <typename Ti>
void append_dst(const AppendParams& p, int dst_dtype, cudaStream_t st) {
  switch (dst_dtype) {
    case KC_F16: append_typed<Ti, __half>(p, st); break;
    case KC_BF16: append_typed<Ti, __nv_bfloat16>(p, st); break;
    default: append_typed<Ti, float>(p, st); break;
  }
}

// SplitMix64 (rng.hpp:13-19) counter-indexed; next_uniform (rng.hpp:22-26)
// with separately rounded multiply/add like the -ffp-contract=off host code.
template <typename T>
__global__ void fill_uniform_kernel(T* dst, uint64_t n, uint64_t seed, uint64_t offset, float lo,
                                    float hi) {
  const float span = __fsub_rn(hi, lo);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (offset + i + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const double u = __dmul_rn((double)(z >> 11), 0x1.0p-53);
    const float f = __double2float_rn(u);
    dst[i] = from_f32<T>(__fadd_rn(lo, __fmul_rn(f, span)));
  }
}


// gather_v slow path / k_row / v_row: listed (slot row, position) pairs -> fp32.
template <typename T>
__global__ void gather_rows_kernel(const T* base, const uint32_t* slot_row, const uint32_t* pos,
                                   int64_t n, int h, int64_t max_seq, float* out) {
  const int64_t total = n * h;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / h, c = e - i * h;
    out[e] = to_f32<T>(base[((int64_t)slot_row[i] * max_seq + pos[i]) * h + c]);
  }
}

int grid_for(int64_t n);

template <typename T>
__global__ void to_f32_kernel(const T* src, float* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = to_f32<T>(src[i]);
}

__global__ void expand_idx_kernel(const uint32_t* src, uint32_t* dst, int rows, int G, int nc) {
  const int64_t n = (int64_t)rows * G * nc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = e / nc, r = e - slot * nc;
    dst[e] = src[(slot / G) * nc + r];
  }
}

int grid_for(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
}

// One CTA: the histogram of this call's selected positions (each kv-row
// index set counts once per q head of its group, like the reference's per-slot
// loop) and the dropped mass added in slot order after the running sum of
// the previous layers -- the reference's accumulation order, so the double
// sum is reproducible.
__global__ void step_stats_kernel(const uint32_t* idx, const double* dropped, int rows, int G, int nc,
                                  uint64_t len, int slots, StepStatsDev* acc) {
  __shared__ unsigned int hist[8];
  if (threadIdx.x < 8) hist[threadIdx.x] = 0u;
  __syncthreads();
  // per-thread counts, then one shared atomic per warp and bin
  unsigned int mine[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t n = (int64_t)rows * nc;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const uint64_t q8 = (uint64_t)idx[e] * 8ull / len;
    const unsigned b = q8 < 7ull ? (unsigned)q8 : 7u;
#pragma unroll
    for (int k = 0; k < 8; ++k) mine[k] += (b == (unsigned)k) ? 1u : 0u;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    unsigned v = mine[k];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&hist[k], v);
  }
  __syncthreads();
  if (threadIdx.x < 8) acc->hist[threadIdx.x] += (unsigned long long)hist[threadIdx.x] * (unsigned long long)G;
  if (threadIdx.x == 0) {
    double s = acc->dropped_sum;
    for (int i = 0; i < slots; ++i) s += dropped[i];
    acc->dropped_sum = s;
  }
}

}  // namespace

void step_stats_launch(const uint32_t* idx, const double* dropped, int rows, int G, int nc, uint64_t len,
                       int slots, StepStatsDev* acc, cudaStream_t st) {
  step_stats_kernel<<<1, 1024, 0, st>>>(idx, dropped, rows, G, nc, len, slots, acc);
}

template <typename T>
void launch_pipe(const RecallParams& p, cudaStream_t st) {
  const size_t smem = 2 * kPipeMaxNc * 256 + 2 * kMaxGroup * kPipeMaxNc * sizeof(float);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(recall_pv_pipe_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured |= 1ull << (dev & 63);
  }
  static unsigned long long configured_lean = 0;
  if (p.lean && !(configured_lean >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(recall_pv_pipe_lean_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured_lean |= 1ull << (dev & 63);
  }
  const int grid = (p.grid > 0 && p.grid < p.rows) ? p.grid : p.rows;
  if (p.lean) recall_pv_pipe_lean_kernel<T><<<grid, kRecallThreads, smem, st>>>(p);
  else recall_pv_pipe_kernel<T><<<grid, kRecallThreads, smem, st>>>(p);
}

template <typename T>
void launch_tma(const RecallParams& p, cudaStream_t st) {
  const size_t smem = 2 * kPipeMaxNc * 256 + 2 * kMaxGroup * kPipeMaxNc * sizeof(float);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(recall_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured |= 1ull << (dev & 63);
  }
  const int grid = (p.grid > 0 && p.grid < p.rows) ? p.grid : p.rows;
  recall_tma_kernel<T><<<grid, kRecallThreads, smem, st>>>(p);
}

void recall_launch(const RecallParams& p, int dtype, cudaStream_t st) {
  if (p.tma && p.h == kH && p.nc <= kPipeMaxNc && p.G <= kMaxGroup && dtype != KC_F32) {
    if (dtype == KC_F16) launch_tma<__half>(p, st);
    else launch_tma<__nv_bfloat16>(p, st);
    return;
  }
  if (p.pipelined && p.h == kH && p.nc <= kPipeMaxNc && p.G <= kMaxGroup && dtype != KC_F32) {
    if (dtype == KC_F16) launch_pipe<__half>(p, st);
    else launch_pipe<__nv_bfloat16>(p, st);
    return;
  }
  const size_t esz = dtype == KC_F32 ? 4 : 2;
  const size_t rowb = (size_t)p.h * esz;
  int rc_max = (int)(kRecallSmem / (rowb + 4 * (size_t)p.G));
  rc_max = std::max(1, std::min(rc_max, p.nc));
  const size_t smem = ((rc_max * rowb + 15) & ~size_t(15)) + 4 * (size_t)p.G * rc_max;
  const int grid = (p.grid > 0 && p.grid < p.rows) ? p.grid : p.rows;
  switch (dtype) {
    case KC_F16: recall_pv_kernel<__half><<<grid, kRecallThreads, smem, st>>>(p, rc_max); break;
    case KC_BF16: recall_pv_kernel<__nv_bfloat16><<<grid, kRecallThreads, smem, st>>>(p, rc_max); break;
    default: recall_pv_kernel<float><<<grid, kRecallThreads, smem, st>>>(p, rc_max); break;
  }
}

void pv_full_launch(const PvFullParams& p, int dtype, cudaStream_t st) {
  dim3 grid(p.n_splits, p.rows);
  const size_t smem = (2 * (size_t)p.G + (size_t)p.G * 256) * sizeof(float);
  switch (dtype) {
    case KC_F16: pv_full_kernel<__half><<<grid, 256, smem, st>>>(p); break;
    case KC_BF16: pv_full_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(p); break;
    default: pv_full_kernel<float><<<grid, 256, smem, st>>>(p); break;
  }
  const int slots = (p.rows / p.n_kv) * p.n_kv * p.G;
  pv_reduce_kernel<<<grid_for((int64_t)slots * p.h), 256, 0, st>>>(p.part_out, p.out, slots,
                                                                    p.n_splits, p.h);
}

// Pitched row copy with 16-B accesses (prefill V stage -> its host arena when
// the arena is host-resident managed memory: the copy engine writes those
// pages at ~2 GB/s, SM stores at the PCIe rate). A small grid: it runs beside
// the caller's next layer.
__global__ void __launch_bounds__(256) copy_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                        int64_t pitch16, int64_t row16, int rows) {
  const int64_t total = row16 * rows;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t r = i / row16, c = i - r * row16;
    dst[r * pitch16 + c] = __ldcs(src + r * pitch16 + c);
  }
}

__global__ void __launch_bounds__(256) copy_rows_bytes_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                              int64_t pitch, int64_t row_bytes, int rows) {
  const int64_t total = row_bytes * rows;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t r = i / row_bytes, c = i - r * row_bytes;
    dst[r * pitch + c] = src[r * pitch + c];
  }
}

void copy_rows_launch(const void* src, void* dst, int64_t pitch, int64_t row_bytes, int rows, int grid,
                      cudaStream_t st) {
  if (rows <= 0 || row_bytes <= 0) return;
  if ((pitch & 15) == 0 && (row_bytes & 15) == 0 && ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0)
    copy_rows_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), pitch / 16,
                                           row_bytes / 16, rows);
  else
    copy_rows_bytes_kernel<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst),
                                                 pitch, row_bytes, rows);
}

void append_launch(const AppendParams& p, int src_dtype, int dst_dtype, cudaStream_t st) {
  switch (src_dtype) {
    case KC_F16: append_dst<__half>(p, dst_dtype, st); break;
    case KC_BF16: append_dst<__nv_bfloat16>(p, dst_dtype, st); break;
    default: append_dst<float>(p, dst_dtype, st); break;
  }
}

void fill_uniform_launch(void* dst, int dtype, uint64_t n, uint64_t seed, uint64_t offset, float lo,
                         float hi, cudaStream_t st) {
  const int g = grid_for((int64_t)std::min<uint64_t>(n, 1ull << 40));
  switch (dtype) {
    case KC_F16: fill_uniform_kernel<__half><<<g, 256, 0, st>>>((__half*)dst, n, seed, offset, lo, hi); break;
    case KC_BF16: fill_uniform_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((__nv_bfloat16*)dst, n, seed, offset, lo, hi); break;
    default: fill_uniform_kernel<float><<<g, 256, 0, st>>>((float*)dst, n, seed, offset, lo, hi); break;
  }
}

void to_f32_launch(const void* src, int dtype, float* dst, int64_t n, cudaStream_t st) {
  switch (dtype) {
    case KC_F16: to_f32_kernel<__half><<<grid_for(n), 256, 0, st>>>((const __half*)src, dst, n); break;
    case KC_BF16: to_f32_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)src, dst, n); break;
    default: cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st); break;
  }
}

// One-thread marker kernel: the join of a dataflow call into the caller's
// stream runs through it (see decode_topn_impl).
__global__ void join_mark_kernel(uint32_t* word) { *word += 1u; }

void join_mark_launch(uint32_t* word, cudaStream_t st) { join_mark_kernel<<<1, 1, 0, st>>>(word); }

// Test hook: one thread sleeping for ~ns nanoseconds (delays a stream).
__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

void spin_launch(uint64_t ns, cudaStream_t st) { spin_kernel<<<1, 1, 0, st>>>(ns); }


void expand_idx_launch(const uint32_t* src, uint32_t* dst, int rows, int G, int nc, cudaStream_t st) {
  expand_idx_kernel<<<grid_for((int64_t)rows * G * nc), 256, 0, st>>>(src, dst, rows, G, nc);
}

}  // namespace kc

namespace kc {
void gather_rows_launch(const void* base, int dtype, const uint32_t* slot_row, const uint32_t* pos,
                        int64_t n, int h, int64_t max_seq, float* out, cudaStream_t st) {
  if (n <= 0) return;
  const int g = grid_for(n * h);
  switch (dtype) {
    case KC_F16: gather_rows_kernel<__half><<<g, 256, 0, st>>>((const __half*)base, slot_row, pos, n, h, max_seq, out); break;
    case KC_BF16: gather_rows_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)base, slot_row, pos, n, h, max_seq, out); break;
    default: gather_rows_kernel<float><<<g, 256, 0, st>>>((const float*)base, slot_row, pos, n, h, max_seq, out); break;
  }
}
}  // namespace kc

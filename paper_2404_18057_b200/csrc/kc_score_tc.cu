// kc_score_tc.cu -- GQA q.K^T scoring on the 5th-generation tensor cores
// (tcgen05.mma, TMEM accumulators, 2-D TMA) for sm_100a.
//
// Replaces head_weights + dot_scaled (proj/core/src/attention.cpp:15-21,66-78)
// for 2 <= G <= 8 q heads per kv head, h = 128, 16-bit K -- the same contract
// as score_mma_kernel (kc_score.cu): fp32 logits (score * scale, the multiply
// after the sum), per-split online (max, sum exp) per q head, the per-row
// completion signal of the dataflow path.
//
// One CTA per (row, split) item, 192 threads, warp-specialised:
//   warp 0  lane 0: TMA producer -- each stage is 128 positions x 128 dims of
//           K, two 2-D boxes (64 dims x 128 positions, SWIZZLE_128B) of the
//           layer's [rows][max_seq][128] tensor map, i.e. the canonical K-major
//           SW128 operand layout; warp 0 also owns the TMEM allocation;
//   warp 1  lane 0: MMA issuer -- D[128 positions][NB] += K_stage . Qparts^T as
//           8 x tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = NB, K = 16),
//           accumulating in TMEM (two buffers of NB columns), tcgen05.commit
//           frees the smem stage and publishes the buffer;
//   warps 2-5: epilogue -- each thread owns one position (its TMEM lane):
//           tcgen05.ld of its NB columns, q parts summed small first,
//           (a * 2^-e) * scale, logits store (coalesced), running (m, l).
// B = the item's q heads split into NP parts of T (fp16: hi + lo at a
// power-of-two prescale, bf16: three parts -- QSplit, kc_device.cuh), written
// by the epilogue warps into shared memory in the same SW128 layout; row
// n = g * NP + k, rows >= G * NP zero. K is exact in the MMA's input type and
// the MMA accumulates in fp32, so the logits agree with score_mma_kernel's to
// fp32 rounding of a different summation order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "kc_device.cuh"
#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace kc {

namespace {

constexpr int kTcRows = 128;                 // positions per stage (UMMA M)
constexpr int kTcStages = 3;                 // 3 x 32 KB: two CTAs per SM
constexpr int kTcThreads = 192;
constexpr int kStageBytes = kTcRows * 256;   // two 64-dim SW128 boxes
constexpr int kBoxBytes = kTcRows * 128;
constexpr uint32_t kTmemCols = 64;           // two accumulator buffers of <= 32 columns

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start >> 4 [0,14), LBO
  // (unused for swizzled K-major) = 1 [16,30), SBO = 1024 B (8 rows x 128 B)
  // [32,46), version 1 [46,48), layout SWIZZLE_128B = 2 [61,64)
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <typename T, int NB>
__host__ __device__ constexpr uint32_t tc_idesc() {
  // InstrDescriptor: D F32 (bit 4), A/B F16 = 0 / BF16 = 1 ([7,10), [10,13)),
  // both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
  constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void mbar_try(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }

__device__ __forceinline__ void tma_box(uint8_t* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                        uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int NB>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[NB]);
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <typename T, int NB>
__global__ void __launch_bounds__(kTcThreads, 2) score_tc_kernel(const ScoreParams p,
                                                                const __grid_constant__ CUtensorMap kmap) {
  using QS = QSplit<T>;
  constexpr int NP = QS::NP;
  constexpr int kMaxG = 8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                            // [kTcStages][2][128 pos][128 B], SW128
  uint8_t* btile = ring + kTcStages * kStageBytes;  // [2 k-blocks][NB rows][128 B], SW128
  __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], dfull[2], dempty[2], bready;
  __shared__ uint32_t tmem_base;
  __shared__ float post_s[kMaxG];
  __shared__ float2 red[4][kMaxG];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.rows * p.n_splits;
  const int G = p.G, n_q = p.n_kv * G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], 4);
    }
    mbar_init(&bready, 4);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // padding rows of B stay zero for every item
  for (int e = threadIdx.x; e < 2 * NB * 128 / 16; e += kTcThreads)
    reinterpret_cast<uint4*>(btile)[e] = make_uint4(0u, 0u, 0u, 0u);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy(p.k_policy);
      uint32_t g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int row = p.row0 + item / p.n_splits;
        const int split = item - (row - p.row0) * p.n_splits;
        const int pos0 = split * p.chunk;
        const int npos = min(p.chunk, p.s - pos0);
        const int n_it = (npos + kTcRows - 1) / kTcRows;
        for (int it = 0; it < n_it; ++it, ++g) {
          const int st = (int)(g % kTcStages);
          if (g >= (uint32_t)kTcStages) mbar_try(&empty[st], ((g / kTcStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[st], (uint32_t)kStageBytes);
          uint8_t* dst = ring + st * kStageBytes;
          tma_box(dst, &kmap, 0, pos0 + it * kTcRows, row, &full[st], pol);
          tma_box(dst + kBoxBytes, &kmap, 64, pos0 + it * kTcRows, row, &full[st], pol);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = tc_idesc<T, NB>();
      uint32_t g = 0, dcnt = 0, icnt = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int row = p.row0 + item / p.n_splits;
        const int split = item - (row - p.row0) * p.n_splits;
        const int npos = min(p.chunk, p.s - split * p.chunk);
        const int n_it = (npos + kTcRows - 1) / kTcRows;
        mbar_try(&bready, icnt & 1);
        ++icnt;
        tc_fence_after();
        for (int it = 0; it < n_it; ++it, ++g, ++dcnt) {
          const int st = (int)(g % kTcStages);
          const uint32_t buf = dcnt & 1;
          mbar_try(&full[st], (g / kTcStages) & 1);
          if (dcnt >= 2) mbar_try(&dempty[buf], ((dcnt >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + st * kStageBytes), sb = smem_u32(btile);
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = sw128_desc(sa + kb * kBoxBytes + k * 32);
              const uint64_t bd = sw128_desc(sb + kb * NB * 128 + k * 32);
              const uint32_t acc = (kb | k) ? 1u : 0u;
              asm volatile(
                  "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                      tmem + buf * NB),
                  "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
          tc_commit(&empty[st]);   // the smem stage is free once these MMAs completed
          tc_commit(&dfull[buf]);  // and the accumulator buffer is ready
        }
      }
    }
  } else {
    // ---------------- epilogue: one position per thread ----------------
    const int ew = warp - 2;        // 0..3
    const int quad = warp & 3;      // TMEM lanes 32*quad .. 32*quad+31
    const int m_local = 32 * quad + lane;
    uint32_t dcnt = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int row = p.row0 + item / p.n_splits;
      const int split = item - (row - p.row0) * p.n_splits;
      const int b = row / p.n_kv;
      const int kvh = row - b * p.n_kv;
      const int pos0 = split * p.chunk;
      const int npos = min(p.chunk, p.s - pos0);
      const int n_it = (npos + kTcRows - 1) / kTcRows;
      // B: the group's q heads in NP parts (rows g*NP + k), dims 4*lane..+3
      for (int gh = ew; gh < G; gh += 4) {
        const float4 qv = *reinterpret_cast<const float4*>(p.q + ((size_t)b * n_q + kvh * G + gh) * 128 + 4 * lane);
        float amax = fmaxf(fmaxf(fabsf(qv.x), fabsf(qv.y)), fmaxf(fabsf(qv.z), fabsf(qv.w)));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        const float pre = QS::prescale(amax);
        float x0 = qv.x * pre, y0 = qv.y * pre, x1 = qv.z * pre, y1 = qv.w * pre;
        const int d = 4 * lane, kb = d >> 6, c = (d & 63) >> 3, wi = (d & 7) >> 1;  // 32-bit word in the chunk
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const uint32_t w0 = QS::pack(x0, y0), w1 = QS::pack(x1, y1);
          const float2 b0 = QS::unpack(w0), b1 = QS::unpack(w1);
          x0 -= b0.x;
          y0 -= b0.y;
          x1 -= b1.x;
          y1 -= b1.y;
          const int n = gh * NP + k;
          uint32_t* dst = reinterpret_cast<uint32_t*>(btile + kb * NB * 128 + n * 128 + ((c ^ (n & 7)) * 16));
          dst[wi] = w0;
          dst[wi + 1] = w1;
        }
        if (lane == 0) post_s[gh] = 1.0f / pre;  // exact: a power of two
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> the MMA's async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&bready);
      named_sync_n(1, 128);  // post_s of every head
      float mrun[kMaxG], lrun[kMaxG];
#pragma unroll
      for (int gh = 0; gh < kMaxG; ++gh) {
        mrun[gh] = -INFINITY;
        lrun[gh] = 0.0f;
      }
      for (int it = 0; it < n_it; ++it, ++dcnt) {
        const uint32_t buf = dcnt & 1;
        mbar_try(&dfull[buf], (dcnt >> 1) & 1);
        tc_fence_after();
        uint32_t r[NB];
        tmem_ld<NB>(tmem + ((uint32_t)(32 * quad) << 16) + buf * NB, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[buf]);
        const int pl = it * kTcRows + m_local;
        if (pl < npos) {
#pragma unroll
          for (int gh = 0; gh < kMaxG; ++gh) {
            if (gh < G) {
              float a = 0.0f;
#pragma unroll
              for (int k = NP - 1; k >= 0; --k) a += __uint_as_float(r[gh * NP + k]);  // small parts first
              const float sc = (a * post_s[gh]) * p.scale;
              p.logits[((size_t)b * n_q + kvh * G + gh) * p.lstride + pos0 + pl] = sc;
              if (sc > mrun[gh]) {
                lrun[gh] = lrun[gh] * __expf(mrun[gh] - sc) + 1.0f;
                mrun[gh] = sc;
              } else {
                lrun[gh] += __expf(sc - mrun[gh]);
              }
            }
          }
        }
      }
      // per-split (max, sum exp) per head: warp, then the four warps
#pragma unroll
      for (int gh = 0; gh < kMaxG; ++gh) {
        if (gh < G) {
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, mrun[gh], o);
            const float l2 = __shfl_xor_sync(0xffffffffu, lrun[gh], o);
            ml_combine(mrun[gh], lrun[gh], m2, l2);
          }
          if (lane == 0) red[ew][gh] = make_float2(mrun[gh], lrun[gh]);
        }
      }
      named_sync_n(1, 128);
      if (ew == 0 && lane < G) {
        float m = -INFINITY, l = 0.0f;
        for (int w = 0; w < 4; ++w) ml_combine(m, l, red[w][lane].x, red[w][lane].y);
        p.partials[((size_t)b * n_q + kvh * G + lane) * p.max_splits + split] = make_float2(m, l);
      }
      named_sync_n(1, 128);  // red, post_s and B are reused by the next item
      if (p.row_done && ew == 0 && lane == 0) {  // dataflow signal (release after the barrier)
        __threadfence();
        atomicAdd(p.row_done + (size_t)row * kRowDoneStride, 1u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

template <typename T, int NB>
void launch_tc(const ScoreParams& p, const CUtensorMap& map, cudaStream_t st) {
  const size_t smem = kTcStages * kStageBytes + 2 * NB * 128 + 1024;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    cudaFuncSetAttribute(score_tc_kernel<T, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[dev & 63] = 1;
  }
  const int n_items = p.rows * p.n_splits;
  const int grid = p.grid > 0 ? std::min(p.grid, n_items) : n_items;
  score_tc_kernel<T, NB><<<grid, kTcThreads, smem, st>>>(p, map);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

}  // namespace

bool score_tc_supported(int dtype, int h, int G) {
  return (dtype == KC_F16 || dtype == KC_BF16) && h == 128 && G >= 1 && G <= 8;
}

bool encode_k_map(void* map_out, const void* k_layer, int dtype, uint64_t rows, uint64_t max_seq) {
  auto fn = encode_fn();
  if (!fn || !(dtype == KC_F16 || dtype == KC_BF16)) return false;
  const cuuint64_t dims[3] = {128, (cuuint64_t)max_seq, (cuuint64_t)rows};
  const cuuint64_t strides[2] = {256, (cuuint64_t)max_seq * 256};
  const cuuint32_t box[3] = {64, (cuuint32_t)kTcRows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap* m = static_cast<CUtensorMap*>(map_out);
  return fn(m, dtype == KC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
            const_cast<void*>(k_layer), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool score_tc_launch(const ScoreParams& p, int dtype, cudaStream_t st) {
  if (!p.kmap || !score_tc_supported(dtype, p.h, p.G)) return false;
  const CUtensorMap& map = *static_cast<const CUtensorMap*>(p.kmap);
  const int np = dtype == KC_BF16 ? 3 : 2;
  const bool wide = p.G * np > 16;
  if (dtype == KC_BF16) {
    if (wide) launch_tc<__nv_bfloat16, 32>(p, map, st);
    else launch_tc<__nv_bfloat16, 16>(p, map, st);
  } else {
    if (wide) launch_tc<__half, 32>(p, map, st);
    else launch_tc<__half, 16>(p, map, st);
  }
  return true;
}

}  // namespace kc

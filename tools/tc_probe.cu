// tc_probe.cu -- development probe (not the product): one tcgen05.mma tile of
// the GQA scoring shape, to validate the descriptors before a kernel uses
// them. D[pos][n] = sum_k K[row][pos][k] * Q[n][k] for 128 positions, N = 16,
// K = 128 (fp16 inputs, fp32 accumulation in TMEM):
//   * K tile: two 2-D TMA boxes (64 dims x 128 positions, SWIZZLE_128B) from a
//     [rows][S][128] fp16 tensor map -> the canonical K-major SW128 layout;
//   * Q: written to shared memory by threads in the same SW128 layout;
//   * 8 x tcgen05.mma.cta_group::1.kind::f16 (M=128, N=16, K=16), commit to an
//     mbarrier, tcgen05.ld 32x32b.x16 by four epilogue warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start >> 4 [0,14), LBO >> 4
  // [16,30) (unused for swizzled K-major: 1), SBO >> 4 [32,46) = 1024 B (8 rows
  // x 128 B), version [46,48) = 1, base offset 0, layout [61,64) = 2 (SW128)
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

constexpr uint32_t kIdesc =  // InstrDescriptor: c F32 (bit 4), a/b F16 (0), K-major, N>>3 at 17, M>>4 at 24
    (1u << 4) | (0u << 7) | (0u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__global__ void __launch_bounds__(192) probe(const __grid_constant__ CUtensorMap tmap, const __half* q, int row,
                                            int pos0, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* atile = smem;            // 2 x 16 KB (dims 0-63, 64-127)
  uint8_t* btile = smem + 32768;    // 2 x 2 KB
  __shared__ __align__(8) uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_tma)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Q -> SW128 K-major: row n, 16-B chunk c of k-block kb at n*128 + ((c ^ (n & 7)) * 16)
  for (int e = threadIdx.x; e < 16 * 16; e += 192) {
    const int n = e >> 4, cc = e & 15, kb = cc >> 3, c = cc & 7;
    const uint4 v = reinterpret_cast<const uint4*>(q + n * 128)[cc];
    *reinterpret_cast<uint4*>(btile + kb * 2048 + n * 128 + ((c ^ (n & 7)) * 16)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_tma)), "r"(32768)
                 : "memory");
    for (int kb = 0; kb < 2; ++kb)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(atile + kb * 16384)),
          "l"(&tmap), "r"(kb * 64), "r"(pos0), "r"(row), "r"(smem_u32(&bar_tma))
          : "memory");
  }
  if (warp == 1) {
    if (lane == 0) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(&bar_tma))
                     : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < 2; ++kb)
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sw128_desc(smem_u32(atile + kb * 16384 + k * 32));
          const uint64_t bd = sw128_desc(smem_u32(btile + kb * 2048 + k * 32));
          const uint32_t acc = (kb | k) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                  tmem),
              "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar_mma))
                   : "memory");
    }
    __syncwarp();
  }
  if (warp >= 2) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem_u32(&bar_mma))
                   : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;  // TMEM lanes 32*quad .. +32
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(32 * quad) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = 32 * quad + lane;
    for (int n = 0; n < 16; ++n) out[m * 16 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  const int R = 3, S = 512, H = 128;
  std::vector<__half> k((size_t)R * S * H), q(16 * H);
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (auto& x : k) x = __float2half(u(rng));
  for (auto& x : q) x = __float2half(u(rng));
  __half *dk = nullptr, *dq = nullptr;
  float* dout = nullptr;
  CK(cudaMalloc(&dk, k.size() * 2));
  CK(cudaMalloc(&dq, q.size() * 2));
  CK(cudaMalloc(&dout, 128 * 16 * 4));
  CK(cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled encode = nullptr;
  cudaDriverEntryPointQueryResult qres;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qres));
  CUtensorMap tmap;
  const cuuint64_t dims[3] = {(cuuint64_t)H, (cuuint64_t)S, (cuuint64_t)R};
  const cuuint64_t strides[2] = {(cuuint64_t)H * 2, (cuuint64_t)S * H * 2};
  const cuuint32_t box[3] = {64, 128, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, dk, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    std::printf("encode failed %d\n", (int)cr);
    return 1;
  }
  const int row = 1, pos0 = 128;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  probe<<<1, 192, 40 * 1024>>>(tmap, dq, row, pos0, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> out(128 * 16);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double ref = 0;
      for (int kk = 0; kk < H; ++kk)
        ref += (double)__half2float(k[((size_t)row * S + pos0 + m) * H + kk]) * (double)__half2float(q[n * H + kk]);
      const double err = std::fabs(ref - out[m * 16 + n]);
      maxerr = std::max(maxerr, err);
      if (err > 1e-3 && bad++ < 5) std::printf("m %d n %d ref %f got %f\n", m, n, ref, out[m * 16 + n]);
    }
  std::printf("{\"probe\": \"tcgen05 f16 M128 N16 K128\", \"max_abs_err\": %g, \"bad\": %d}\n", maxerr, bad);
  return bad ? 1 : 0;
}

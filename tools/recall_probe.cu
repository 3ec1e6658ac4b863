// recall_probe.cu -- development probe (not the product): how fast can the
// SMs gather scattered 256-B V rows (one C2 layer's selection: 256 rows x
// 128 positions = 8 MiB) out of a host-resident UVM arena, by method:
//   ld16  : 16-B loads, U in flight per thread (the product's recall pattern)
//   tma   : one thread per CTA issues cp.async.bulk of each 256-B row into a
//           shared-memory stage (mbarrier complete_tx), R rows per stage
// and by grid size. Reference: the copy engine's pinned H2D rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/recall_probe tools/recall_probe.cu
//   tools/recall_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int kRowB = 256;          // one V row: h=128 fp16
constexpr int kSel = 128;           // selected positions per (batch, kv head)
constexpr int kRows = 256;          // (batch, kv head) rows of a C2 layer
constexpr long kSeq = 32768;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int U>
__global__ void __launch_bounds__(256) gather_ld16(const uint4* __restrict__ v, const unsigned* __restrict__ idx,
                                                   float* sink) {
  float acc = 0.f;
  for (int row = blockIdx.x; row < kRows; row += gridDim.x) {
    const uint4* base = v + (size_t)row * kSeq * (kRowB / 16);
    const unsigned* ir = idx + row * kSel;
    constexpr int total = kSel * (kRowB / 16);  // 2048 16-B pieces
    for (int v0 = threadIdx.x; v0 < total; v0 += 256 * U) {
      uint4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = v0 + u * 256;
        if (e < total) t[u] = base[(size_t)ir[e >> 4] * 16 + (e & 15)];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __uint_as_float(t[u].x ^ t[u].w);
    }
  }
  if (acc == 1.2345f) sink[0] = acc;
}

// R rows per stage, 2 stages; thread 0 issues, everyone consumes (xor-sum)
template <int R>
__global__ void __launch_bounds__(256) gather_tma(const char* __restrict__ v, const unsigned* __restrict__ idx,
                                                  float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  unsigned phase[2] = {0, 0};
  constexpr int stages_per_row = kSel / R;
  int g = 0;
  auto issue = [&](int gi) {
    const int row = blockIdx.x + (gi / stages_per_row) * gridDim.x;
    if (row >= kRows) return;
    const int st = gi & 1;
    const int r0 = (gi % stages_per_row) * R;
    const char* base = v + (size_t)row * kSeq * kRowB;
    const unsigned* ir = idx + row * kSel + r0;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(R * kRowB)
                 : "memory");
    for (int r = 0; r < R; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + (st * R + r) * kRowB)),
          "l"(base + (size_t)ir[r] * kRowB), "r"(kRowB), "r"(smem_u32(&bar[st]))
          : "memory");
  };
  const int my_rows = (kRows - (int)blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int n_st = my_rows * stages_per_row;
  if (threadIdx.x == 0) {
    issue(0);
    if (n_st > 1) issue(1);
  }
  for (g = 0; g < n_st; ++g) {
    const int st = g & 1;
    unsigned done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem_u32(&bar[st])), "r"(phase[st])
                   : "memory");
    } while (!done);
    phase[st] ^= 1;
    const uint4* s4 = reinterpret_cast<const uint4*>(sm + st * R * kRowB);
    for (int e = threadIdx.x; e < R * kRowB / 16; e += 256) acc += __uint_as_float(s4[e].x ^ s4[e].w);
    __syncthreads();
    if (threadIdx.x == 0 && g + 2 < n_st) issue(g + 2);
  }
  if (acc == 1.2345f) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)kRows * kSeq * kRowB;  // 2 GiB
  int dev = 0;
  CK(cudaSetDevice(dev));
  void* v = nullptr;
  CK(cudaMallocManaged(&v, bytes, cudaMemAttachGlobal));
  cudaMemLocation host{};
  host.type = cudaMemLocationTypeHost;
  cudaMemLocation gpu{};
  gpu.type = cudaMemLocationTypeDevice;
  gpu.id = dev;
  CK(cudaMemAdvise(v, bytes, cudaMemAdviseSetPreferredLocation, host));
  CK(cudaMemAdvise(v, bytes, cudaMemAdviseSetAccessedBy, gpu));
  CK(cudaMemPrefetchAsync(v, bytes, host, 0, nullptr));
  CK(cudaDeviceSynchronize());
  for (size_t i = 0; i < bytes; i += 4096) static_cast<char*>(v)[i] = (char)i;

  constexpr int kReps = 24;
  std::vector<unsigned> hidx((size_t)kReps * kRows * kSel);
  std::mt19937 rng(1);
  for (int rep = 0; rep < kReps; ++rep)
    for (int r = 0; r < kRows; ++r) {
      std::vector<unsigned> pos(kSel);
      for (auto& p : pos) p = rng() % kSeq;
      std::sort(pos.begin(), pos.end());
      std::copy(pos.begin(), pos.end(), hidx.begin() + ((size_t)rep * kRows + r) * kSel);
    }
  unsigned* didx = nullptr;
  float* sink = nullptr;
  CK(cudaMalloc(&didx, hidx.size() * 4));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemcpy(didx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double gather_bytes = (double)kRows * kSel * kRowB;
  // L2 flush between timed reps (every method reuses the same index sets)
  void* flush = nullptr;
  const size_t flush_bytes = 512ull << 20;
  CK(cudaMalloc(&flush, flush_bytes));

  auto run = [&](const char* name, int grid, auto launch) {
    for (int w = 0; w < 2; ++w) launch(grid, didx + (size_t)w * kRows * kSel);
    CK(cudaDeviceSynchronize());
    float best = 1e9, tot = 0;
    for (int rep = 2; rep < kReps; ++rep) {
      CK(cudaMemsetAsync(flush, rep, flush_bytes));
      CK(cudaEventRecord(a));
      launch(grid, didx + (size_t)rep * kRows * kSel);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
      tot += ms;
    }
    CK(cudaGetLastError());
    const float avg = tot / (kReps - 2);
    std::printf("{\"method\": \"%s\", \"grid\": %d, \"avg_us\": %.1f, \"best_us\": %.1f, \"avg_gbs\": %.1f}\n", name,
                grid, avg * 1e3, best * 1e3, gather_bytes / (avg * 1e-3) / 1e9);
  };
  for (int grid : {32, 64, 128, 256}) {
    run("ld16_u8", grid, [&](int g, unsigned* ix) { gather_ld16<8><<<g, 256>>>((const uint4*)v, ix, sink); });
    run("ld16_u16", grid, [&](int g, unsigned* ix) { gather_ld16<16><<<g, 256>>>((const uint4*)v, ix, sink); });
    run("tma_r32", grid, [&](int g, unsigned* ix) {
      gather_tma<32><<<g, 256, 2 * 32 * kRowB>>>((const char*)v, ix, sink);
    });
    run("tma_r64", grid, [&](int g, unsigned* ix) {
      gather_tma<64><<<g, 256, 2 * 64 * kRowB>>>((const char*)v, ix, sink);
    });
    run("tma_r128", grid, [&](int g, unsigned* ix) {
      cudaFuncSetAttribute(gather_tma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * kRowB);
      gather_tma<128><<<g, 256, 2 * 128 * kRowB>>>((const char*)v, ix, sink);
    });
  }
  // copy engine reference: pinned 256 MiB H2D
  {
    void *hp = nullptr, *dp = nullptr;
    const size_t n = 256 << 20;
    CK(cudaHostAlloc(&hp, n, 0));
    CK(cudaMalloc(&dp, n));
    float best = 1e9;
    for (int i = 0; i < 6; ++i) {
      CK(cudaEventRecord(a));
      CK(cudaMemcpyAsync(dp, hp, n, cudaMemcpyHostToDevice));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    std::printf("{\"method\": \"copy_engine_h2d\", \"gbs\": %.1f}\n", n / (best * 1e-3) / 1e9);
  }
  return 0;
}

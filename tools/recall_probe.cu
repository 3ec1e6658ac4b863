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

template <int U, int HINT, int NT>
__global__ void __launch_bounds__(NT) gather_ld16(const uint4* __restrict__ v, const unsigned* __restrict__ idx,
                                                  float* sink) {
  float acc = 0.f;
  for (int row = blockIdx.x; row < kRows; row += gridDim.x) {
    const uint4* base = v + (size_t)row * kSeq * (kRowB / 16);
    const unsigned* ir = idx + row * kSel;
    constexpr int total = kSel * (kRowB / 16);  // 2048 16-B pieces
    for (int v0 = threadIdx.x; v0 < total; v0 += NT * U) {
      uint4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = v0 + u * NT;
        if (e < total) {
          const uint4* a = base + (size_t)ir[e >> 4] * 16 + (e & 15);
          if (HINT == 1)
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t[u].x), "=r"(t[u].y), "=r"(t[u].z), "=r"(t[u].w) : "l"(a));
          else if (HINT == 2)
            asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t[u].x), "=r"(t[u].y), "=r"(t[u].z), "=r"(t[u].w) : "l"(a));
          else
            t[u] = *a;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __uint_as_float(t[u].x ^ t[u].w);
    }
  }
  if (acc == 1.2345f) sink[0] = acc;
}

// background HBM stream (stands in for the scoring kernel)
__global__ void __launch_bounds__(512) hbm_stream(const uint4* __restrict__ a, size_t n16, float* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * 512ull + threadIdx.x; i < n16; i += (size_t)gridDim.x * 512) {
    uint4 t = __ldcs(a + i);
    acc += __uint_as_float(t.x ^ t.y);
  }
  if (acc == 1.2345f) sink[1] = acc;
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
  for (int grid : {32, 64, 148, 296}) {
    run("ld16_u8", grid, [&](int g, unsigned* ix) { gather_ld16<8, 0, 256><<<g, 256>>>((const uint4*)v, ix, sink); });
    run("ld16_u8_l2_256", grid, [&](int g, unsigned* ix) { gather_ld16<8, 1, 256><<<g, 256>>>((const uint4*)v, ix, sink); });
    run("ld16_u8_l2_128", grid, [&](int g, unsigned* ix) { gather_ld16<8, 2, 256><<<g, 256>>>((const uint4*)v, ix, sink); });
    run("ld16_u2_t1024", grid, [&](int g, unsigned* ix) { gather_ld16<2, 0, 1024><<<g, 1024>>>((const uint4*)v, ix, sink); });
    run("ld16_u2_t1024_l2_256", grid, [&](int g, unsigned* ix) { gather_ld16<2, 1, 1024><<<g, 1024>>>((const uint4*)v, ix, sink); });
    run("tma_r32", grid, [&](int g, unsigned* ix) {
      gather_tma<32><<<g, 256, 2 * 32 * kRowB>>>((const char*)v, ix, sink);
    });
    run("tma_r64", grid, [&](int g, unsigned* ix) {
      gather_tma<64><<<g, 256, 2 * 64 * kRowB>>>((const char*)v, ix, sink);
    });
  }
  // under a concurrent HBM stream (the in-step condition)
  {
    const size_t hb = 8ull << 30;
    void* hbm = nullptr;
    CK(cudaMalloc(&hbm, hb));
    CK(cudaMemset(hbm, 1, hb));
    cudaStream_t bg;
    CK(cudaStreamCreateWithPriority(&bg, cudaStreamNonBlocking, 0));
    cudaEvent_t h0, h1;
    CK(cudaEventCreate(&h0));
    CK(cudaEventCreate(&h1));
    CK(cudaEventRecord(h0, bg));
    hbm_stream<<<148 * 2, 512, 0, bg>>>((const uint4*)hbm, hb / 16, sink);
    CK(cudaEventRecord(h1, bg));
    CK(cudaDeviceSynchronize());
    float hms = 0;
    CK(cudaEventElapsedTime(&hms, h0, h1));
    std::printf("{\"method\": \"hbm_stream_alone\", \"ms\": %.3f, \"gbs\": %.1f}\n", hms, hb / (hms * 1e-3) / 1e9);
    for (int grid : {32, 64, 148}) {
      for (int m = 0; m < 3; ++m) {
        float tot = 0;
        const int reps = 6;
        float hsum = 0;
        for (int rep = 0; rep < reps; ++rep) {
          CK(cudaEventRecord(h0, bg));
          hbm_stream<<<148 * 2, 512, 0, bg>>>((const uint4*)hbm, hb / 16, sink);
          CK(cudaEventRecord(h1, bg));
          // let the stream ramp, then gather 8 layers back to back
          CK(cudaEventRecord(a));
          for (int l = 0; l < 8; ++l) {
            unsigned* ix = didx + (size_t)((rep * 8 + l) % kReps) * kRows * kSel;
            if (m == 0) gather_ld16<8, 0, 256><<<grid, 256>>>((const uint4*)v, ix, sink);
            else if (m == 1) gather_ld16<8, 1, 256><<<grid, 256>>>((const uint4*)v, ix, sink);
            else gather_tma<32><<<grid, 256, 2 * 32 * kRowB>>>((const char*)v, ix, sink);
          }
          CK(cudaEventRecord(b));
          CK(cudaDeviceSynchronize());
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a, b));
          tot += ms / 8;
          CK(cudaEventElapsedTime(&ms, h0, h1));
          hsum += ms;
        }
        const char* nm[3] = {"ld16_u8", "ld16_u8_l2_256", "tma_r32"};
        std::printf("{\"method\": \"%s+hbm\", \"grid\": %d, \"avg_us\": %.1f, \"avg_gbs\": %.1f, \"hbm_ms\": %.3f}\n",
                    nm[m], grid, tot / reps * 1e3, gather_bytes / (tot / reps * 1e-3) / 1e9, hsum / reps);
      }
    }
  }
  // copy engine, batched 256-B copies (pointer arrays prebuilt: the best case)
  {
    const size_t n = (size_t)kRows * kSel;
    std::vector<void*> dsts(n), srcs(n);
    std::vector<size_t> sizes(n, kRowB);
    char* dbuf = nullptr;
    CK(cudaMalloc(&dbuf, n * kRowB));
    for (size_t i = 0; i < n; ++i) {
      const size_t row = i / kSel;
      dsts[i] = dbuf + i * kRowB;
      srcs[i] = static_cast<char*>(v) + (row * kSeq + hidx[i]) * kRowB;
    }
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.srcLocHint.type = cudaMemLocationTypeHost;
    attr.dstLocHint.type = cudaMemLocationTypeDevice;
    attr.dstLocHint.id = 0;
    size_t aidx = 0, fail = 0;
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    float best = 1e9, tot = 0;
    for (int rep = 0; rep < 6; ++rep) {
      CK(cudaEventRecord(a, cs));
      cudaError_t e = cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), n, &attr, &aidx, 1, &fail, cs);
      if (e != cudaSuccess) { std::printf("{\"method\": \"memcpy_batch\", \"error\": \"%s\"}\n", cudaGetErrorString(e)); cudaGetLastError(); break; }
      CK(cudaEventRecord(b, cs));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
      if (rep) tot += ms;
    }
    std::printf("{\"method\": \"memcpy_batch_256B\", \"best_us\": %.1f, \"avg_us\": %.1f, \"gbs\": %.1f}\n", best * 1e3,
                tot / 5 * 1e3, gather_bytes / (best * 1e-3) / 1e9);
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

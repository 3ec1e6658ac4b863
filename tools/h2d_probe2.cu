// h2d_probe2.cu -- why does a device-memory sweep slow down zero-copy row
// gathers, and how fast is a host-side gather + one contiguous DMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_probe2 h2d_probe2.cu -lpthread
#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void seq_read(const uint4* src, size_t n16, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__global__ void seq_read_ef(const uint4* src, size_t n16, uint4* sink) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i), "l"(pol));
    acc ^= v.x;
  }
  if (acc == 0x12345678) sink[0].x = acc;
}

// read then discard the L2 lines (no write-back) so the sweep leaves L2 empty
__global__ void seq_read_discard(const uint4* src, size_t n16, uint4* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc ^= v.x;
    if ((i & 7) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(src + i) : "memory");
  }
  if (acc == 0x12345678) sink[0].x = acc;
}

// gather with an L2 cache-policy hint on the sysmem loads (kind: 0 evict_last, 1 evict_unchanged, 2 evict_first)
__global__ void slot_gather_pol(const uint4* base, const uint32_t* rows, uint4* out, int kind) {
  __shared__ uint4 sm[2048];
  uint64_t pol;
  if (kind == 0) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint32_t* r = rows + blockIdx.x * 128;
  uint4 t[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    int v = threadIdx.x + u * 256;
    const uint4* a = base + (size_t)r[v >> 4] * 16 + (v & 15);
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(t[u].x), "=r"(t[u].y), "=r"(t[u].z), "=r"(t[u].w)
                 : "l"(a), "l"(pol));
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) sm[threadIdx.x + u * 256] = t[u];
  __syncthreads();
  if (threadIdx.x < 16) out[blockIdx.x * 16 + threadIdx.x] = sm[threadIdx.x * 7];
}

__global__ void slot_gather(const uint4* base, const uint32_t* rows, uint4* out) {
  __shared__ uint4 sm[2048];
  const uint32_t* r = rows + blockIdx.x * 128;
  uint4 t[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    int v = threadIdx.x + u * 256;
    t[u] = base[(size_t)r[v >> 4] * 16 + (v & 15)];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) sm[threadIdx.x + u * 256] = t[u];
  __syncthreads();
  if (threadIdx.x < 16) out[blockIdx.x * 16 + threadIdx.x] = sm[threadIdx.x * 7];
}

int main() {
  const size_t region = 2ull << 30;
  const int nregions = 8;
  const size_t total = region * nregions;
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  char* a = (char*)mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  for (size_t i = 0; i < total; i += 4096) a[i] = (char)i;
  CK(cudaHostRegister(a, total, cudaHostRegisterMapped));
  void* a_dev;
  CK(cudaHostGetDevicePointer(&a_dev, a, 0));
  const int nrows = 32768;
  std::vector<uint32_t> h_rows(nrows * nregions);
  srand(1);
  for (int rg = 0; rg < nregions; ++rg)
    for (int slot = 0; slot < 256; ++slot) {
      uint32_t* p = &h_rows[rg * nrows + slot * 128];
      for (int k = 0; k < 128; ++k) p[k] = slot * 32768 + rand() % 32768;
      std::sort(p, p + 128);
    }
  uint32_t* d_rows;
  CK(cudaMalloc(&d_rows, h_rows.size() * 4));
  CK(cudaMemcpy(d_rows, h_rows.data(), h_rows.size() * 4, cudaMemcpyHostToDevice));
  uint4 *gout, *dbuf, *big;
  CK(cudaMalloc(&gout, (size_t)nrows * 256));
  CK(cudaMalloc(&dbuf, 1 << 20));
  CK(cudaMalloc(&big, 2ull << 30));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto gather_after = [&](size_t sweep_bytes, int sleep_us) {
    float tot = 0;
    for (int rg = 0; rg < nregions; ++rg) {
      if (sweep_bytes) seq_read<<<1184, 256, 0, st>>>(big, sweep_bytes / 16, dbuf);
      CK(cudaStreamSynchronize(st));
      if (sleep_us) std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
      cudaEventRecord(e0, st);
      slot_gather<<<256, 256, 0, st>>>((const uint4*)((char*)a_dev + rg * region), d_rows + rg * nrows, gout);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    return tot / nregions * 1e3;
  };
  printf("gather, no sweep: %.1f us\n", gather_after(0, 0));
  for (size_t sw : {32ull << 20, 96ull << 20, 256ull << 20, 1ull << 30, 2ull << 30})
    printf("gather after %zu MiB device sweep: %.1f us\n", sw >> 20, gather_after(sw, 0));
  printf("gather after 2 GiB sweep + 2 ms idle: %.1f us\n", gather_after(2ull << 30, 2000));
  auto gather_after_k = [&](int kind) {
    float tot = 0, tot2 = 0;
    for (int rg = 0; rg < nregions; ++rg) {
      if (kind == 0) seq_read_ef<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
      if (kind == 1) seq_read_discard<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
      if (kind == 2) seq_read<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0, st);
        slot_gather<<<256, 256, 0, st>>>((const uint4*)((char*)a_dev + rg * region), d_rows + rg * nrows, gout);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        (rep ? tot2 : tot) += ms;
      }
    }
    printf("  first gather %.1f us, second gather %.1f us\n", tot / nregions * 1e3, tot2 / nregions * 1e3);
  };
  printf("after evict_first sweep:\n");
  gather_after_k(0);
  printf("after sweep + discard.global.L2:\n");
  gather_after_k(1);
  printf("after normal sweep:\n");
  gather_after_k(2);
  for (size_t carve : {0ull, 16ull << 20, 64ull << 20}) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
    for (int kind = 0; kind < 3; ++kind) {
      float tot = 0;
      for (int rg = 0; rg < nregions; ++rg) {
        seq_read<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
        cudaEventRecord(e0, st);
        slot_gather_pol<<<256, 256, 0, st>>>((const uint4*)((char*)a_dev + rg * region), d_rows + rg * nrows, gout,
                                             kind);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      printf("persist carve %zu MiB, gather policy %s, after sweep: %.1f us\n", carve >> 20,
             kind == 0 ? "evict_last" : kind == 1 ? "evict_unchanged" : "evict_first", tot / nregions * 1e3);
    }
  }
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);

  // host-side gather of one layer's 32768 rows into pinned staging + one DMA
  char* stage;
  CK(cudaHostAlloc((void**)&stage, (size_t)nrows * 256, cudaHostAllocPortable));
  for (int threads : {1, 2, 4, 8, 16}) {
    double best = 1e9;
    for (int rg = 0; rg < nregions; ++rg) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
          const uint32_t* rows = &h_rows[rg * nrows];
          const char* base = a + rg * region;
          for (int r = t; r < nrows; r += threads) memcpy(stage + (size_t)r * 256, base + (size_t)rows[r] * 256, 256);
        });
      for (auto& th : pool) th.join();
      double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, us);
    }
    printf("host gather 8 MiB with %d threads (incl. spawn): %.1f us (%.1f GB/s)\n", threads, best,
           (8 << 20) / (best * 1e-6) / 1e9);
  }
  for (int sweep = 0; sweep < 2; ++sweep) {
    float tot = 0;
    for (int rg = 0; rg < nregions; ++rg) {
      if (sweep) seq_read<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
      cudaEventRecord(e0, st);
      cudaMemcpyAsync(gout, stage, (size_t)nrows * 256, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("DMA 8 MiB contiguous %s sweep: %.1f us\n", sweep ? "after" : "without", tot / nregions * 1e3);
  }
  // DMA concurrent with a device sweep on another stream
  {
    cudaStream_t s2;
    cudaStreamCreate(&s2);
    cudaEvent_t f0, f1;
    cudaEventCreate(&f0);
    cudaEventCreate(&f1);
    seq_read<<<1184, 256, 0, s2>>>(big, (2ull << 30) / 16, dbuf);
    cudaEventRecord(f0, st);
    cudaMemcpyAsync(gout, stage, (size_t)nrows * 256, cudaMemcpyHostToDevice, st);
    cudaEventRecord(f1, st);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, f0, f1);
    printf("DMA 8 MiB concurrent with a 2 GiB sweep: %.1f us\n", ms * 1e3);
    cudaEventRecord(f0, s2);
    seq_read<<<1184, 256, 0, s2>>>(big, (2ull << 30) / 16, dbuf);
    cudaEventRecord(f1, s2);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, f0, f1);
    printf("2 GiB sweep alone: %.1f us (%.0f GB/s)\n", ms * 1e3, (2ull << 30) / (ms * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}

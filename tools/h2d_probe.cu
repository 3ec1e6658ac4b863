// h2d_probe.cu -- host->device recall microbenchmarks on the B200 box.
// Measures: DMA H2D bandwidth, zero-copy sequential reads, and zero-copy
// random 256-B row gathers (the V-recall access pattern) from pinned host
// memory allocated three ways, cold (fresh region per launch) and warm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_probe h2d_probe.cu
#include <sys/mman.h>
#include <cuda.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));      \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__global__ void seq_read(const uint4* src, size_t n16, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// rows: list of 256-B row indices; each warp gathers rows 2 at a time (16 lanes x 16 B)
template <int UNROLL>
__global__ void gather_rows(const uint4* base, const uint32_t* rows, int nrows, uint4* out) {
  const int lane = threadIdx.x & 15;
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int ngrp = (gridDim.x * blockDim.x) >> 4;
  for (int r0 = grp; r0 < nrows; r0 += ngrp * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int r = r0 + u * ngrp;
      if (r < nrows) v[u] = base[(size_t)rows[r] * 16 + lane];
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int r = r0 + u * ngrp;
      if (r < nrows) out[(size_t)r * 16 + lane] = v[u];
    }
  }
}

// recall-like: one CTA per slot, 128 sorted rows, 256 threads x 8 loads -> smem
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

__global__ void gpu_write(uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4(i, i, i, i);
}

float time_it(cudaStream_t st, void (*fn)(void*), void* ctx, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  fn(ctx);
  CK(cudaStreamSynchronize(st));
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < reps; ++i) fn(ctx);
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  const size_t region = 2ull << 30;    // one layer's V arena (C2)
  const int nregions = 8;
  const size_t total = region * nregions;
  cudaStream_t st;
  CK(cudaStreamCreate(&st));

  // allocation A: mmap + THP + cudaHostRegister(mapped)
  void* a = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(a, total, MADV_HUGEPAGE);
  memset(a, 1, total);
  CK(cudaHostRegister(a, total, cudaHostRegisterMapped | cudaHostRegisterPortable));
  void* a_dev;
  CK(cudaHostGetDevicePointer(&a_dev, a, 0));
  // allocation B: cudaHostAlloc(mapped)
  void* bh;
  CK(cudaHostAlloc(&bh, total, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(bh, 1, total);
  void* b_dev;
  CK(cudaHostGetDevicePointer(&b_dev, bh, 0));

  uint4* dbuf;
  CK(cudaMalloc(&dbuf, 256 << 20));
  // DMA
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int i = 0; i < 5; ++i) {
      cudaEventRecord(e0, st);
      cudaMemcpyAsync(dbuf, a, 256 << 20, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = best < ms ? best : ms;
    }
    printf("DMA H2D 256MiB (mmap+register): %.1f GB/s\n", (256 << 20) / (best * 1e-3) / 1e9);
  }
  // sequential zero-copy
  for (int which = 0; which < 2; ++which) {
    const uint4* src = (const uint4*)(which ? b_dev : a_dev);
    for (int grid : {148, 296, 592, 1184}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      seq_read<<<grid, 256, 0, st>>>(src, (256 << 20) / 16, dbuf);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("zero-copy seq 256MiB alloc=%s grid=%d: %.1f GB/s\n", which ? "cudaHostAlloc" : "mmap+reg", grid,
             (256 << 20) / (ms * 1e-3) / 1e9);
    }
  }
  // random row gathers: 32768 rows (8 MiB) per launch; rows = 256 slots x 128
  // rows each, each slot's rows within its own 8 MiB (32768 positions x 256 B)
  const int nrows = 32768;
  std::vector<uint32_t> h_rows(nrows * nregions);
  srand(1);
  for (int rg = 0; rg < nregions; ++rg)
    for (int slot = 0; slot < 256; ++slot) {
      for (int k = 0; k < 128; ++k) {
        uint32_t pos = rand() % 32768;
        h_rows[rg * nrows + slot * 128 + k] = slot * 32768 + pos;
      }
    }
  uint32_t* d_rows;
  CK(cudaMalloc(&d_rows, h_rows.size() * 4));
  CK(cudaMemcpy(d_rows, h_rows.data(), h_rows.size() * 4, cudaMemcpyHostToDevice));
  uint4* gout;
  CK(cudaMalloc(&gout, (size_t)nrows * 256));
  for (int which = 0; which < 2; ++which) {
    char* base = (char*)(which ? b_dev : a_dev);
    for (int grid : {64, 148, 296, 592}) {
      for (int threads : {128, 256}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        // cold: a different 2 GiB region each launch
        float cold = 0, warm = 0;
        for (int rep = 0; rep < 2; ++rep) {
          for (int rg = 0; rg < nregions; ++rg) {
            cudaEventRecord(e0, st);
            gather_rows<8><<<grid, threads, 0, st>>>((const uint4*)(base + rg * region), d_rows + rg * nrows, nrows,
                                                     gout);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 1) cold += ms;
          }
        }
        for (int rep = 0; rep < 8; ++rep) {
          cudaEventRecord(e0, st);
          gather_rows<8><<<grid, threads, 0, st>>>((const uint4*)base, d_rows, nrows, gout);
          cudaEventRecord(e1, st);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep > 0) warm += ms;
        }
        cold /= nregions;
        warm /= 7;
        printf("gather 8MiB of 256B rows alloc=%s grid=%d thr=%d: cold %.1f us (%.1f GB/s), warm %.1f us (%.1f GB/s)\n",
               which ? "cudaHostAlloc" : "mmap+reg", grid, threads, cold * 1e3, (8 << 20) / (cold * 1e-3) / 1e9,
               warm * 1e3, (8 << 20) / (warm * 1e-3) / 1e9);
      }
    }
  }
  // allocation C: library style (MAP_NORESERVE, THP advice, no CPU touch,
  // register, then filled by GPU mapped writes); sorted rows per slot
  void* c = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  madvise(c, total, MADV_HUGEPAGE);
  CK(cudaHostRegister(c, total, cudaHostRegisterMapped | cudaHostRegisterPortable));
  void* c_dev;
  CK(cudaHostGetDevicePointer(&c_dev, c, 0));
  gpu_write<<<1184, 256, 0, st>>>((uint4*)c_dev, total / 16);
  CK(cudaStreamSynchronize(st));
  for (int rg = 0; rg < nregions; ++rg)
    for (int slot = 0; slot < 256; ++slot) {
      uint32_t* p = &h_rows[rg * nrows + slot * 128];
      std::sort(p, p + 128);
    }
  CK(cudaMemcpy(d_rows, h_rows.data(), h_rows.size() * 4, cudaMemcpyHostToDevice));
  for (int which = 0; which < 3; ++which) {
    char* base = (char*)(which == 0 ? a_dev : which == 1 ? b_dev : c_dev);
    const char* nm = which == 0 ? "mmap+reg" : which == 1 ? "cudaHostAlloc" : "lib-style";
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int kind = 0; kind < 2; ++kind) {
      float tot = 0;
      for (int rg = 0; rg < nregions; ++rg) {
        cudaEventRecord(e0, st);
        if (kind == 0)
          slot_gather<<<256, 256, 0, st>>>((const uint4*)(base + rg * region), d_rows + rg * nrows, gout);
        else
          gather_rows<8><<<296, 256, 0, st>>>((const uint4*)(base + rg * region), d_rows + rg * nrows, nrows, gout);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      tot /= nregions;
      printf("%s alloc=%s sorted rows: %.1f us (%.1f GB/s)\n", kind ? "gather_rows" : "slot_gather", nm, tot * 1e3,
             (8 << 20) / (tot * 1e-3) / 1e9);
    }
  }
  // TLB hypothesis: sweep 2 GiB of device memory between gathers
  {
    uint4* big;
    CK(cudaMalloc(&big, 2ull << 30));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int sweep = 0; sweep < 2; ++sweep) {
      float tot = 0;
      for (int rg = 0; rg < nregions; ++rg) {
        if (sweep) seq_read<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
        cudaEventRecord(e0, st);
        slot_gather<<<256, 256, 0, st>>>((const uint4*)((char*)a_dev + rg * region), d_rows + rg * nrows, gout);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      tot /= nregions;
      printf("slot_gather %s device sweep between: %.1f us (%.1f GB/s)\n", sweep ? "WITH" : "without", tot * 1e3,
             (8 << 20) / (tot * 1e-3) / 1e9);
    }
    // allocation D: cuMemCreate on the host NUMA node, mapped with the VMM API
    {
      CUmemAllocationProp prop = {};
      prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
      prop.location.id = 0;
      size_t gmin = 0, grec = 0;
      cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
      cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
      printf("host-numa granularity min %zu rec %zu\n", gmin, grec);
      CUmemGenericAllocationHandle hnd;
      CUresult r = cuMemCreate(&hnd, total, &prop, 0);
      printf("cuMemCreate host numa: %d\n", (int)r);
      if (r == CUDA_SUCCESS) {
        CUdeviceptr va;
        r = cuMemAddressReserve(&va, total, 2ull << 20, 0, 0);
        r = r ? r : cuMemMap(va, total, 0, hnd, 0);
        CUmemAccessDesc acc[2] = {};
        acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[0].location.id = 0;
        acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
        acc[1].location.id = 0;
        acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CUresult r2 = cuMemSetAccess(va, total, acc, 2);
        if (r2) r2 = cuMemSetAccess(va, total, acc, 1);
        printf("map %d access %d\n", (int)r, (int)r2);
        gpu_write<<<1184, 256, 0, st>>>((uint4*)va, total / 16);
        CK(cudaStreamSynchronize(st));
        for (int sweep = 0; sweep < 2; ++sweep) {
          float tot = 0;
          for (int rg = 0; rg < nregions; ++rg) {
            if (sweep) seq_read<<<1184, 256, 0, st>>>(big, (2ull << 30) / 16, dbuf);
            cudaEventRecord(e0, st);
            slot_gather<<<256, 256, 0, st>>>((const uint4*)((char*)va + rg * region), d_rows + rg * nrows, gout);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            tot += ms;
          }
          tot /= nregions;
          printf("VMM host-numa slot_gather %s device sweep: %.1f us (%.1f GB/s)\n", sweep ? "WITH" : "without",
                 tot * 1e3, (8 << 20) / (tot * 1e-3) / 1e9);
        }
        cudaEventRecord(e0, st);
        seq_read<<<592, 256, 0, st>>>((const uint4*)va, (256 << 20) / 16, dbuf);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("VMM host-numa seq read: %.1f GB/s\n", (256 << 20) / (ms * 1e-3) / 1e9);
        // host access?
        volatile char* hp = (volatile char*)va;
        printf("host read through VA: %d\n", (int)hp[12345]);
      }
    }
    // DMA gather: one cudaMemcpyAsync per row (row-batched copies)
    float tot = 0;
    std::vector<uint32_t> rows0(h_rows.begin(), h_rows.begin() + nrows);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 4096; ++r)
      cudaMemcpyAsync((char*)gout + (size_t)r * 256, (char*)a + (size_t)rows0[r] * 256, 256, cudaMemcpyHostToDevice, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tot, e0, e1);
    printf("DMA per-row memcpy x4096 (1 MiB): %.1f us (%.2f GB/s)\n", tot * 1e3, (1 << 20) / (tot * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}

// tlb_probe.cu -- does the size of the mapped host V arena slow the zero-copy
// recall (GPU page-table walks for sysmem), and does the host allocation
// method (THP mmap + cudaHostRegister, cudaHostAlloc, VMM host-NUMA 2 MB
// granules) change it?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlb_probe tools/tlb_probe.cu -lcuda
//   tools/tlb_probe <arena GiB> <method: reg|alloc|vmm> [sweep 0/1]
// A "layer" window is 2 GiB ([256 rows][32768 pos][256 B]); each gather
// pulls 128 random positions of every row (8 MiB) like recall_pv_kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)
#define CU(x)                                                         \
  do {                                                                \
    CUresult r = (x);                                                 \
    if (r != CUDA_SUCCESS) {                                          \
      const char* s = nullptr;                                        \
      cuGetErrorString(r, &s);                                        \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, s ? s : "?"); \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

constexpr int kRows = 256, kSel = 128, kPos = 32768, kRowB = 256;

__global__ void gather(const uint4* base, const uint32_t* idx, uint32_t* sink) {
  // CTA-looping over rows like recall_pv_kernel: 8 x 16-B loads in flight
  uint32_t acc = 0;
  for (int row = blockIdx.x; row < kRows; row += gridDim.x) {
    const uint4* slot = base + (size_t)row * kPos * (kRowB / 16);
    const uint32_t* id = idx + row * kSel;
    const int total = kSel * (kRowB / 16);
    for (int v0 = threadIdx.x; v0 < total; v0 += blockDim.x * 8) {
      uint4 t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * blockDim.x;
        if (v < total) t[u] = slot[(size_t)id[v >> 4] * (kRowB / 16) + (v & 15)];
        else t[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= t[u].x ^ t[u].w;
    }
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// mode 1: read + discard (L2 left empty); 2: plain read (L2 full of clean
// lines); 3: write (L2 full of dirty lines)
__global__ void sweep(uint4* p, size_t n16, uint32_t* sink, int mode) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    if (mode == 3) {
      p[i] = make_uint4((uint32_t)i, 0, 0, 0);
      continue;
    }
    if (mode == 4) {  // write with an L2 evict_first hint
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p + i),
                   "r"((uint32_t)i), "r"(0), "r"(0), "r"(0), "l"(pol) : "memory");
      continue;
    }
    acc ^= p[i].x;
    if (mode == 1 && (i & 7) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + i) : "memory");
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// scoring-like K stream: CTA i reads chunk i (contiguous) of the 2 GiB region,
// many CTAs in flight at scattered offsets; optional immediate discard
__global__ void chunked(const uint4* p, size_t chunk16, uint32_t* sink, int disc) {
  const uint4* c = p + (size_t)blockIdx.x * chunk16;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < chunk16; i += blockDim.x) {
    acc ^= c[i].x;
    if (disc && (i & 7) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(c + i) : "memory");
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

__global__ void fill(uint4* p, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? atoll(argv[1]) : 16;
  const char* method = argc > 2 ? argv[2] : "reg";
  const int do_sweep = argc > 3 ? atoi(argv[3]) : 1;
  const int ctas = argc > 4 ? atoi(argv[4]) : 32;
  // index pattern: 0 random positions; 1 dense (positions p0..p0+127: 8
  // distinct 4-KB pages per row instead of ~128); 2 one row per 32 KB
  const int pattern = argc > 5 ? atoi(argv[5]) : 0;
  const size_t bytes = gib << 30;
  const size_t window = (size_t)kRows * kPos * kRowB;  // 2 GiB
  const int n_win = (int)(bytes / window);
  CK(cudaSetDevice(0));
  CU(cuInit(0));
  void* dev_ptr = nullptr;
  std::vector<char*> wbase;
  if (!strcmp(method, "managed_split")) {
    // one managed allocation per 2 GiB window (what the product does per layer)
    cudaMemLocation cpu{};
    cpu.type = cudaMemLocationTypeHost;
    cpu.id = 0;
    cudaMemLocation gpu{};
    gpu.type = cudaMemLocationTypeDevice;
    gpu.id = 0;
    for (int w = 0; w < n_win; ++w) {
      void* q = nullptr;
      CK(cudaMallocManaged(&q, window));
      CK(cudaMemAdvise(q, window, cudaMemAdviseSetPreferredLocation, cpu));
      CK(cudaMemAdvise(q, window, cudaMemAdviseSetAccessedBy, gpu));
      madvise(q, window, MADV_HUGEPAGE);
      if (getenv("PROBE_PREFETCH")) {
        CK(cudaMemPrefetchAsync(q, window, cpu, 0));
      } else {
        memset(q, 1, window);
      }
      wbase.push_back((char*)q);
    }
    CK(cudaDeviceSynchronize());
    dev_ptr = wbase[0];
  } else if (!strcmp(method, "reg")) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    madvise(p, bytes, MADV_HUGEPAGE);
    CK(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    CK(cudaHostGetDevicePointer(&dev_ptr, p, 0));
  } else if (!strcmp(method, "huge")) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (p == MAP_FAILED) {
      printf("MAP_HUGETLB failed\n");
      return 1;
    }
    CK(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    CK(cudaHostGetDevicePointer(&dev_ptr, p, 0));
  } else if (!strcmp(method, "managed")) {
    // UVM: host-preferred managed memory the GPU maps remotely (AccessedBy)
    CK(cudaMallocManaged(&dev_ptr, bytes));
    cudaMemLocation cpu{};
    cpu.type = cudaMemLocationTypeHost;
    cpu.id = 0;
    cudaMemLocation gpu{};
    gpu.type = cudaMemLocationTypeDevice;
    gpu.id = 0;
    CK(cudaMemAdvise(dev_ptr, bytes, cudaMemAdviseSetPreferredLocation, cpu));
    CK(cudaMemAdvise(dev_ptr, bytes, cudaMemAdviseSetAccessedBy, gpu));
    madvise(dev_ptr, bytes, MADV_HUGEPAGE);
    if (getenv("PROBE_PREFETCH")) {
      CK(cudaMemPrefetchAsync(dev_ptr, bytes, cpu, 0));  // populate on the host, driver-side
      CK(cudaDeviceSynchronize());
    } else {
      memset(dev_ptr, 1, bytes);  // first touch on the CPU
    }
  } else if (!strcmp(method, "alloc")) {
    void* p = nullptr;
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer(&dev_ptr, p, 0));
  } else {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
    prop.location.id = 0;
    size_t gran = 0;
    CU(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("vmm host granularity %zu\n", gran);
    CUdeviceptr va = 0;
    CU(cuMemAddressReserve(&va, bytes, 1ull << 30, 0, 0));
    const size_t piece = 1ull << 30;
    for (size_t off = 0; off < bytes; off += piece) {
      CUmemGenericAllocationHandle h;
      CU(cuMemCreate(&h, piece, &prop, 0));
      CU(cuMemMap(va + off, piece, 0, h, 0));
      CU(cuMemRelease(h));
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(va, bytes, &acc, 1));
    dev_ptr = (void*)va;
  }
  {
    FILE* f = fopen("/proc/meminfo", "r");
    char line[256];
    while (f && fgets(line, sizeof line, f))
      if (strstr(line, "AnonHugePages") || strstr(line, "HugePages_Total") || strstr(line, "HugePages_Free")) printf("%s", line);
    if (f) fclose(f);
  }
  if (wbase.empty())
    for (int w = 0; w < n_win; ++w) wbase.push_back((char*)dev_ptr + (size_t)w * window);
  {
    cudaEvent_t f0, f1;
    CK(cudaEventCreate(&f0));
    CK(cudaEventCreate(&f1));
    CK(cudaEventRecord(f0));
    for (int w = 0; w < n_win; ++w) fill<<<148 * 4, 256>>>((uint4*)wbase[w], window / 16);
    CK(cudaEventRecord(f1));
    CK(cudaDeviceSynchronize());
    float fms = 0;
    CK(cudaEventElapsedTime(&fms, f0, f1));
    printf("GPU fill of the arena: %.1f ms (%.1f GB/s)\n", fms, bytes / (fms * 1e-3) / 1e9);
  }

  std::mt19937 rng(7);
  std::vector<uint32_t> hidx((size_t)n_win * kRows * kSel);
  for (int w = 0; w < n_win; ++w)
    for (int r = 0; r < kRows; ++r) {
      std::vector<uint32_t> sel;
      const uint32_t p0 = rng() % (kPos - 128 * kSel);
      while ((int)sel.size() < kSel) {
        const uint32_t k = (uint32_t)sel.size();
        sel.push_back(pattern == 0 ? rng() % kPos : pattern == 1 ? p0 + k : p0 + 128 * k);
      }
      std::sort(sel.begin(), sel.end());
      memcpy(&hidx[((size_t)w * kRows + r) * kSel], sel.data(), kSel * 4);
    }
  uint32_t* didx;
  CK(cudaMalloc(&didx, hidx.size() * 4));
  CK(cudaMemcpy(didx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice));
  // mode 4/5: rotate the 2 GiB read+discard sweep over a larger device buffer
  // (like the scoring kernel streaming a different layer's K each time)
  const size_t sw_total = (do_sweep == 4 || do_sweep >= 10) ? (64ull << 30) : do_sweep == 5 ? (16ull << 30) : (2ull << 30);
  const size_t sw_bytes = 2ull << 30;
  uint4* sw;
  uint32_t* sink;
  CK(cudaMalloc(&sw, sw_total));
  CK(cudaMemset(sw, 0, sw_total));
  size_t sw_off = 0;
  CK(cudaMalloc(&sink, 64));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int rep = 0; rep < 3; ++rep) {
    double tot = 0;
    for (int w = 0; w < n_win; ++w) {
      if (do_sweep == 10 || do_sweep == 11) {
        const int nch = 6912;
        chunked<<<nch, 256>>>(sw + sw_off / 16, sw_bytes / 16 / nch, sink, do_sweep == 10);
        sw_off = (sw_off + sw_bytes) % sw_total;
      } else if (do_sweep >= 6) {
        // logits-like: 2 GiB read+discard (K), then write `lg` MiB (dirty
        // logits), then read + discard them (selection)
        const size_t lg = (size_t)(do_sweep == 6 || do_sweep == 9 ? 32 : do_sweep == 7 ? 16 : 8) << 20;
        sweep<<<148 * 4, 256>>>(sw, sw_bytes / 16, sink, 1);
        sweep<<<148 * 4, 256>>>(sw + (1ull << 30) / 16, lg / 16, sink, do_sweep == 9 ? 4 : 3);
        sweep<<<148 * 4, 256>>>(sw + (1ull << 30) / 16, lg / 16, sink, 1);
      } else if (do_sweep) {
        sweep<<<148 * 4, 256>>>(sw + sw_off / 16, sw_bytes / 16, sink, do_sweep == 4 || do_sweep == 5 ? 1 : do_sweep);
        sw_off = (sw_off + sw_bytes) % sw_total;
      }
      CK(cudaEventRecord(a));
      gather<<<ctas, 256>>>((const uint4*)wbase[w], didx + (size_t)w * kRows * kSel, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      tot += ms;
    }
    const double us = tot / n_win * 1e3;
    if (rep < 2) continue;
    printf("pattern %d arena %zu GiB %s sweep=%d ctas=%d rep %d: gather %.1f us/window (%.1f GB/s)\n", pattern, gib, method, do_sweep,
           ctas, rep, us, (double)kRows * kSel * kRowB / (us * 1e-6) / 1e9);
  }
  if (!strcmp(method, "managed") || !strcmp(method, "reg") || !strcmp(method, "managed_split")) {
    // host-side check of what the GPU wrote (managed: no migration expected)
    const uint4* hp = (const uint4*)dev_ptr;
    size_t bad = 0;
    for (size_t i = 0; i < window / 16; i += 1000003) bad += hp[i].x != (uint32_t)i || hp[i].y != 1;
    printf("host check: %zu mismatches\n", bad);
  }
  return 0;
}

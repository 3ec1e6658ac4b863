// Development probe (not product code): hold k whole SMs with spinning CTAs
// (one 1024-thread CTA per SM, 200 KB of shared memory so nothing else fits
// beside it) to measure how the scoring kernel's bandwidth depends on the
// number of SMs it can use -- the feasibility question behind the SM
// partitioning plan in DESIGN.md section 9.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o tools/libsm_blocker.so tools/sm_blocker.cu
#include <cuda_runtime.h>
#include <cstdint>

__global__ void blocker_kernel(volatile uint32_t* flag) {
  extern __shared__ uint8_t smem[];
  if (threadIdx.x == 0) {
    smem[0] = 1;
    while (*flag == 0u) __nanosleep(2000);
  }
  __syncthreads();
}

extern "C" {
// launches `ctas` blocking CTAs on `stream`; they exit once *flag != 0
int sm_blocker_launch(int ctas, uint32_t* flag, void* stream) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(blocker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  blocker_kernel<<<ctas, 1024, smem, (cudaStream_t)stream>>>(flag);
  return (int)cudaGetLastError();
}
}

// kc_device.cuh -- device helpers shared by the sm_100a kernels: element
// conversion, 128-bit unpacking, and the mbarrier / TMA bulk-copy PTX used by
// the K streaming pipeline.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace kc {

// ---- element conversion ----------------------------------------------------
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// 16 bytes of 16-bit elements -> 8 floats (exact widening).
template <typename T>
__device__ __forceinline__ void unpack8(const uint4& raw, float (&f)[8]);
template <>
__device__ __forceinline__ void unpack8<__half>(const uint4& raw, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void unpack8<__nv_bfloat16>(const uint4& raw, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Packed fp32 FMA (sm_100 FFMA2): (a.x*b.x + c.x, a.y*b.y + c.y), each
// lane rounded like fmaf.
__device__ __forceinline__ float2 ffma2(float a0, float a1, float b0, float b1, float2 c) {
  float2 d;
  asm("{ .reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
      "mov.b64 {%0, %1}, rd; }"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c.x), "f"(c.y));
  return d;
}

// ---- softmax partial-stat combine (m = running max, l = sum exp(s - m)) ----
__device__ __forceinline__ void ml_combine(float& m, float& l, float m2, float l2) {
  const float M = fmaxf(m, m2);
  if (M == -INFINITY) {
    m = M;
    l = 0.0f;
    return;
  }
  const float a = (m == -INFINITY) ? 0.0f : l * expf(m - M);
  const float b = (m2 == -INFINITY) ? 0.0f : l2 * expf(m2 - M);
  m = M;
  l = a + b;
}

// Global softmax stats of one (batch, q head) from the scoring kernel's
// per-split (max, sum exp): M = max m_i, Z = sum_i l_i exp(m_i - M). Called
// by a full warp; every kernel that needs p = exp(s - M) / Z uses this one
// function, so selection, weights and the observer path agree bit for bit.
// CG: read through L2 only (partials written by other CTAs of the running
// kernel: the fused selection in kc_rowsel.cuh).
template <bool CG = false>
__device__ __forceinline__ void softmax_stats(const float2* part, int n_splits, int lane, float& M,
                                              float& Z) {
  auto ld = [&](int i) { return CG ? __ldcg(part + i) : part[i]; };
  float m = -INFINITY;
  for (int i = lane; i < n_splits; i += 32) m = fmaxf(m, ld(i).x);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float z = 0.0f;
  for (int i = lane; i < n_splits; i += 32) {
    const float2 ml = ld(i);
    if (ml.y > 0.0f) z += ml.y * expf(ml.x - m);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  M = m;
  Z = z;
}

// ---- shared-memory address / mbarrier / TMA bulk copy (PTX) ----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// L2 policy for data streamed exactly once (K during scoring).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Other L2 policies for the K stream (tuning experiments).
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t pol;
  switch (kind) {
    case 1: asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol)); break;
    case 2: asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol)); break;
    case 3: asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol)); break;
    case 4: asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 0.5;" : "=l"(pol)); break;
    default: asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol)); break;
  }
  return pol;
}

// 1-D TMA bulk copy global -> shared, completion signalled on `bar` as
// transaction bytes (SASS: UBLKCP). bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void tma_bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                             uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Invalidate one 128-B L2 line without write-back (PTX: a weak write of an
// indeterminate value). Used only on dead scratch -- logits whose row has been
// selected and that are overwritten before they are read again -- never on
// K/V cache data.
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// 16-B read-only load that marks its L2 line evict-first (V rows read once per
// decode step: the recall's lines should be the first to leave L2, without
// dropping anything).
__device__ __forceinline__ uint4 ld_stream16(const void* p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- GQA tensor-core scoring: q in NP parts of the MMA input type ------------
// (score_mma_kernel, score_tc_kernel). fp16: q * 2^e = hi + lo (2^e puts the
// head's max |q| at 2^14, both parts normal); bf16: three parts.
// q split into NP parts of T; returns the scale to undo (2^-e for fp16)
template <typename T>
struct QSplit;
template <>
struct QSplit<__half> {
  static constexpr int NP = 2;
  __device__ static float prescale(float amax) {
    if (!(amax > 0.0f) || !isfinite(amax)) return 1.0f;
    return ldexpf(1.0f, 14 - ilogbf(amax));
  }
  __device__ static uint32_t pack(float x, float y) {
    const __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  __device__ static float2 unpack(uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
};
template <>
struct QSplit<__nv_bfloat16> {
  static constexpr int NP = 3;
  __device__ static float prescale(float) { return 1.0f; }
  __device__ static uint32_t pack(float x, float y) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  __device__ static float2 unpack(uint32_t w) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  }
};


// named barrier over `n` threads (bar.sync id, n)
__device__ __forceinline__ void named_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- selection keys (kc_select.cu) -------------------------------------------
// Order-preserving bits of a float; -0.0 and +0.0 compare equal, so they must
// tie (one key).
__device__ __forceinline__ uint32_t ordered_bits(float x) {
  const uint32_t u = x == 0.0f ? 0u : __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float from_ordered(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// The p-tie window around a score Ts: outside it p = expf(s - M)/Z differs
// from p(Ts) strictly, provided p(Ts) is a normal float (see
// score_fast_kernel's candidate bound).
__device__ __forceinline__ float tie_window(float Ts, float M) {
  return 4e-5f * (1.0f + fabsf(Ts) + fabsf(M));
}

}  // namespace kc

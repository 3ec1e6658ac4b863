// kc_prefill.cu -- causal prefill attention (the reference's
// prefill_attention, proj/core/src/attention.cpp:31-62), called by
// Engine::prefill once per sequence and layer (engine.cpp:106).
//
// Not on the decode hot path; what matters here is that it is the
// reference's arithmetic: per (head, query i) the scores s_j = dot(q_i, k_j)
// * scale for j <= i with the dot summed in ascending element order
// (separately rounded multiply and add, as -ffp-contract=off compiles
// `acc += a[i]*b[i]`), softmax_inplace's max / ordered sum of exp(s - max) /
// division (matrix.cpp:45-61), and out += p_j * v_j in ascending j. A CTA
// owns a tile of 32 queries of one head and streams 32-key tiles of K and V
// through shared memory three times (max, sum, weighted sum) instead of
// materialising the s x s score matrix.
#include <algorithm>
#include <cfloat>

#include "kc_device.cuh"
#include "kc_kernels.cuh"

namespace kc {

namespace {

constexpr int kTq = 32;   // queries per CTA
constexpr int kTk = 32;   // keys per shared-memory tile
constexpr int kPT = 256;  // threads per CTA

__global__ void __launch_bounds__(kPT) prefill_attn_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                          const float* __restrict__ v, float* __restrict__ out,
                                                          int s, int d, int h, float scale) {
  extern __shared__ float sm[];
  const int hp = h + 1;  // padded rows: lanes reading different keys hit different banks
  float* Qs = sm;                     // [kTq][hp]
  float* Ks = Qs + kTq * hp;          // [kTk][hp]
  float* Vs = Ks + kTk * hp;          // [kTk][h]
  float* S = Vs + kTk * h;            // [kTq][kTk + 1]
  float* Mx = S + kTq * (kTk + 1);    // [kTq]
  float* Zs = Mx + kTq;               // [kTq]
  float* Acc = Zs + kTq;              // [kTq][h]
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTq;
  const int off = blockIdx.y * h;
  const int nq = min(kTq, s - q0);
  const int n_tiles = (q0 + nq - 1) / kTk + 1;  // keys 0 .. q0+nq-1

  for (int e = tid; e < kTq * h; e += kPT) {
    const int qi = e / h, t = e - qi * h;
    Qs[qi * hp + t] = qi < nq ? q[(size_t)(q0 + qi) * d + off + t] : 0.0f;
    Acc[e] = 0.0f;
  }
  if (tid < kTq) {
    Mx[tid] = -FLT_MAX;
    Zs[tid] = 0.0f;
  }

  // scores of key tile kt into S (causal: key j > query i -> not used)
  auto score_tile = [&](int kt) {
    const int j0 = kt * kTk;
    __syncthreads();  // previous users of Ks / S are done
    for (int e = tid; e < kTk * h; e += kPT) {
      const int kj = e / h, t = e - kj * h;
      const int j = j0 + kj;
      Ks[kj * hp + t] = j < s ? k[(size_t)j * d + off + t] : 0.0f;
    }
    __syncthreads();
    for (int e = tid; e < kTq * kTk; e += kPT) {
      const int qi = e / kTk, kj = e - qi * kTk;
      const float* a = Qs + qi * hp;
      const float* b = Ks + kj * hp;
      float acc = 0.0f;
      for (int t = 0; t < h; ++t) acc = __fadd_rn(acc, __fmul_rn(a[t], b[t]));
      S[qi * (kTk + 1) + kj] = __fmul_rn(acc, scale);  // dot_scaled: multiply after the sum
    }
    __syncthreads();
  };
  auto n_valid = [&](int qi, int kt) {  // keys of tile kt that query qi sees
    return max(0, min(kTk, q0 + qi + 1 - kt * kTk));
  };

  // pass 1: row max
  for (int kt = 0; kt < n_tiles; ++kt) {
    score_tile(kt);
    if (tid < nq) {
      float m = Mx[tid];
      const int nv = n_valid(tid, kt);
      for (int kj = 0; kj < nv; ++kj) m = fmaxf(m, S[tid * (kTk + 1) + kj]);
      Mx[tid] = m;
    }
  }
  // pass 2: sum of exp(s - max) in ascending key order
  for (int kt = 0; kt < n_tiles; ++kt) {
    score_tile(kt);
    if (tid < nq) {
      float z = Zs[tid];
      const float m = Mx[tid];
      const int nv = n_valid(tid, kt);
      for (int kj = 0; kj < nv; ++kj) z = __fadd_rn(z, expf(S[tid * (kTk + 1) + kj] - m));
      Zs[tid] = z;
    }
  }
  // pass 3: out += (exp(s - max) / sum) * v, ascending key order
  for (int kt = 0; kt < n_tiles; ++kt) {
    score_tile(kt);
    const int j0 = kt * kTk;
    for (int e = tid; e < kTq * kTk; e += kPT) {
      const int qi = e / kTk, kj = e - qi * kTk;
      float& sv = S[qi * (kTk + 1) + kj];
      sv = qi < nq ? __fdiv_rn(expf(sv - Mx[qi]), Zs[qi]) : 0.0f;
    }
    for (int e = tid; e < kTk * h; e += kPT) {
      const int kj = e / h, t = e - kj * h;
      const int j = j0 + kj;
      Vs[e] = j < s ? v[(size_t)j * d + off + t] : 0.0f;
    }
    __syncthreads();
    for (int e = tid; e < nq * h; e += kPT) {
      const int qi = e / h, c = e - qi * h;
      const int nv = n_valid(qi, kt);
      const float* p = S + qi * (kTk + 1);
      float a = Acc[e];
      for (int kj = 0; kj < nv; ++kj) a = __fadd_rn(a, __fmul_rn(p[kj], Vs[kj * h + c]));
      Acc[e] = a;
    }
  }
  __syncthreads();
  for (int e = tid; e < nq * h; e += kPT) {
    const int qi = e / h, c = e - qi * h;
    out[(size_t)(q0 + qi) * d + off + c] = Acc[e];
  }
}

}  // namespace

size_t prefill_smem_bytes(int h) {
  const int hp = h + 1;
  return sizeof(float) * ((size_t)kTq * hp + (size_t)kTk * hp + (size_t)kTk * h + (size_t)kTq * (kTk + 1) +
                          2 * kTq + (size_t)kTq * h);
}

bool prefill_attention_launch(const float* q, const float* k, const float* v, float* out, int s, int n_heads,
                              int h, cudaStream_t st) {
  const size_t smem = prefill_smem_bytes(h);
  if (smem > 200 * 1024) return false;
  if (cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return false;
  const dim3 grid((unsigned)((s + kTq - 1) / kTq), (unsigned)n_heads);
  prefill_attn_kernel<<<grid, kPT, smem, st>>>(q, k, v, out, s, n_heads * h, h,
                                               1.0f / sqrtf(static_cast<float>(h)));
  return true;
}

}  // namespace kc

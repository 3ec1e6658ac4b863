/*
 * kcache_oracle.c -- TEST INFRASTRUCTURE ONLY (see kcache_oracle.h).
 *
 * CPU restatement of the reference decode-step TopN attention. Every function
 * names the reference file:line it follows. Build: oracle/Makefile
 * (-O2 -ffp-contract=off, like proj/CMakeLists.txt:11-13).
 */
#include "kcache_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* SplitMix64, proj/core/include/kcache/rng.hpp:13-19. The generator adds the
 * golden-ratio increment before mixing, so draw i sees state seed+(i+1)*inc. */
static uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* next_double / next_uniform, rng.hpp:22-26. */
float kco_uniform(uint64_t seed, uint64_t i, float lo, float hi) {
  double u = (double)(splitmix_at(seed, i) >> 11) * 0x1.0p-53;
  float f = (float)u;
  float span = hi - lo;
  float t = f * span;
  return lo + t;
}

float kco_round_f16(float x) { return (float)(_Float16)x; }

float kco_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate, keep nan quiet */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    u &= 0xffff0000u;
  }
  float r;
  memcpy(&r, &u, 4);
  return r;
}

void kco_fill_uniform(float* dst, uint64_t n, uint64_t seed, uint64_t offset, float lo, float hi,
                      int round_dtype) {
  for (uint64_t i = 0; i < n; ++i) {
    float x = kco_uniform(seed, offset + i, lo, hi);
    if (round_dtype == 1) x = kco_round_f16(x);
    else if (round_dtype == 2) x = kco_round_bf16(x);
    dst[i] = x;
  }
}

/* softmax_inplace, proj/core/src/matrix.cpp:45-61. std::max(mx, v) keeps mx
 * unless mx < v. */
void kco_softmax_inplace(float* row, size_t n) {
  if (n == 0) return;
  float mx = row[0];
  for (size_t i = 0; i < n; ++i) {
    if (mx < row[i]) mx = row[i];
  }
  float sum = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    row[i] = expf(row[i] - mx);
    sum += row[i];
  }
  for (size_t i = 0; i < n; ++i) row[i] /= sum;
}

/* Stable merge sort of index array by descending value: an element from the
 * right run is taken first only when its value is strictly greater, which is
 * what std::stable_sort with `values[a] > values[b]` produces
 * (proj/core/src/matrix.cpp:116-117). */
static void merge_desc(const float* values, uint32_t* a, uint32_t* tmp, size_t n) {
  if (n < 2) return;
  size_t mid = n / 2;
  merge_desc(values, a, tmp, mid);
  merge_desc(values, a + mid, tmp, n - mid);
  size_t i = 0, j = mid, o = 0;
  while (i < mid && j < n) {
    if (values[a[j]] > values[a[i]]) tmp[o++] = a[j++];
    else tmp[o++] = a[i++];
  }
  while (i < mid) tmp[o++] = a[i++];
  while (j < n) tmp[o++] = a[j++];
  memcpy(a, tmp, n * sizeof(uint32_t));
}

static int cmp_u32(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return (a > b) - (a < b);
}

/* arg_topk, proj/core/src/matrix.cpp:109-122. */
size_t kco_arg_topk(const float* values, size_t n, size_t k, uint32_t* out) {
  if (k == 0) return (size_t)-1;
  uint32_t* idx = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t* tmp = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  merge_desc(values, idx, tmp, n);
  size_t m = k < n ? k : n;
  qsort(idx, m, sizeof(uint32_t), cmp_u32);
  memcpy(out, idx, m * sizeof(uint32_t));
  free(idx);
  free(tmp);
  return m;
}

/* attention_score_scale, proj/core/include/kcache/attention.hpp:15-17. */
static float score_scale(size_t h) { return 1.0f / sqrtf((float)h); }

/* dot_scaled, proj/core/src/attention.cpp:15-21: sequential fp32 sum, scale
 * applied after the sum. */
static float dot_scaled(const float* a, const float* b, size_t n, float scale) {
  float acc = 0.0f;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc * scale;
}

/* head_weights, proj/core/src/attention.cpp:66-78, over a contiguous slot. */
void kco_head_weights(size_t h, size_t s, const float* qhead, const float* kslot, float* probs) {
  float scale = score_scale(h);
  for (size_t j = 0; j < s; ++j) probs[j] = dot_scaled(qhead, kslot + j * h, h, scale);
  kco_softmax_inplace(probs, s);
}

/* Strided variant over the position-major cache layout. */
static void head_weights_strided(size_t h, size_t s, const float* qhead, const float* kbase,
                                 size_t row_stride, float* probs) {
  float scale = score_scale(h);
  for (size_t j = 0; j < s; ++j) probs[j] = dot_scaled(qhead, kbase + j * row_stride, h, scale);
  kco_softmax_inplace(probs, s);
}

/* One (batch, kv head) group: selection + gather + P.V
 * (proj/core/src/attention.cpp:134-188; gather_v kv_cache.cpp:150-187).
 * probs: [G][s] softmax rows. vbase/vstride address the slot's V rows. */
static void group_select_pv(size_t G, size_t h, size_t s, float* probs, const float* vbase,
                            size_t vstride, size_t top_n, int renormalize, int ordered,
                            float* out /*[G][h], stride out_stride*/, size_t out_stride,
                            uint32_t* idx /*[nc], written once*/, float* w /*[G][nc]*/,
                            size_t w_stride, double* dropped /*[G]*/, size_t dropped_stride) {
  size_t nc = top_n < s ? top_n : s;
  const float* key = probs;
  float* gsum = NULL;
  if (G > 1) {
    gsum = (float*)malloc(s * sizeof(float));
    for (size_t j = 0; j < s; ++j) {
      float acc = probs[j];
      for (size_t g = 1; g < G; ++g) acc += probs[g * s + j];
      gsum[j] = acc;
    }
    key = gsum;
  }
  kco_arg_topk(key, s, top_n, idx);
  for (size_t g = 0; g < G; ++g) {
    const float* p = probs + g * s;
    float* wg = w + g * w_stride;
    double mass = 0.0;
    for (size_t r = 0; r < nc; ++r) {
      wg[r] = p[idx[r]];
      mass += (double)wg[r];
    }
    dropped[g * dropped_stride] = 1.0 - mass;
    float norm = 1.0f;
    if (renormalize) {
      float sum = 0.0f;
      for (size_t r = 0; r < nc; ++r) sum += wg[r];
      norm = sum > 0.0f ? 1.0f / sum : 1.0f;
    }
    float* dst = out + g * out_stride;
    for (size_t c = 0; c < h; ++c) dst[c] = 0.0f;
    for (size_t t = 0; t < nc; ++t) {
      size_t r = ordered ? t : nc - 1 - t;
      float wr = renormalize ? wg[r] * norm : wg[r];
      const float* vrow = vbase + (size_t)idx[r] * vstride;
      for (size_t c = 0; c < h; ++c) dst[c] += wr * vrow[c]; /* add_scaled, attention.cpp:23-27 */
    }
  }
  free(gsum);
}

int kco_decode_topn(size_t batch, size_t n_heads, size_t n_kv_heads, size_t h, size_t s,
                    const float* q, const float* k, const float* v, size_t top_n, int renormalize,
                    int ordered, float* out, uint32_t* idx, float* w, double* dropped) {
  if (top_n == 0 || s == 0 || n_kv_heads == 0 || n_heads % n_kv_heads != 0) return -1;
  size_t G = n_heads / n_kv_heads;
  size_t d = n_heads * h, dkv = n_kv_heads * h;
  size_t nc = top_n < s ? top_n : s;
  float* probs = (float*)malloc(G * s * sizeof(float));
  uint32_t* gidx = (uint32_t*)malloc(nc * sizeof(uint32_t));
  for (size_t b = 0; b < batch; ++b) {
    for (size_t kvh = 0; kvh < n_kv_heads; ++kvh) {
      for (size_t g = 0; g < G; ++g) {
        size_t head = kvh * G + g;
        head_weights_strided(h, s, q + b * d + head * h, k + b * dkv + kvh * h, batch * dkv,
                             probs + g * s);
      }
      size_t slot0 = b * n_heads + kvh * G;
      group_select_pv(G, h, s, probs, v + b * dkv + kvh * h, batch * dkv, top_n, renormalize,
                      ordered, out + b * d + kvh * G * h, h, gidx, w + slot0 * nc, nc,
                      dropped + slot0, 1);
      for (size_t g = 0; g < G; ++g) memcpy(idx + (slot0 + g) * nc, gidx, nc * sizeof(uint32_t));
    }
  }
  free(probs);
  free(gidx);
  return 0;
}

int kco_decode_topn_group(size_t G, size_t h, size_t s, const float* q_group, const float* kslot,
                          const float* vslot, size_t top_n, int renormalize, int ordered,
                          float* out, uint32_t* idx, float* w, double* dropped) {
  if (top_n == 0 || s == 0 || G == 0) return -1;
  size_t nc = top_n < s ? top_n : s;
  float* probs = (float*)malloc(G * s * sizeof(float));
  for (size_t g = 0; g < G; ++g) kco_head_weights(h, s, q_group + g * h, kslot, probs + g * s);
  group_select_pv(G, h, s, probs, vslot, h, top_n, renormalize, ordered, out, h, idx, w, nc,
                  dropped, 1);
  free(probs);
  return 0;
}

/* decode_attention_full, proj/core/src/attention.cpp:91-114. */
int kco_decode_full(size_t batch, size_t n_heads, size_t n_kv_heads, size_t h, size_t s,
                    const float* q, const float* k, const float* v, float* out) {
  if (s == 0 || n_kv_heads == 0 || n_heads % n_kv_heads != 0) return -1;
  size_t G = n_heads / n_kv_heads;
  size_t d = n_heads * h, dkv = n_kv_heads * h;
  float* probs = (float*)malloc(s * sizeof(float));
  for (size_t b = 0; b < batch; ++b) {
    for (size_t head = 0; head < n_heads; ++head) {
      size_t kvh = head / G;
      head_weights_strided(h, s, q + b * d + head * h, k + b * dkv + kvh * h, batch * dkv, probs);
      float* dst = out + b * d + head * h;
      for (size_t c = 0; c < h; ++c) dst[c] = 0.0f;
      for (size_t j = 0; j < s; ++j) {
        const float* vrow = v + (j * batch + b) * dkv + kvh * h;
        for (size_t c = 0; c < h; ++c) dst[c] += probs[j] * vrow[c];
      }
    }
  }
  free(probs);
  return 0;
}

/*
 * kcache_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's decode-step TopN attention
 * (arXiv 2404.18057 reference, /root/reference/proj). It is the parity
 * checker for the CUDA path and the "port" CPU baseline; nothing in the
 * product (paper_2404_18057_b200/, include/) links or calls it. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself (oracle/_ref, built
 * from the reference sources by oracle/Makefile; fixtures in tests/golden/,
 * generator tests/golden/make_golden.py) and against the reference's own
 * known-answer tests (proj/tests/test_attention.cpp:153-178,
 * proj/tests/test_matrix.cpp:123-159, proj/tests/test_kv_cache.cpp:114-131).
 *
 * Compiled with -ffp-contract=off, as the reference is
 * (proj/CMakeLists.txt:11-13): fp32 accumulation order is part of the
 * contract.
 */
#ifndef KCACHE_ORACLE_H
#define KCACHE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Element i (0-based) of the SplitMix64 stream seeded with `seed`, mapped to
 * [lo, hi) exactly as SeededRng::next_uniform
 * (proj/core/include/kcache/rng.hpp:13-30). Counter-indexed, so any element
 * can be produced without generating its predecessors. */
float kco_uniform(uint64_t seed, uint64_t i, float lo, float hi);

/* Fill dst[0..n) with elements [offset, offset+n) of the stream, then round
 * each to the storage dtype (0 = keep fp32, 1 = fp16 RNE, 2 = bf16 RNE). */
void kco_fill_uniform(float* dst, uint64_t n, uint64_t seed, uint64_t offset, float lo, float hi,
                      int round_dtype);

float kco_round_f16(float x);
float kco_round_bf16(float x);

/* softmax_inplace (proj/core/src/matrix.cpp:45-61): max, exp(v - max) with a
 * sequential fp32 sum, then divide. */
void kco_softmax_inplace(float* row, size_t n);

/* arg_topk (proj/core/src/matrix.cpp:109-122): indices of the k largest
 * values, ties to the lowest index, returned ascending. Returns the count
 * min(k, n); returns (size_t)-1 when k == 0 (the reference throws
 * std::invalid_argument). */
size_t kco_arg_topk(const float* values, size_t n, size_t k, uint32_t* out);

/* decode_attention_topn (proj/core/src/attention.cpp:116-190) over one
 * layer's cache.
 *   q        [batch][n_heads*h]           fp32
 *   k, v     [s][batch][n_kv_heads*h]     fp32, position-major like
 *                                         TieredKVCache (kv_cache.cpp:189-197)
 * MHA (n_kv_heads == n_heads) reproduces the reference exactly. GQA
 * (n_heads = G*n_kv_heads) uses the repository's stated extension
 * (DESIGN.md "GQA selection rule"): each q head has its own softmax; the
 * selection key per (batch, kv head) is sum_g p_g[j] in ascending g (fp32);
 * every q head of the group uses the shared indices with its own p.
 * Outputs, slot = b*n_heads + head:
 *   out      [batch][n_heads*h]
 *   idx      [slot][nc]  nc = min(top_n, s), ascending
 *   w        [slot][nc]  raw softmax values at idx
 *   dropped  [slot]      1 - sum(double(w))
 * ordered = 0 is the reference's fault hook (descending accumulation,
 * attention.cpp:180-186). Returns 0, or -1 for top_n == 0 / s == 0 /
 * bad head split (the reference throws). */
int kco_decode_topn(size_t batch, size_t n_heads, size_t n_kv_heads, size_t h, size_t s,
                    const float* q, const float* k, const float* v, size_t top_n, int renormalize,
                    int ordered, float* out, uint32_t* idx, float* w, double* dropped);

/* decode_attention_full (proj/core/src/attention.cpp:91-114). */
int kco_decode_full(size_t batch, size_t n_heads, size_t n_kv_heads, size_t h, size_t s,
                    const float* q, const float* k, const float* v, float* out);

/* Single slot variant used for sampled parity at full size: kslot/vslot are
 * the s rows of one (batch, kv head), each h wide, contiguous. q_group holds
 * the G query heads of that kv head ([G][h]). Outputs for the G q heads:
 * out [G][h], idx [nc] (shared), w [G][nc], dropped [G]. */
int kco_decode_topn_group(size_t G, size_t h, size_t s, const float* q_group, const float* kslot,
                          const float* vslot, size_t top_n, int renormalize, int ordered,
                          float* out, uint32_t* idx, float* w, double* dropped);

/* Full scores/softmax of one q head against one kv slot (head_weights,
 * proj/core/src/attention.cpp:66-78): probs[s]. */
void kco_head_weights(size_t h, size_t s, const float* qhead, const float* kslot, float* probs);

#ifdef __cplusplus
}
#endif

#endif

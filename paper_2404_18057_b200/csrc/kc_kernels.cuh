// kc_kernels.cuh -- launch interfaces of the sm_100a kernels (host side).
//
// One decode_attention_topn call (proj/core/src/attention.cpp:116-190) is
//   score_launch    q.K^T over every cached position + per-split (max, sum exp)
//   select_launch   global softmax stats, top-N radix select, weights, dropped
//   recall_launch   V recall of the selected rows (HBM or mapped host) + P.V
// decode_attention_full (attention.cpp:91-114) is score_launch + pv_full_launch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kc {

struct ScoreParams {
  const void* k;        // layer's K: [rows][max_seq][h], rows = batch*n_kv
  const float* q;       // [batch][n_q][h] fp32
  float* logits;        // [batch][n_q][lstride]
  float2* partials;     // [batch][n_q][max_splits]  (max, sum exp)
  int64_t max_seq;      // K slot stride in positions
  int64_t lstride;      // logits row stride
  int s;                // current length
  int h;                // head_dim
  int n_kv;
  int G;                // q heads per kv head
  int rows;             // batch*n_kv
  int chunk;            // positions per CTA (multiple of 64)
  int n_splits;
  int max_splits;
  float scale;          // 1/sqrt(h) as the reference computes it
  int stages;           // TMA ring depth (4, 6 or 8 stages of 64 positions)
  int row0;             // first row of this launch (row groups); rows = rows in this launch
  // candidate mode (MHA, h=128 16-bit fast path, cand_nc > 0): instead of the
  // dense logits, every split writes the positions that can still be in the
  // row's top-cand_nc -- a provable superset, see kc_score.cu -- as (score
  // bits, position) pairs at cand[row][pos0..], plus {count, exclusion bound}
  // at cand_meta[row][split]. Positions with score < bound were dropped.
  uint2* cand;          // [rows][lstride]
  uint2* cand_meta;     // [rows][max_splits]
  int cand_nc;          // 0: dense logits
  int k_policy;         // L2 policy of the K stream (0 evict_first; see l2_policy)
  int use_mma;          // GQA (2 <= G <= 8): tensor-core scoring (score_mma_kernel)
  int tlb_ahead;        // rows ahead whose K translations the producer warms (0: off)
  // dataflow (consume_launch): every CTA bumps row_done[row] (release) once
  // its split's logits and statistics are written; null: no signalling
  uint32_t* row_done;
  // score_tc_kernel: the layer's K tensor map (CUtensorMap, host memory; see
  // encode_k_map), or null
  const void* kmap;
  // score_tc_kernel: CTAs in the launch (0: one per item; otherwise a
  // persistent grid walking items blockIdx.x, +gridDim.x, ...)
  int grid;
};
// one-thread marker kernel (increments *word)
void join_mark_launch(uint32_t* word, cudaStream_t st);
// test hook: one thread sleeping ~ns nanoseconds on the stream
void spin_launch(uint64_t ns, cudaStream_t st);
// row_done counters: one per kRowDoneStride words (a 128-B line per row)
constexpr int kRowDoneStride = 32;
// dtype: KC_F32 / KC_F16 / KC_BF16 (storage)
void score_launch(const ScoreParams& p, int dtype, cudaStream_t st);
// positions per CTA for a given shape (tuning override when > 0)
int score_pick_chunk(int s, int rows, int override_chunk, int G = 1);
// SMs of the current device
int sm_count();
// GQA scoring on tcgen05 (kc_score_tc.cu): shapes it covers, the K tensor map
// of one layer ([rows][max_seq][128] 16-bit, 64 x 128 SW128 boxes) written to
// map_out (128 B, 64-B aligned), and the launch (false: not covered)
bool score_tc_supported(int dtype, int h, int G);
bool encode_k_map(void* map_out, const void* k_layer, int dtype, uint64_t rows, uint64_t max_seq);
bool score_tc_launch(const ScoreParams& p, int dtype, cudaStream_t st);
// whether the candidate-mode scoring kernel covers this shape
bool score_cand_supported(int dtype, int h, int G, int chunk, int nc);

struct SelectParams {
  const float* logits;    // [batch][n_q][lstride]
  const float2* partials; // [batch][n_q][max_splits]
  uint32_t* keys;         // scratch [rows][kstride]
  uint32_t* idx;          // [rows][nc]
  float* w;               // [batch*n_q][nc]
  double* dropped;        // [batch*n_q]
  float* norm;            // [batch*n_q]  1/sum(w) for renormalize (1 if sum == 0)
  int64_t lstride;
  int64_t kstride;
  int s;
  int nc;                 // min(top_n, s)
  int n_kv;
  int G;
  int n_splits;
  int max_splits;
  int rows;
  int force_global;       // 1: the global-memory-keys kernel even when s fits registers
  int row0;               // first row of this launch (row groups); rows = rows in this launch
  // candidate mode (ScoreParams::cand_nc): select from the scoring kernel's
  // per-split candidates; rows whose candidate set cannot be proven complete
  // are flagged in fb_flags and redone densely by select_fallback_launch,
  // which recomputes the row's scores bit-identically from q and K.
  const uint2* cand;      // [rows][lstride]
  const uint2* cand_meta; // [rows][max_splits] {count, bound bits}
  uint32_t* fb_flags;     // [rows]
  int chunk;              // scoring split length (candidate slots start at split*chunk)
  const void* k;          // layer's K [rows][max_seq][h] (fallback recompute)
  const float* q;         // [batch][n_q][h] fp32
  int64_t max_seq;
  int h;
  int kdtype;             // KC_F16 / KC_BF16
  float scale;
  int force_fallback;     // test hook: flag every row for the dense redo
  int keep_logits;        // 1: leave the dead logits in L2 (no discard.global.L2)
};
void select_launch(const SelectParams& p, cudaStream_t st);
// longest row the dense selection keeps in registers (select_reg_kernel)
constexpr int kDenseRegMaxS = 32 * 1024;
// candidate-mode selection (MHA, fast scoring path) + the dense redo of any
// row it flags; returns false when the shape is outside candidate mode
bool select_cand_launch(const SelectParams& p, cudaStream_t st);

// Dataflow consumer (kc_consume.cu): a persistent grid that, row by row as
// the scoring kernel completes them (row_done[row] == n_splits), runs the
// selection, the V recall and P.V of the row -- bit-identical to
// select_launch + recall_launch -- while the scoring streams later rows.
struct ConsumeParams {
  const float* logits;     // [batch][n_q][lstride]
  const float2* partials;  // [batch][n_q][max_splits]
  uint32_t* idx;           // [rows][nc]
  float* w;                // [batch*n_q][nc]
  double* dropped;         // [batch*n_q]
  float* norm;             // [batch*n_q]
  int64_t lstride;
  int s;
  int nc;
  int n_kv;
  int G;
  int n_splits;
  int max_splits;
  int row0;
  int rows;
  int keep_logits;
  const void* v;           // layer's V [rows][max_seq][h] (device or mapped host); null: select only
  float* out;              // [batch][n_q*h]
  int64_t max_seq;
  int h;
  int renormalize;
  int reverse;
  uint32_t* row_done;      // [rows][kRowDoneStride] split completion counters; null: rows are complete
  uint32_t* err;           // set before trapping on a row that never completes
  uint64_t* dbg;           // development probe: [rows][8] phase timestamps (ns), or null
};
bool consume_supported(int G, int h);
// stream-ordered GQA row selection with the selection values cached in shared
// memory (one row per CTA); false when the shape is outside it (G not 2/4/8,
// rows too long for the cache) -- the caller then uses select_launch
bool select_rows_cached_launch(const ConsumeParams& p, cudaStream_t st);
// grid: persistent CTAs (<= rows); vdtype: V storage dtype
void consume_launch(const ConsumeParams& p, int vdtype, int grid, cudaStream_t st);

// p = exp(s - M)/Z for every position of every (batch, q head) -> probs
// [batch*n_q][s] (ScoreObserver debug path).
void probs_launch(const SelectParams& p, float* probs, cudaStream_t st);

// Standalone arg_topk over raw floats (ordered-float keys).
void arg_topk_launch(const float* values, int n, int k, uint32_t* keys_scratch, uint32_t* out,
                     cudaStream_t st);

struct RecallParams {
  const void* v;          // layer's V: [rows][max_seq][h] (device or mapped host)
  const uint32_t* idx;    // [rows][nc]
  const float* w;         // [batch*n_q][nc]
  const float* norm;      // [batch*n_q]
  float* out;             // [batch][n_q*h]
  int64_t max_seq;
  int nc;
  int h;
  int n_kv;
  int G;
  int rows;
  int renormalize;
  int reverse;            // fault hook: descending accumulation
  int row_offset;         // first row of this launch (pipelined chunks)
  int staged;             // v is the compacted [rows][nc][h] block (DMA recall)
  int grid;               // CTAs (0: one per row); CTAs loop over rows
  int pipelined;          // use recall_pv_pipe_kernel where the shape allows
  int dbg;                // development probe (pipelined kernel): 1 skip the V loads, 2 no work
  int lean;               // pipelined kernel capped at 72 registers
  int tma;                // recall_tma_kernel (TMA bulk copies of the V rows) where the shape allows
};
void recall_launch(const RecallParams& p, int dtype, cudaStream_t st);

// StepStats accumulation of one TopN layer call (engine.cpp:146-156)
struct StepStatsDev {
  double dropped_sum;
  unsigned long long hist[8];
};
void step_stats_launch(const uint32_t* idx, const double* dropped, int rows, int G, int nc, uint64_t len,
                       int slots, StepStatsDev* acc, cudaStream_t st);

struct PvFullParams {
  const void* v;          // [rows][max_seq][h]
  const float* logits;
  const float2* partials;
  float* part_out;        // scratch [batch*n_q][n_splits][h]
  float* out;             // [batch][n_q*h]
  int64_t max_seq;
  int64_t lstride;
  int s;
  int h;
  int n_kv;
  int G;
  int rows;
  int chunk;
  int n_splits;
  int max_splits;
};
void pv_full_launch(const PvFullParams& p, int dtype, cudaStream_t st);

// decode_attention_full fused (K and V in HBM, h = 128, 16-bit storage):
// one pass per (row, split) streams the split's K then its V through one TMA
// ring -- scores and the split's softmax stay in shared memory -- and leaves
// unnormalised split partials (m, l, sum_j exp(s_j - m) V_j) that
// full_combine folds in split order. Returns false outside its shapes.
struct FullParams {
  const void* k;          // [rows][max_seq][h]
  const void* v;
  const float* q;         // [batch][n_q][h] fp32
  float* part_out;        // [batch*n_q][max_splits][h]
  float2* part_ml;        // [batch*n_q][max_splits] (m, l)
  float* out;             // [batch][n_q*h]
  int64_t max_seq;
  int s;
  int n_kv;
  int G;
  int rows;
  int chunk;
  int n_splits;
  int max_splits;
  float scale;
};
bool full_fast_launch(const FullParams& p, int dtype, cudaStream_t st);

// ---- prefill attention (kc_prefill.cu) ----
// q, k, v, out: device fp32 [s][n_heads*h]; false if h is too large
bool prefill_attention_launch(const float* q, const float* k, const float* v, float* out, int s, int n_heads,
                              int h, cudaStream_t st);

// Position-major [rows][n_kv*h] input rows -> [b][n_kv][max_seq][h] storage
// at positions [pos0, pos0 + rows/batch).
struct AppendParams {
  const void* src;
  void* dst;
  int64_t n_rows;         // m*batch
  int64_t max_seq;
  int64_t pos0;
  int batch;
  int n_kv;
  int h;
};
void append_launch(const AppendParams& p, int src_dtype, int dst_dtype, cudaStream_t st);
// rows x row_bytes at a common pitch, src -> dst, on `grid` CTAs (SM copy)
void copy_rows_launch(const void* src, void* dst, int64_t pitch, int64_t row_bytes, int rows, int grid,
                      cudaStream_t st);

void fill_uniform_launch(void* dst, int dtype, uint64_t n, uint64_t seed, uint64_t offset, float lo,
                         float hi, cudaStream_t st);
// q of any dtype -> fp32
void to_f32_launch(const void* src, int dtype, float* dst, int64_t n, cudaStream_t st);
// [rows][nc] kv-head indices -> [rows*G][nc] q-head slots
void expand_idx_launch(const uint32_t* src, uint32_t* dst, int rows, int G, int nc,
                       cudaStream_t st);

// (slot row, position) pairs of a [rows][max_seq][h] store -> fp32 [n][h]
void gather_rows_launch(const void* base, int dtype, const uint32_t* slot_row, const uint32_t* pos,
                        int64_t n, int h, int64_t max_seq, float* out, cudaStream_t st);

}  // namespace kc

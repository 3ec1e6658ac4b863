/*
 * kcache_c.h -- C ABI of the B200-native KCache decode-attention library
 * (libkcache_b200.so). Plain pointers and sizes only; no torch or C++ types.
 *
 * This is the drop-in boundary for the reference's decode-step TopN attention
 * operator (arXiv 2404.18057 reference, /root/reference/proj). The reference
 * has no FFI of its own: its operator API is the C++ header surface of
 * kcache_core (proj/core/include/kcache/{attention,kv_cache}.hpp). The C++
 * headers under include/kcache/ re-declare that surface source-compatibly and
 * are implemented on top of the functions below (see INTEGRATION.md for the
 * ctypes / C++ bindings a maintainer adds on the reference side).
 *
 * Storage:
 *   K   HBM            [layer][batch][kv_head][max_seq][head_dim]   fp16/bf16/fp32
 *   V   layers <  L    HBM, same layout
 *   V   layers >= L    pinned, device-mapped host memory, same layout
 * Every function returns KC_OK or an error code; kc_last_error() returns a
 * thread-local message. A cache handle is single-owner and not thread-safe,
 * like TieredKVCache.
 */
#ifndef KCACHE_C_H
#define KCACHE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ shim rethrows them as the reference's exceptions
 * (proj/core/include/kcache/errors.hpp:10-38): */
#define KC_OK 0
#define KC_ESHAPE 1     /* kcache::ShapeError            */
#define KC_ESTATE 2     /* kcache::StateError            */
#define KC_ECAPACITY 3  /* kcache::CapacityError         */
#define KC_EARG 4       /* std::invalid_argument         */
#define KC_ERANGE 5     /* std::out_of_range             */
#define KC_ECUDA 6      /* std::runtime_error (CUDA)     */
#define KC_EOVERFLOW 7  /* std::overflow_error (checked_mul, checked.hpp:10-20) */

/* Element types for storage and for q inputs. */
#define KC_F32 0
#define KC_F16 1
#define KC_BF16 2

/* kc_decode_* flags. */
#define KC_RENORMALIZE 1u    /* renormalize=true (attention.cpp:167-174)            */
#define KC_REVERSE_ACCUM 2u  /* ordered_accumulation=false fault hook (:180-186)    */
#define KC_IO_DEVICE 4u      /* q and every output pointer are device pointers;
                                the call is asynchronous on `stream`. Otherwise
                                host pointers and the call returns finished.     */

/* Ledger directions / phases (kv_cache.hpp:14-29). */
#define KC_D2H 0
#define KC_H2D 1
#define KC_PREFILL 0
#define KC_DECODE 1

/* ModelConfig's attention shape (proj/core/include/kcache/model.hpp:18-40).
 * n_kv_heads == n_heads is the reference's MHA; n_heads = G*n_kv_heads is
 * GQA (a B200-side extension). */
typedef struct kc_config {
  uint64_t n_layers;
  uint64_t d_model; /* n_heads * head_dim */
  uint64_t n_heads;
  uint64_t n_kv_heads;
  uint64_t head_dim;
  uint64_t max_seq;
} kc_config;

typedef struct kc_cache kc_cache;

/* Result of one decode_attention_topn call (attention.hpp:20-30,48-52).
 * slot = b*n_heads + head; nc = min(top_n, len). Optional outputs may be NULL. */
typedef struct kc_topn_out {
  float* out;            /* [batch][n_heads*head_dim]                  */
  uint32_t* indices;     /* [batch*n_heads][nc], ascending per slot    */
  float* weights;        /* [batch*n_heads][nc], raw softmax values     */
  double* dropped_mass;  /* [batch*n_heads], 1 - sum(double(weights))  */
  uint64_t nc;           /* written: entries per slot                  */
  uint64_t h2d_bytes;    /* written: ledger H2D bytes of this call     */
} kc_topn_out;

const char* kc_last_error(void);
const char* kc_version(void);

/* TieredKVCache(config, batch, TierPlacement{resident_layers, n_layers,
 * bytes_per_element}, fast_capacity) -- kv_cache.hpp:100-102,
 * kv_cache.cpp:68-81. bytes_per_element is ledger accounting (as in the
 * reference); storage_dtype is the physical element type. device = CUDA
 * ordinal; numa_node < 0 = no binding of the pinned V arena. */
int kc_cache_create(const kc_config* config, uint64_t batch, uint64_t resident_layers,
                    uint64_t bytes_per_element, int storage_dtype, int has_fast_capacity,
                    uint64_t fast_capacity_bytes, int device, int numa_node, kc_cache** out);
int kc_cache_destroy(kc_cache* cache);

/* append_kv (kv_cache.hpp:106, kv_cache.cpp:96-121). k, v: host fp32
 * [rows][n_kv_heads*head_dim], position-major (all batch rows of a position
 * together); rows a positive multiple of batch. Converted on device. */
int kc_append_kv(kc_cache* cache, uint64_t layer, const float* k, const float* v, uint64_t rows);
/* Same, from device buffers of `dtype`, asynchronous on `stream`. The cache's
 * host-mode calls (and kc_sync) are ordered after the last such append; a
 * KC_IO_DEVICE call on another stream than `stream` must be ordered by the
 * caller (same stream, or an event). */
int kc_append_kv_device(kc_cache* cache, uint64_t layer, const void* k, const void* v, int dtype,
                        uint64_t rows, void* stream);

/* offload_prefill_v / begin_decode (kv_cache.cpp:123-148). */
int kc_offload_prefill_v(kc_cache* cache, uint64_t layer);
int kc_begin_decode(kc_cache* cache);

/* decode_attention_topn (attention.hpp:64-67, attention.cpp:116-190).
 * q: [batch][n_heads*head_dim] of q_dtype. */
int kc_decode_topn(kc_cache* cache, uint64_t layer, const void* q, int q_dtype, uint64_t top_n,
                   uint32_t flags, kc_topn_out* out, void* stream);

/* n independent decode_attention_topn calls (one q per layer), pipelined:
 * the V recall + P.V of layers[i] overlaps the scoring of layers[i+1]. This is
 * the attention-only step the bench times; results equal n single calls. */
int kc_decode_topn_layers(kc_cache* cache, uint64_t n, const uint64_t* layers,
                          const void* const* q, int q_dtype, uint64_t top_n, uint32_t flags,
                          kc_topn_out* outs, void* stream);

/* decode_attention_full (attention.hpp:45-46, attention.cpp:91-114):
 * softmax over every position, V read from whichever tier holds it, nothing
 * ledgered. */
int kc_decode_full(kc_cache* cache, uint64_t layer, const void* q, int q_dtype, uint32_t flags,
                   float* out, void* stream);

/* Engine::forward_decode's attention block for one layer
 * (proj/core/src/engine.cpp:139-160): append this step's K/V rows (k_new,
 * v_new: [batch][n_kv_heads*head_dim] of `dtype`; an offloaded layer's new V
 * goes to the pinned arena with the D2H ledger event, kv_cache.cpp:107-112),
 * then decode_attention_topn -- or decode_attention_full with KC_FULL -- with
 * q ([batch][n_heads*head_dim] of `dtype`), writing out [batch][d_model].
 * TopN calls accumulate the step statistics (StepStats, engine.hpp:37-45)
 * on the device: H2D bytes, the dropped mass summed over the selections in
 * slot order, and the 8-bin histogram of selected positions
 * (bin = min(7, idx*8/len), engine.cpp:150-156). KC_IO_DEVICE: q, k_new,
 * v_new and out are device pointers and the call is asynchronous. */
#define KC_FULL 8u
#define KC_POSITION_HISTOGRAM_BINS 8
typedef struct kc_step_stats {
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint64_t selections;     /* dropped-mass terms summed (q-head slots x TopN layers) */
  double dropped_sum;      /* mean_dropped_mass = dropped_sum / selections */
  uint64_t position_histogram[KC_POSITION_HISTOGRAM_BINS];
} kc_step_stats;
int kc_decode_step(kc_cache* cache, uint64_t layer, const void* q, const void* k_new, const void* v_new,
                   int dtype, uint64_t top_n, uint32_t flags, float* out, void* stream);
/* Statistics accumulated by kc_decode_step since the last reset (waits for
 * the cache's queued work); reset != 0 starts a new step. */
int kc_step_stats_read(kc_cache* cache, kc_step_stats* out, int reset);

/* One CUDA Graph per decode step (the reference has no GPU, so
 * no reference counterpart): kc_step_graph_begin allocates every buffer the
 * step may need for this top_n and starts capturing `stream` (thread-local
 * mode); the step's KC_IO_DEVICE kc_decode_step / kc_decode_full calls on
 * that stream are recorded instead of launched -- their host-side effects
 * (cache lengths, ledger events, StepStats counters) happen at capture time
 * exactly as in an eager call. kc_step_graph_launch ends the capture, updates
 * the cache's instantiated graph in place (cudaGraphExecUpdate; a new
 * instantiation when the step's shape changed) and launches it on `stream`.
 * Kernel arguments change every step (the cache grows), so every step is
 * captured once and launched once; the graph removes the per-kernel launch
 * gaps on the device. Host-memory I/O calls are not capturable (KC_ESTATE). */
int kc_step_graph_begin(kc_cache* cache, uint64_t top_n, void* stream);
int kc_step_graph_launch(kc_cache* cache, void* stream);

/* Full softmax rows of every (batch, q head) -- the ScoreObserver debug path
 * (attention.hpp:34-35, attention.cpp:137-139): probs [batch*n_heads][len]
 * fp32, host. Not on the hot path. */
int kc_score_probs(kc_cache* cache, uint64_t layer, const void* q, int q_dtype, float* probs);

/* gather_v (kv_cache.hpp:121, kv_cache.cpp:150-187): counts[batch*n_heads],
 * indices concatenated per slot; out [sum(counts)][head_dim] fp32 (host). */
int kc_gather_v(kc_cache* cache, uint64_t layer, const uint32_t* indices, const uint64_t* counts,
                float* out, uint64_t* h2d_bytes);

/* k_row / v_row (kv_cache.hpp:123-124): one position of one batch row,
 * [n_kv_heads*head_dim] fp32 into host `out`. which: 0 = K, 1 = V. */
int kc_read_row(kc_cache* cache, uint64_t layer, uint64_t pos, uint64_t batch_idx, int which,
                float* out);

/* Accessors (kv_cache.hpp:126-136). */
int kc_current_len(const kc_cache* cache, uint64_t* len);
int kc_phase(const kc_cache* cache, int* phase);
int kc_fast_bytes_used(const kc_cache* cache, uint64_t* bytes);
int kc_slow_bytes_used(const kc_cache* cache, uint64_t* bytes);
int kc_d2h_bytes_total(const kc_cache* cache, uint64_t* bytes);
int kc_h2d_bytes_total(const kc_cache* cache, uint64_t* bytes);
int kc_ledger_size(const kc_cache* cache, uint64_t* n);
int kc_ledger_event(const kc_cache* cache, uint64_t i, int* phase, uint64_t* layer, int* dir,
                    uint64_t* bytes, uint64_t* elements);
/* Device pointers of one layer's K and V storage (V may be a mapped host
 * pointer) and the element strides; for tests and tooling. */
int kc_layer_storage(const kc_cache* cache, uint64_t layer, void** k, void** v, int* v_on_host);
/* Where offloaded V lives: 0 = host-resident UVM managed memory, one
 * allocation per layer (default), 1 = mmap + cudaHostRegister pinned arena
 * (KCACHE_V_ARENA=pinned, or when managed memory is unavailable), 2 = no
 * offloaded layer, 3 = the first layers managed, the rest pinned (the
 * driver's managed-memory cap). */
int kc_v_arena_kind(const kc_cache* cache, int* kind);
/* Wait for all work the cache enqueued: every stream it owns and the last
 * kc_append_kv_device on the caller's stream. */
int kc_sync(kc_cache* cache);
/* Tuning knobs ("score_chunk", "recall_ctas", ...); DESIGN.md lists them. */
int kc_set_tuning(kc_cache* cache, const char* key, int64_t value);

/* Per-kernel CUDA-event timing of subsequent decode calls (bench / roofline):
 * kc_profile(c, 1) clears and starts recording one event pair around every
 * scoring, selection and recall launch on the stream it runs on
 * (kc_profile(c, mask << 1) for a subset: mask bit 0 score, 1 select,
 * 2 recall; kc_profile(c, 0) stops);
 * kc_profile_read(c, "score"|"select"|"recall", ...) returns the summed
 * device time and the launch count. */
int kc_profile(kc_cache* cache, int enable);
int kc_profile_read(kc_cache* cache, const char* kernel, double* total_ms, uint64_t* launches);
int kc_profile_launch(kc_cache* cache, const char* kernel, uint64_t i, double* ms);
/* start / end of launch i in ms since the first profiled event (timelines) */
int kc_profile_span(kc_cache* cache, const char* kernel, uint64_t i, double* t0, double* t1);

/* Development probes (not part of the reference interface): "consume" copies
 * the dataflow consumer's per-row phase timestamps ([rows][8] u64 ns; tuning
 * consume_dbg 1) of the last decode call. */
int kc_debug_read(kc_cache* cache, const char* what, void* out, uint64_t bytes);

/* The split length (positions per scoring work item) the store picks on its
 * own ("score_chunk" 0) for s positions over `rows` (batch x kv head) rows of
 * GQA group `group`. Setting it explicitly on a cache holding a subset of the
 * rows reproduces the full cache's softmax rounding bit for bit (sharding). */
int kc_score_chunk_plan(uint64_t s, uint64_t rows, uint64_t group, int64_t* chunk);

/* prefill_attention (attention.hpp:40, attention.cpp:31-62) on the GPU:
 * causal attention of one sequence, q/k/v/out [s][n_heads*head_dim] fp32,
 * the reference's dot, softmax and accumulation order. Host pointers,
 * synchronous, on `device` (< 0: the calling thread's current device). */
int kc_prefill_attention(const float* q, const float* k, const float* v, uint64_t s, uint64_t n_heads,
                         uint64_t head_dim, float* out, int device);
/* Same with device pointers, asynchronous on `stream`. */
int kc_prefill_attention_device(const float* q, const float* k, const float* v, uint64_t s, uint64_t n_heads,
                                uint64_t head_dim, float* out, void* stream);

/* arg_topk (matrix.hpp:49-52, matrix.cpp:109-122) on the GPU: indices of the
 * k largest of n host floats, ties to the lowest index, ascending. */
int kc_arg_topk(const float* values, uint64_t n, uint64_t k, uint32_t* out, uint64_t* count);

/* Synthetic input generator: elements [offset, offset+n) of SeededRng(seed)
 * .next_uniform(lo, hi) (rng.hpp:13-26), rounded to dtype, written to the
 * device buffer dst. Counter-based, so any slice is reproducible. */
int kc_fill_uniform(void* dst, int dtype, uint64_t n, uint64_t seed, uint64_t offset, float lo,
                    float hi, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KCACHE_C_H */

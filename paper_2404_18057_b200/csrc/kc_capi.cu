// kc_capi.cu -- the C ABI (include/kcache_c.h): the tiered store, its ledger
// and phase machine, and the decode-step orchestration over the sm_100a
// kernels.
//
// Store semantics follow TieredKVCache (proj/core/src/kv_cache.cpp:68-235):
// byte counters, ledger events and errors are the reference's, but storage is
// physical: K in HBM, V of layers >= L in pinned device-mapped host memory
// (from the first append -- the "fast tier" of a not-yet-offloaded layer is a
// ledger state, the bytes already live in the host arena), V of layers < L in
// HBM. Layout [layer][b][kv_head][max_seq][h] so one (b, kv head) row of K is
// a contiguous run the scoring kernel can stream with TMA bulk copies.
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include <memory>


#include "kc_kernels.cuh"
#include "kcache_c.h"

namespace {

thread_local std::string g_err;

struct KcError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw KcError{code, msg}; }

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      fail(KC_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

uint64_t checked_mul(std::initializer_list<uint64_t> f) {
  unsigned __int128 acc = 1;
  for (uint64_t x : f) {
    acc *= x;
    if (acc > (unsigned __int128)UINT64_MAX) fail(KC_EOVERFLOW, "checked_mul: product exceeds 64 bits");
  }
  return (uint64_t)acc;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case KC_F32: return 4;
    case KC_F16:
    case KC_BF16: return 2;
    default: fail(KC_EARG, "unknown dtype " + std::to_string(dt));
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CK(cudaMalloc(&p, std::max<size_t>(n, 256)));
    bytes = std::max<size_t>(n, 256);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    CK(cudaHostAlloc(&p, std::max<size_t>(n, 256), cudaHostAllocPortable));
    bytes = std::max<size_t>(n, 256);
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

struct LedgerEvent {
  int phase;
  uint64_t layer;
  int dir;
  uint64_t bytes;
  uint64_t elements;
};

struct LayerState {
  uint64_t len = 0;
  bool offloaded = false;
  int stage = -1;  // prefill V staged in HBM slot `stage` (see kc_cache::v_stage), -1: in its arena
  uint64_t k_elems = 0, vfast_elems = 0, vslow_elems = 0;
};

constexpr int kRing = 3;

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

struct kc_cache {
  kc_config cfg{};
  uint64_t batch = 0, L = 0, bpe = 2;
  int dtype = KC_F16;
  size_t esz = 2;
  bool has_cap = false;
  uint64_t cap = 0;
  int device = 0;
  int phase = KC_PREFILL;
  uint64_t G = 1, n_kv = 1, h = 1, dkv = 1, n_q = 1, rows = 1;
  std::vector<LayerState> layers;
  std::vector<LedgerEvent> ledger;
  uint64_t d2h_total = 0, h2d_total = 0;

  // storage
  void* k_arena = nullptr;
  size_t k_layer_bytes = 0;
  void* v_dev = nullptr;
  // V of offloaded layers, in host memory. Default: one UVM managed
  // allocation per layer, preferred location host (the GPU's NUMA node),
  // remote-mapped into the GPU (AccessedBy) -- the driver maps it with large
  // GPU pages, so the recall's scattered 256-B reads do not pay a page walk
  // per 4 KB. KCACHE_V_ARENA=pinned selects the mmap +
  // cudaHostRegister arena (4 KB GPU pages).
  std::vector<void*> v_managed;  // [layer - L - n_pin], same pointer on host and device
  uint64_t n_pin = 0;             // offloaded layers in the pinned arena (the first ones)
  void* v_host = nullptr;       // pinned arena: mmap'd, registered
  void* v_host_dev = nullptr;   // device alias of v_host
  size_t v_host_bytes = 0;
  size_t v_layer_bytes = 0;

  // scratch
  int64_t lstride = 0, kstride = 0;
  int max_splits = 0;
  DevBuf logits, partials, keys, part_out, stage_src, stage_k, stage_v, sel_rows, sel_pos, gather_out;
  // dataflow path (kc_consume.cu): a second scoring buffer (slot 1; slot 0 is
  // logits/partials above), per-row split counters per slot, the consumer's
  // error word, and "slot s is free" events
  DevBuf logits_b, partials_b, row_done[2], cons_err;
  // tcgen05 GQA scoring: one 2-D TMA tensor map of K per layer (kc_score_tc.cu)
  struct alignas(64) KMap {
    uint8_t bytes[128];
    bool ok = false;
  };
  std::vector<KMap> kmaps;
  cudaEvent_t ev_cons[2] = {}, ev_scored = nullptr;
  bool cons_pending[2] = {};
  bool cons_dirty = false;   // a scoring launch signalled rows no consumer read
  uint64_t cons_seq = 0;     // layers scored on the dataflow path (slot = seq & 1)
  float* logits_slot(int ls) const { return ls ? logits_b.as<float>() : logits.as<float>(); }
  float2* partials_slot(int ls) const { return ls ? partials_b.as<float2>() : partials.as<float2>(); }
  DevBuf cand, cand_meta, fb_flags;  // candidate-mode selection scratch
  DevBuf part_ml;                    // fused full attention: split (m, l)
  DevBuf step_dev;                   // kc_decode_step: StepStatsDev accumulator
  cudaGraphExec_t step_exec = nullptr;  // kc_step_graph_*: the instantiated step graph
  cudaStream_t capture_st = nullptr;    // stream being captured (nullptr: none)
  kc_step_stats step_host{};         // kc_decode_step: host-known counters
  DevBuf q32[kRing], idx[kRing], w[kRing], dropped[kRing], norm[kRing], out_tmp[kRing], idx_exp[kRing];
  PinnedBuf host_in, host_out;
  DevBuf q_all;  // host-mode multi-layer calls: every layer's q, staged up front
  cudaStream_t in_st = nullptr;  // host-mode q uploads (off the scoring stream)
  cudaEvent_t ev_q0 = nullptr, ev_qall = nullptr;
  cudaStream_t main_st = nullptr, side_st = nullptr, out_st = nullptr;
  cudaStream_t cons_st = nullptr;  // dataflow with a separate recall: the consumer's stream
  cudaEvent_t ev_join = nullptr;
  cudaEvent_t ev_ctr = nullptr;  // the dataflow counters' last reset (on the stream that enqueued it)
  bool ctr_pending = false;      // the next consumer must wait for ev_ctr
  DevBuf join_word;
  int dbg_ctr_race = 0;  // test hook: stale new dataflow counters and a delayed reset
  int flow_join = 1;  // join dataflow calls through out_st + a marker kernel
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_sel[kRing] = {}, ev_rec[kRing] = {},
              ev_out[kRing] = {}, ev_cp[kRing] = {},
              ev_stats = nullptr;
  bool cp_pending[kRing] = {};  // ev_cp[slot] guards a device-mode copy of that slot
  // Device-mode calls (kc_append_kv_device, device decode / full attention)
  // enqueue on the caller's stream: ev_append marks the last of them; the
  // cache's own streams -- and a device-mode call on another stream -- wait
  // on it before touching K/V, logits or the selection ring. Not recorded
  // inside a step-graph capture (a captured event cannot be waited on outside
  // it; kc_step_graph_launch's caller orders the graph on its own stream).
  cudaEvent_t ev_append = nullptr;
  bool append_pending = false;
  void order_after_appends(cudaStream_t st) {
    if (append_pending && !capture_st) CK(cudaStreamWaitEvent(st, ev_append, 0));
    order_after_offloads(st);
  }
  void mark_device_work(cudaStream_t st) {
    if (capture_st) return;
    CK(cudaEventRecord(ev_append, st));
    append_pending = true;
  }

  // Prefill V staging (the paper's overlapped offload): the
  // prefill V of an offloaded layer is appended into one of two HBM stages
  // and leaves for the host arena as ONE copy-engine D2H at
  // offload_prefill_v, on off_st -- behind the caller's next layer instead of
  // as PCIe stores inside the append kernel. A layer whose first append finds
  // both stages still owned (offload not called yet) is appended straight
  // into the arena (mapped stores), as are decode-phase rows.
  DevBuf v_stage[2];
  int stage_owner[2] = {-1, -1};  // layer appended into the slot and not yet offloaded
  bool stage_copy[2] = {};        // ev_off[slot] marks an enqueued D2H of the slot
  int next_stage = 0;
  bool off_pending = false;       // some D2H may still be running
  // tuning: 1 stage (default), 0 mapped stores inside the append (the r01 path)
  int prefill_stage = 1;
  // staged layers in host-resident managed memory leave through an SM copy
  // kernel on off_st (the copy engine writes those pages at 2.2 GB/s, r02
  // tools/prefill_offload_bench.py); pinned-arena layers through the copy
  // engine. stage_copy_ctas: that kernel's grid
  int stage_copy_ctas = 8;  // 8..64 CTAs all reach 52 GB/s (r02)
  cudaStream_t off_st = nullptr;
  cudaEvent_t ev_staged[2] = {}, ev_off[2] = {};
  void order_after_offloads(cudaStream_t st) {
    if (!off_pending) return;
    bool busy = false;
    for (int k = 0; k < 2; ++k) {
      if (!stage_copy[k]) continue;
      if (cudaEventQuery(ev_off[k]) == cudaSuccess) {
        stage_copy[k] = false;
        continue;
      }
      cudaGetLastError();
      busy = true;
      CK(cudaStreamWaitEvent(st, ev_off[k], 0));
    }
    off_pending = busy;
  }

  // tuning
  int score_chunk = 0;
  int pipeline = 1;
  int select_global = 0;
  int score_stages = 4;
  int score_groups = 0;
  int group_first_pct = 0;  // row groups: % of the rows in the first group (0: equal groups)   // row groups per layer (score -> select -> recall each); 0 = auto
  int tlb_ahead = -1;      // K translation warm-up distance in rows (-1 auto: ~3 CTA waves, 0 off); r01: -2 %
  int recall_tma = 0;      // recall_tma_kernel: V rows by TMA bulk copies
  int recall_lean = -1;    // pipelined recall at <= 72 registers (-1: multi-layer calls)
  int recall_dbg = 0;      // development probe: 1 recall without V loads, 2 recall kernel without work
  int tc_grid = 0;         // score_tc_kernel: CTAs per SM of a persistent grid (0: one CTA per item)
  int score_mma = 1;       // GQA scoring on the tensor cores (TF32 split-q mma.sync)
  int k_policy = 0;        // L2 policy of the K stream (kc_device.cuh l2_policy)
  // MHA candidate selection: 0 auto (rows longer than the register-resident
  // dense select), 1 always, 2 never
  int select_cand = 0;
  int cand_force_fallback = 0;  // test hook: every candidate-mode row takes the dense redo
  int full_fused = 1;      // decode_attention_full: fused K+V pass when V is in HBM
  int keep_logits = 0;     // leave dead logits in L2 instead of discarding them
  int recall_pipe = -1;   // software-pipelined recall kernel: -1 auto = GQA only (r01, managed
                          // arena: C3 8.35 -> 7.9 ms per step; MHA C2 no gain)
  int recall_ctas = 32;  // CTAs of the recall kernel (0: one per (batch, kv head)); 32 measured best at C2
  // dataflow consumer (selection + recall + P.V per row as the scoring
  // completes it, kc_consume.cu): 1 on, 0 the stream-ordered select + recall
  //   1 (default) MHA only: GQA keys need the 4 heads' exp per position twice
  //   per row, which the consumer cannot hide behind the shorter GQA scoring
  //   (C3: 329 vs 241 us per layer), 2 every supported shape
  int consume = 1;
  // persistent consumer CTAs; 0 auto: 64 for multi-layer calls (C2 pipelined
  // 338 vs 376 us per layer at 48), 40 for single-layer calls (the engine's
  // layer-by-layer step: 372 vs 425 us at 64 -- fewer CTAs queue fewer PCIe
  // reads ahead of the last rows')
  int consume_ctas = 0;
  int select_cached = 1;
  // dataflow recall: -1 auto (inside the consumer for single-layer calls, the
  // recall kernel on the side stream for multi-layer calls), 1 / 0 force
  int consume_recall = -1;
  // recall grid beside the select-only consumer; 0 = auto: 20 CTAs for calls
  // of >= 8 layers whose recall is short next to the scoring (nc * 256 <= s:
  // C2 under sw_power_cap 334 vs 339 us per layer with 24, 345 with 16),
  // else 24 (the call's last recall is exposed, or the recall is the longer
  // stream: C5 4-layer calls at 16 k / 32 k x N=256 475 / 515 vs 516 / 558)
  int flow_recall_ctas = 0;
  int consume_dbg = 0;    // development probe: consumer phase timestamps (kc_debug_read "consume")
  DevBuf cons_dbg;
  // per-kernel CUDA-event timing (kc_profile): [kind] -> (start, stop) pairs
  bool prof_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof[3];
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  cudaEvent_t prof_event() {
    if (prof_used == prof_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      prof_pool.push_back(e);
    }
    return prof_pool[prof_used++];
  }
  // record around one launch when profiling is on
  int prof_mask = 0;  // bit k: time launches of kind k (0 score, 1 select, 2 recall)
  template <typename F>
  void timed(int kind, cudaStream_t st, F&& launch) {
    if (!prof_on || !((prof_mask >> kind) & 1)) {
      launch();
      return;
    }
    cudaEvent_t a = prof_event(), b = prof_event();
    CK(cudaEventRecord(a, st));
    launch();
    CK(cudaEventRecord(b, st));
    prof[kind].push_back({a, b});
  }

  void* k_layer(uint64_t layer) const { return (char*)k_arena + layer * k_layer_bytes; }
  // offloaded layer j = layer - L: managed layers first, the rest (beyond the
  // driver's managed-memory cap) in the pinned arena
  void* v_layer(uint64_t layer) const {
    if (layer >= L && layers[layer].stage >= 0) return v_stage[layers[layer].stage].p;
    return v_arena_layer(layer);
  }
  // Offloaded layers beyond the driver's managed-memory grant live in the
  // pinned arena -- the FIRST n_pin offloaded layers, so that their slower
  // recall (GPU page walks, section 5 of DESIGN.md) runs under a later
  // layer's scoring rather than as a step's exposed last recall.
  bool layer_managed(uint64_t layer) const { return layer >= L && layer - L >= n_pin; }
  void* v_arena_layer(uint64_t layer) const {
    if (layer < L) return (void*)((char*)v_dev + layer * v_layer_bytes);
    const uint64_t j = layer - L;
    if (j >= n_pin) return v_managed[j - n_pin];
    return (void*)((char*)v_host_dev + j * v_layer_bytes);
  }
  // host view of an offloaded layer's V (host gather path)
  const char* v_host_layer(uint64_t layer) const {
    const uint64_t j = layer - L;
    if (j >= n_pin) return static_cast<const char*>(v_managed[j - n_pin]);
    return static_cast<const char*>(v_host) + j * v_layer_bytes;
  }
  bool v_in_slow(uint64_t layer) const { return layer >= L && layers[layer].offloaded; }
  void check_layer(uint64_t layer) const {
    if (layer >= layers.size())
      fail(KC_ERANGE, "TieredKVCache: layer " + std::to_string(layer) + " out of range");
  }
  uint64_t current_len() const { return layers.empty() ? 0 : layers[0].len; }
  uint64_t fast_bytes() const {
    uint64_t e = 0;
    for (const auto& l : layers) e += l.k_elems + l.vfast_elems;
    return checked_mul({bpe, e});
  }
  uint64_t slow_bytes() const {
    uint64_t e = 0;
    for (const auto& l : layers) e += l.vslow_elems;
    return checked_mul({bpe, e});
  }
  void record(int ph, uint64_t layer, int dir, uint64_t bytes, uint64_t elements) {
    ledger.push_back({ph, layer, dir, bytes, elements});
    (dir == KC_D2H ? d2h_total : h2d_total) += bytes;
  }
};

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return KC_OK;
  } catch (const KcError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return KC_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KC_ECUDA;
  }
}

void set_dev(const kc_cache* c) { CK(cudaSetDevice(c->device)); }

void* alloc_pinned_arena(size_t bytes, int numa_node, void** dev_alias) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE,
                 -1, 0);
  if (p == MAP_FAILED) fail(KC_ECUDA, "mmap of the pinned V arena failed");
  madvise(p, bytes, MADV_HUGEPAGE);
  if (numa_node >= 0 && numa_node < 64) {
    // MPOL_BIND to the GPU's NUMA node (no libnuma in the image: raw syscall);
    // best effort -- single-node hosts simply keep the default policy.
    unsigned long mask = 1ul << numa_node;
    syscall(SYS_mbind, p, bytes, 2 /*MPOL_BIND*/, &mask, 64, 0);
  }
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, bytes);
    fail(KC_ECUDA, std::string("cudaHostRegister(V arena): ") + cudaGetErrorString(e));
  }
  CK(cudaHostGetDevicePointer(dev_alias, p, 0));
  return p;
}

// One managed allocation per offloaded layer: preferred location host (the
// given NUMA node when known), accessed by the cache's GPU (remote mapping,
// no migration), populated on the host up front. Allocates as many of the n
// layers as the driver grants (its managed-memory cap was 64 GiB per process
// on the r01 box) and returns how many; the caller puts the rest in the
// pinned arena.
uint64_t alloc_managed_layers(kc_cache* c, uint64_t n, int numa_node) {
  int concurrent = 0;
  cudaDeviceGetAttribute(&concurrent, cudaDevAttrConcurrentManagedAccess, c->device);
  if (!concurrent) return 0;
  cudaMemLocation host{};
  host.type = numa_node >= 0 ? cudaMemLocationTypeHostNuma : cudaMemLocationTypeHost;
  host.id = numa_node >= 0 ? numa_node : 0;
  cudaMemLocation gpu{};
  gpu.type = cudaMemLocationTypeDevice;
  gpu.id = c->device;
  auto stop = [&](const char* what, cudaError_t e, void* last) {
    if (last) cudaFree(last);
    cudaGetLastError();
    fprintf(stderr, "kcache: %zu of %zu offloaded V layers in managed memory (%s: %s); the rest pinned\n",
            c->v_managed.size(), (size_t)n, what, cudaGetErrorString(e));
    return (uint64_t)c->v_managed.size();
  };
  for (uint64_t i = 0; i < n; ++i) {
    void* p = nullptr;
    cudaError_t e = cudaMallocManaged(&p, c->v_layer_bytes, cudaMemAttachGlobal);
    if (e != cudaSuccess) return stop("cudaMallocManaged", e, nullptr);
    if ((e = cudaMemAdvise(p, c->v_layer_bytes, cudaMemAdviseSetPreferredLocation, host)) != cudaSuccess)
      return stop("SetPreferredLocation", e, p);
    if ((e = cudaMemAdvise(p, c->v_layer_bytes, cudaMemAdviseSetAccessedBy, gpu)) != cudaSuccess)
      return stop("SetAccessedBy", e, p);
    if ((e = cudaMemPrefetchAsync(p, c->v_layer_bytes, host, 0, nullptr)) != cudaSuccess)
      return stop("prefetch to host", e, p);
    c->v_managed.push_back(p);
  }
  CK(cudaDeviceSynchronize());
  return n;
}

void destroy(kc_cache* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->main_st) cudaStreamSynchronize(c->main_st);
  if (c->side_st) cudaStreamSynchronize(c->side_st);
  if (c->cons_st) cudaStreamSynchronize(c->cons_st);
  if (c->out_st) cudaStreamSynchronize(c->out_st);
  if (c->off_st) cudaStreamSynchronize(c->off_st);
  cudaDeviceSynchronize();
  if (c->out_st) cudaStreamDestroy(c->out_st);
  if (c->off_st) cudaStreamDestroy(c->off_st);
  for (int k = 0; k < 2; ++k) {
    c->v_stage[k].release();
    if (c->ev_staged[k]) cudaEventDestroy(c->ev_staged[k]);
    if (c->ev_off[k]) cudaEventDestroy(c->ev_off[k]);
  }
  if (c->in_st) cudaStreamDestroy(c->in_st);
  if (c->ev_q0) cudaEventDestroy(c->ev_q0);
  if (c->ev_qall) cudaEventDestroy(c->ev_qall);
  c->q_all.release();
  if (c->k_arena) cudaFree(c->k_arena);
  if (c->v_dev) cudaFree(c->v_dev);
  if (c->v_host) {
    cudaHostUnregister(c->v_host);
    munmap(c->v_host, c->v_host_bytes);
  }
  for (void* p : c->v_managed) cudaFree(p);
  c->v_managed.clear();
  for (DevBuf* b : {&c->logits_b, &c->partials_b, &c->row_done[0], &c->row_done[1], &c->cons_err}) b->release();
  for (int i = 0; i < 2; ++i)
    if (c->ev_cons[i]) cudaEventDestroy(c->ev_cons[i]);
  if (c->ev_scored) cudaEventDestroy(c->ev_scored);
  for (DevBuf* b : {&c->logits, &c->partials, &c->keys, &c->part_out, &c->stage_src, &c->stage_k,
                    &c->stage_v, &c->sel_rows, &c->sel_pos, &c->gather_out, &c->cand, &c->cand_meta,
                    &c->fb_flags, &c->part_ml, &c->step_dev})
    b->release();
  for (int i = 0; i < kRing; ++i) {
    c->q32[i].release(); c->idx[i].release(); c->w[i].release(); c->dropped[i].release();
    c->norm[i].release(); c->out_tmp[i].release(); c->idx_exp[i].release();
    if (c->ev_sel[i]) cudaEventDestroy(c->ev_sel[i]);
    if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
    if (c->ev_cp[i]) cudaEventDestroy(c->ev_cp[i]);
    if (c->ev_rec[i]) cudaEventDestroy(c->ev_rec[i]);
  }
  c->host_in.release();
  c->host_out.release();
  for (cudaEvent_t e : c->prof_pool) cudaEventDestroy(e);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_ctr) cudaEventDestroy(c->ev_ctr);
  if (c->ev_end) cudaEventDestroy(c->ev_end);
  if (c->ev_stats) cudaEventDestroy(c->ev_stats);
  if (c->ev_append) cudaEventDestroy(c->ev_append);
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  if (c->main_st) cudaStreamDestroy(c->main_st);
  if (c->side_st) cudaStreamDestroy(c->side_st);
  if (c->cons_st) cudaStreamDestroy(c->cons_st);
  delete c;
}

// ---- append ----------------------------------------------------------------
void append_checks(kc_cache* c, uint64_t layer, uint64_t rows) {
  c->check_layer(layer);
  if (rows == 0 || rows % c->batch != 0)
    fail(KC_ESHAPE, "append_kv: need a positive multiple of batch rows for K and V");
  const uint64_t m = rows / c->batch;
  if (c->layers[layer].len + m > c->cfg.max_seq) fail(KC_ESTATE, "append_kv: cache grew past max_seq");
}

// kv_cache.cpp:96-121 accounting after the rows are stored
void append_account(kc_cache* c, uint64_t layer, uint64_t rows) {
  LayerState& st = c->layers[layer];
  const uint64_t elements = rows * c->dkv;
  st.k_elems += elements;
  const bool to_slow = c->phase == KC_DECODE && layer >= c->L;
  if (to_slow) {
    st.vslow_elems += elements;
    c->record(c->phase, layer, KC_D2H, checked_mul({c->bpe, elements}), elements);
  } else {
    st.vfast_elems += elements;
  }
  st.len += rows / c->batch;
  if (c->has_cap && c->fast_bytes() > c->cap)
    fail(KC_ECAPACITY, "fast tier over budget: " + std::to_string(c->fast_bytes()) + " > " +
                           std::to_string(c->cap) + " bytes");
}

// Prefill V of an offloaded layer: on its first append, take a free HBM stage
// (the stream waits for the stage's previous D2H). No free stage -> the layer
// is appended straight into its host arena.
void acquire_stage(kc_cache* c, uint64_t layer, cudaStream_t st) {
  LayerState& ls = c->layers[layer];
  if (!c->prefill_stage || c->phase != KC_PREFILL || layer < c->L || ls.offloaded || ls.stage >= 0 || ls.len > 0)
    return;
  for (int k = 0; k < 2; ++k) {
    const int slot = (c->next_stage + k) & 1;
    if (c->stage_owner[slot] >= 0) continue;
    if (!c->v_stage[slot].p) {
      if (cudaMalloc(&c->v_stage[slot].p, c->v_layer_bytes) != cudaSuccess) {
        cudaGetLastError();  // HBM too tight for a stage: mapped stores instead
        c->v_stage[slot].p = nullptr;
        return;
      }
      c->v_stage[slot].bytes = c->v_layer_bytes;
    }
    if (c->stage_copy[slot]) CK(cudaStreamWaitEvent(st, c->ev_off[slot], 0));
    c->stage_owner[slot] = (int)layer;
    ls.stage = slot;
    c->next_stage = slot ^ 1;
    return;
  }
}

void enqueue_append(kc_cache* c, uint64_t layer, const void* k, const void* v, int dt, uint64_t rows,
                    cudaStream_t st) {
  acquire_stage(c, layer, st);
  kc::AppendParams ap{};
  ap.n_rows = (int64_t)rows;
  ap.max_seq = (int64_t)c->cfg.max_seq;
  ap.pos0 = (int64_t)c->layers[layer].len;
  ap.batch = (int)c->batch;
  ap.n_kv = (int)c->n_kv;
  ap.h = (int)c->h;
  ap.src = k;
  ap.dst = c->k_layer(layer);
  kc::append_launch(ap, dt, c->dtype, st);
  ap.src = v;
  ap.dst = c->v_layer(layer);
  kc::append_launch(ap, dt, c->dtype, st);
  CK(cudaGetLastError());
  const int slot = c->layers[layer].stage;
  if (slot >= 0) CK(cudaEventRecord(c->ev_staged[slot], st));
}

// ---- decode ----------------------------------------------------------------
void decode_checks(kc_cache* c, uint64_t layer) {
  if (c->current_len() == 0) fail(KC_ESTATE, "decode attention: cache is empty");
  c->check_layer(layer);
  if (c->layers[layer].len < c->current_len())
    fail(KC_ERANGE, "k_row: position or batch index out of range");
}

struct StepGeom {
  int s, nc, chunk, n_splits;
};

// chunk_g: the group size the split length is tuned for (the GQA scoring
// kernel wants long items; the fused full-attention kernel the MHA sizing)
StepGeom geom(kc_cache* c, uint64_t top_n, int chunk_g = -1) {
  StepGeom g{};
  g.s = (int)c->current_len();
  g.nc = (int)std::min<uint64_t>(top_n, (uint64_t)g.s);
  g.chunk = kc::score_pick_chunk(g.s, (int)c->rows, c->score_chunk, chunk_g < 0 ? (int)c->G : chunk_g);
  g.n_splits = (g.s + g.chunk - 1) / g.chunk;
  if (g.n_splits > c->max_splits) {
    g.chunk = ((g.s + c->max_splits - 1) / c->max_splits + 63) / 64 * 64;
    g.n_splits = (g.s + g.chunk - 1) / g.chunk;
  }
  return g;
}

void enqueue_score(kc_cache* c, uint64_t layer, const float* q32, const StepGeom& g, cudaStream_t st,
                   int row0, int nrows, bool cand = false, int ls = 0, uint32_t* row_done = nullptr) {
  kc::ScoreParams sp{};
  sp.row0 = row0;
  sp.row_done = row_done;
  if (cand) {
    sp.cand = c->cand.as<uint2>();
    sp.cand_meta = c->cand_meta.as<uint2>();
    sp.cand_nc = g.nc;
  }
  sp.k = c->k_layer(layer);
  sp.q = q32;
  sp.logits = c->logits_slot(ls);
  sp.partials = c->partials_slot(ls);
  sp.max_seq = (int64_t)c->cfg.max_seq;
  sp.lstride = c->lstride;
  sp.s = g.s;
  sp.h = (int)c->h;
  sp.n_kv = (int)c->n_kv;
  sp.G = (int)c->G;
  sp.rows = nrows;
  sp.chunk = g.chunk;
  sp.n_splits = g.n_splits;
  sp.max_splits = c->max_splits;
  sp.scale = 1.0f / std::sqrt(static_cast<float>(c->h));  // attention.hpp:15-17
  sp.stages = c->score_stages;
  sp.k_policy = c->k_policy;
  sp.use_mma = c->score_mma;
  if (c->score_mma == 3 && kc::score_tc_supported(c->dtype, (int)c->h, (int)c->G)) {
    if (c->kmaps.size() < c->layers.size()) c->kmaps.resize(c->layers.size());
    auto& km = c->kmaps[layer];
    if (!km.ok) km.ok = kc::encode_k_map(km.bytes, c->k_layer(layer), c->dtype, c->rows, c->cfg.max_seq);
    sp.kmap = km.ok ? km.bytes : nullptr;
    sp.grid = c->tc_grid > 0 ? c->tc_grid * kc::sm_count() : 0;
  }
  // ~3 waves of CTAs ahead (one CTA per item, 3 per SM)
  sp.tlb_ahead = c->tlb_ahead >= 0 ? c->tlb_ahead
                                    : std::max(1, (3 * kc::sm_count() + g.n_splits - 1) / std::max(g.n_splits, 1));
  c->timed(0, st, [&] { kc::score_launch(sp, c->dtype, st); });
}

// q (any dtype, host or device) -> fp32 device buffer for ring slot
// host_slot/host_slots: position of this q in the call's pageable staging
// (each q of a multi-layer call gets its own slot: the async H2D of q_i may
// still be pending when q_{i+1} is staged).
const float* stage_q(kc_cache* c, int slot, const void* q, int q_dtype, bool io_device,
                     cudaStream_t st, uint64_t host_slot = 0, uint64_t host_slots = 1) {
  const uint64_t nq = c->batch * c->n_q * c->h;
  if (io_device && q_dtype == KC_F32) return static_cast<const float*>(q);
  c->q32[slot].ensure(nq * sizeof(float));
  const void* src = q;
  if (!io_device) {
    const size_t bytes = nq * dtype_size(q_dtype);
    c->stage_src.ensure(bytes * kRing);
    void* dst = (char*)c->stage_src.p + slot * bytes;
    const void* hsrc = q;
    if (!host_pinned(q)) {
      // pageable input: stage through pinned memory so the copy stays async
      c->host_in.ensure(bytes * host_slots);
      void* hp = (char*)c->host_in.p + host_slot * bytes;
      std::memcpy(hp, q, bytes);
      hsrc = hp;
    }
    CK(cudaMemcpyAsync(dst, hsrc, bytes, cudaMemcpyHostToDevice, st));
    src = dst;
  }
  kc::to_f32_launch(src, q_dtype, c->q32[slot].as<float>(), (int64_t)nq, st);
  return c->q32[slot].as<float>();
}

// Multi-layer call: upload (host q, pinned) and/or convert (16-bit q) every
// layer's q up front on in_st, so no H2D or conversion sits between one
// layer's selection and the next layer's scoring on the main stream. The main
// stream waits for layer 0's q now and for the rest before layer 1 (long
// done by then). nullptr: nothing to stage (device fp32 q) or some host q is
// pageable (staged per layer instead).
const float* stage_q_all(kc_cache* c, uint64_t n, const void* const* q, int q_dtype, bool io_device,
                         cudaStream_t st) {
  if (n < 2 || (io_device && q_dtype == KC_F32)) return nullptr;
  if (!io_device)
    for (uint64_t i = 0; i < n; ++i)
      if (!host_pinned(q[i])) return nullptr;
  const uint64_t nq = c->batch * c->n_q * c->h;
  const size_t bytes = nq * dtype_size(q_dtype);
  c->q_all.ensure(checked_mul({n, nq, 4}));
  if (q_dtype != KC_F32 && !io_device) c->stage_src.ensure(bytes * n);
  // the previous call's readers of q_all / stage_src ran on st
  CK(cudaEventRecord(c->ev_q0, st));
  CK(cudaStreamWaitEvent(c->in_st, c->ev_q0, 0));
  float* all = c->q_all.as<float>();
  for (uint64_t i = 0; i < n; ++i) {
    if (io_device) {  // device q of a 16-bit dtype: convert only
      kc::to_f32_launch(q[i], q_dtype, all + i * nq, (int64_t)nq, c->in_st);
    } else if (q_dtype == KC_F32) {
      CK(cudaMemcpyAsync(all + i * nq, q[i], bytes, cudaMemcpyHostToDevice, c->in_st));
    } else {
      void* dst = (char*)c->stage_src.p + i * bytes;
      CK(cudaMemcpyAsync(dst, q[i], bytes, cudaMemcpyHostToDevice, c->in_st));
      kc::to_f32_launch(dst, q_dtype, all + i * nq, (int64_t)nq, c->in_st);
    }
    if (i == 0) CK(cudaEventRecord(c->ev_q0, c->in_st));
  }
  CK(cudaEventRecord(c->ev_qall, c->in_st));
  CK(cudaStreamWaitEvent(st, c->ev_q0, 0));
  return all;
}

void decode_topn_impl(kc_cache* c, uint64_t n, const uint64_t* layers, const void* const* q,
                      int q_dtype, uint64_t top_n, uint32_t flags, kc_topn_out* outs,
                      cudaStream_t user_st) {
  if (top_n == 0) fail(KC_EARG, "decode_attention_topn: top_n must be >= 1");
  dtype_size(q_dtype);
  for (uint64_t i = 0; i < n; ++i) decode_checks(c, layers[i]);
  if (c->G * c->h > 1024) fail(KC_ESHAPE, "decode attention: group*head_dim > 1024 unsupported");
  set_dev(c);
  const bool io_device = flags & KC_IO_DEVICE;
  cudaStream_t st = io_device ? user_st : c->main_st;
  c->order_after_appends(st);
  const StepGeom g = geom(c, top_n);
  const uint64_t nc = (uint64_t)g.nc;
  const uint64_t slots = c->batch * c->n_q;
  for (int r = 0; r < kRing; ++r) {
    c->idx[r].ensure(c->rows * nc * 4);
    c->w[r].ensure(slots * nc * 4);
    c->dropped[r].ensure(slots * 8);
    c->norm[r].ensure(slots * 4);
    if (!io_device) c->out_tmp[r].ensure(slots * c->h * 4);
    if (c->G > 1) c->idx_exp[r].ensure(slots * nc * 4);
  }
  // host outputs land in one pinned staging block per call
  const size_t o_out = slots * c->h * 4, o_idx = slots * nc * 4, o_w = slots * nc * 4, o_dr = slots * 8;
  const size_t per_layer = o_out + o_idx + o_w + o_dr;
  if (!io_device) c->host_out.ensure(per_layer * n);
  // host mode: whether each user output buffer is pinned (D2H straight into
  // it) -- asked once per buffer while enqueueing, reused after the sync
  std::vector<signed char> pinned(io_device ? 0 : n * 4, -1);
  auto user_pinned = [&](uint64_t i, int k, const void* user) {
    signed char& f = pinned[i * 4 + k];
    if (f < 0) f = host_pinned(user) ? 1 : 0;
    return f != 0;
  };

  if (!io_device && c->capture_st) fail(KC_ESTATE, "host-memory I/O inside a step graph capture");
  bool out_used = false;  // c->out_st carries work of this call
  const float* q_all = c->capture_st ? nullptr : stage_q_all(c, n, q, q_dtype, io_device, st);
  // The main stream runs q staging, scoring and selection of layer i; a
  // high-priority side stream runs the recall + P.V of layer i under the
  // scoring of layer i+1. A ring of kRing selection slots orders the two.
  cudaStream_t side = c->pipeline ? c->side_st : st;
  CK(cudaEventRecord(c->ev_start, st));
  if (side != st) {
    CK(cudaStreamWaitEvent(side, c->ev_start, 0));
    CK(cudaStreamWaitEvent(c->cons_st, c->ev_start, 0));
  }

  bool flow_call = false;  // some layer's recalling consumer ran on the side stream
  for (uint64_t i = 0; i < n; ++i) {
    const int slot = (int)(i % kRing);
    const uint64_t layer = layers[i];
    if (q_all && i == 1) CK(cudaStreamWaitEvent(st, c->ev_qall, 0));
    const float* q32 = q_all ? q_all + i * (c->batch * c->n_q * c->h)
                             : stage_q(c, slot, q[i], q_dtype, io_device, st, i, n);
    kc_topn_out& o = outs[i];
    // Dataflow (default): the scoring kernel signals each (batch, kv head) row
    // as its splits complete and a persistent consumer grid on the side stream
    // selects, recalls and reduces the row meanwhile (kc_consume.cu) -- the
    // scoring stream carries nothing but scoring. Scoring buffers alternate
    // between two slots so layer i+1's scoring never waits for layer i's
    // consumer; layer i+2's waits for it (ev_cons).
    // auto (consume 1): MHA rows of >= 16 k positions with N <= 256 -- shorter
    // rows and larger N measured faster stream-ordered (r02 C5 sweep: 4 k x
    // N=128 237 vs 224 us per layer, 32 k x N=512 1097 vs 885: > 1024
    // candidates take the consumer's exact path), and inside a step-graph
    // capture the consumer could only follow its scoring. GQA stays
    // stream-ordered: multi-layer calls hide the recall under the next layer
    // (C3 237 vs 267 us per layer); single-layer calls gain with a small
    // consumer grid on some boxes and lose on others (C3 engine step 11.78 vs
    // 13.43 ms, and 14.10 vs 13.58 ms: the consumer's CTAs reaching the SMs
    // before the scoring's) -- consume 2 opts in
    const bool flow_auto = c->G == 1 && g.nc <= 256 && g.s >= 16384 && !c->capture_st;
    const bool flow = (c->consume == 2 || (c->consume == 1 && flow_auto)) &&
                      kc::consume_supported((int)c->G, (int)c->h) && !c->select_global && c->select_cand != 1;
    if (flow) {
      const int ls = (int)(c->cons_seq & 1);
      const int rows_i = (int)c->rows;
      if (ls == 1) {
        c->logits_b.ensure(c->logits.bytes);
        c->partials_b.ensure(c->partials.bytes);
      }
      // counters zeroed on this call (first use, or after an interrupted
      // call): the consumer, on another stream, must not poll them before
      // the reset -- it orders after ev_ctr below (a fresh cudaMalloc can hold
      // any stale value, e.g. one >= n_splits: a consumer that polled it would
      // take the row as complete and read partials the scoring has not written)
      bool ctr_reset = false;
      DevBuf* fresh[2] = {nullptr, nullptr};
      int n_fresh = 0;
      for (DevBuf* b : {&c->row_done[ls], &c->cons_err}) {
        const size_t want = b == &c->cons_err ? 4 : c->rows * 4 * kc::kRowDoneStride;
        if (b->bytes < want) {
          b->ensure(want);
          if (c->dbg_ctr_race) CK(cudaMemset(b->p, 0xff, b->bytes));  // test hook: stale contents
          fresh[n_fresh++] = b;
        }
      }
      if (n_fresh && c->dbg_ctr_race) {  // test hook: ... and a late reset
        CK(cudaDeviceSynchronize());
        kc::spin_launch(20000000, st);
      }
      for (int k = 0; k < n_fresh; ++k) CK(cudaMemsetAsync(fresh[k]->p, 0, fresh[k]->bytes, st));
      ctr_reset = n_fresh > 0;
      if (c->cons_dirty) {  // an earlier call threw between a scoring launch and its consumer
        // earlier consumers may still be waiting on the counters: reset after them
        if (side != st) {
          for (cudaStream_t o : {c->side_st, c->cons_st}) {
            CK(cudaEventRecord(c->ev_scored, o));
            CK(cudaStreamWaitEvent(st, c->ev_scored, 0));
          }
        }
        for (int k = 0; k < 2; ++k)
          if (c->row_done[k].p) CK(cudaMemsetAsync(c->row_done[k].p, 0, c->row_done[k].bytes, st));
        c->cons_dirty = false;
        ctr_reset = true;
      }
      if (ctr_reset && !c->capture_st) {
        CK(cudaEventRecord(c->ev_ctr, st));
        c->ctr_pending = true;
      }
      if (c->cons_pending[ls]) CK(cudaStreamWaitEvent(st, c->ev_cons[ls], 0));
      c->cons_dirty = true;
      enqueue_score(c, layer, q32, g, st, 0, rows_i, false, ls, c->row_done[ls].as<uint32_t>());
      // Multi-layer calls: the consumer selects only (its own stream) and the
      // recall + P.V of the layer runs as the stream-ordered recall kernel on
      // the side stream under the next layer's scoring -- a consumer that also
      // recalls slows the scoring it runs beside (C2: 334-348 vs 310 us per
      // layer, r02). Single-layer calls (the engine's layer-by-layer step)
      // recall inside the consumer, row by row, so the layer ends shortly after
      // its scoring.
      const bool own_recall = c->consume_recall < 0 ? n == 1 : c->consume_recall != 0;
      cudaStream_t cs = (own_recall || side == st) ? side : c->cons_st;
      flow_call |= own_recall && cs == side;
      if (cs != st) {
        // (inside a capture the consumer node follows its scoring node, and
        // the reset was enqueued before the capture began)
        if (c->ctr_pending && !c->capture_st) {
          CK(cudaStreamWaitEvent(cs, c->ev_ctr, 0));
          c->ctr_pending = false;
        }
        // ring slot `slot` is rewritten: the output copies of layer i-kRing must be done
        if (i >= (uint64_t)kRing) {
          CK(cudaStreamWaitEvent(cs, c->ev_rec[slot], 0));
          if (c->cp_pending[slot]) CK(cudaStreamWaitEvent(cs, c->ev_cp[slot], 0));
        }
        if (c->capture_st) {  // inside a graph the consumer follows the scoring (no spinning node)
          CK(cudaEventRecord(c->ev_scored, st));
          CK(cudaStreamWaitEvent(cs, c->ev_scored, 0));
        }
      }
      kc::ConsumeParams cp{};
      cp.logits = c->logits_slot(ls);
      cp.partials = c->partials_slot(ls);
      cp.idx = c->idx[slot].as<uint32_t>();
      cp.w = c->w[slot].as<float>();
      cp.dropped = c->dropped[slot].as<double>();
      cp.norm = c->norm[slot].as<float>();
      cp.lstride = c->lstride;
      cp.s = g.s;
      cp.nc = g.nc;
      cp.n_kv = (int)c->n_kv;
      cp.G = (int)c->G;
      cp.n_splits = g.n_splits;
      cp.max_splits = c->max_splits;
      cp.row0 = 0;
      cp.rows = rows_i;
      cp.keep_logits = c->keep_logits;
      cp.v = own_recall ? c->v_layer(layer) : nullptr;
      cp.out = io_device ? o.out : c->out_tmp[slot].as<float>();
      cp.max_seq = (int64_t)c->cfg.max_seq;
      cp.h = (int)c->h;
      cp.renormalize = (flags & KC_RENORMALIZE) ? 1 : 0;
      cp.reverse = (flags & KC_REVERSE_ACCUM) ? 1 : 0;
      cp.row_done = c->row_done[ls].as<uint32_t>();
      cp.err = c->cons_err.as<uint32_t>();
      if (c->consume_dbg) {
        c->cons_dbg.ensure(c->rows * 8 * sizeof(uint64_t));
        cp.dbg = c->cons_dbg.as<uint64_t>();
      }
      // auto grid: MHA 44 recalling (r02 final, kc_decode_step at C2: 401-404
      // us per layer vs 410-412 at 40, 404 at 48) / 32 selecting only; GQA 64
      // at <= 16 k positions, 48 beyond, at most one per row (r02
      // kc_decode_step sweeps, us per layer: 32 x 16 k 368 at 64 CTAs vs
      // 387-477 at 72-96 and ~440 stream-ordered; 16 x 32 k 328 at 48, 349 at
      // 64; 8 x 64 k 339-343 at 32-48; 4 x 128 k 367 at 32 vs 464
      // stream-ordered)
      const int ctas = c->consume_ctas > 0 ? c->consume_ctas
                       : c->G > 1 ? std::min(rows_i, g.s <= 16384 ? 64 : 48)
                                  : (own_recall ? 44 : 32);
      c->timed(1, cs, [&] { kc::consume_launch(cp, c->dtype, ctas, cs); });
      c->cons_dirty = false;
      ++c->cons_seq;
      CK(cudaEventRecord(c->ev_cons[ls], cs));
      c->cons_pending[ls] = true;
      CK(cudaEventRecord(c->ev_sel[slot], cs));
      if (!own_recall) {
        if (side != cs) CK(cudaStreamWaitEvent(side, c->ev_sel[slot], 0));
        kc::RecallParams rp{};
        rp.v = c->v_layer(layer);
        rp.grid = c->flow_recall_ctas > 0 ? c->flow_recall_ctas
                  : (n >= 8 && (int64_t)g.nc * 256 <= (int64_t)g.s) ? 20 : 24;
        rp.pipelined = c->recall_pipe < 0 ? (c->G > 1 ? 1 : 0) : c->recall_pipe;
        rp.dbg = c->recall_dbg;
        rp.lean = c->recall_lean > 0 ? 1 : 0;
        rp.tma = c->recall_tma;
        rp.idx = c->idx[slot].as<uint32_t>();
        rp.w = c->w[slot].as<float>();
        rp.norm = c->norm[slot].as<float>();
        rp.out = cp.out;
        rp.max_seq = (int64_t)c->cfg.max_seq;
        rp.nc = g.nc;
        rp.h = (int)c->h;
        rp.n_kv = (int)c->n_kv;
        rp.G = (int)c->G;
        rp.rows = rows_i;
        rp.renormalize = cp.renormalize;
        rp.reverse = cp.reverse;
        rp.row_offset = 0;
        c->timed(2, side, [&] { kc::recall_launch(rp, c->dtype, side); });
      }
    } else {
    // Row groups: score -> select -> recall per group of (batch, kv head)
    // rows, so the recall of group g overlaps the scoring of group g+1.
    // score_groups 0 = auto: one group when layers pipeline against each
    // other, two for a single-layer call (the engine's per-layer block),
    // where only the intra-layer overlap is available (r01: 730 -> 690 us)
    const int64_t want_groups = c->score_groups > 0 ? c->score_groups : (n == 1 ? 2 : 1);
    const int n_groups = (int)std::max<int64_t>(1, std::min<int64_t>(want_groups, (int64_t)c->rows));
    // Candidate mode (MHA, N <= 128): scoring emits only each split's
    // possible top-N positions instead of an fp32 logit per position, and the
    // selection ranks ~1.3 N per split -- automatic for rows longer than the
    // register-resident dense selection.
    const bool cand = (c->select_cand == 1 || (c->select_cand == 0 && g.s > kc::kDenseRegMaxS)) &&
                      !c->select_global && kc::score_cand_supported(c->dtype, (int)c->h, (int)c->G, g.chunk, g.nc);
    if (cand) {
      c->cand.ensure(checked_mul({c->rows, (uint64_t)c->lstride, 8}));
      c->cand_meta.ensure(checked_mul({c->rows, (uint64_t)c->max_splits, 8}));
      c->fb_flags.ensure(c->rows * 4);
    }
    // group sizes: the first group takes group_first_pct % of the rows (0:
    // equal groups), the rest split evenly -- a smaller last group shortens
    // the tail (its selection + recall) that nothing overlaps
    const int rows_i = (int)c->rows;
    int first = (rows_i + n_groups - 1) / n_groups;
    if (n_groups > 1 && c->group_first_pct > 0)
      first = std::max(1, std::min(rows_i - (n_groups - 1), (rows_i * c->group_first_pct + 50) / 100));
    const int rest = n_groups > 1 ? (rows_i - first + n_groups - 2) / (n_groups - 1) : 0;
    for (int gi = 0; gi < n_groups; ++gi) {
      const int r0 = gi == 0 ? 0 : first + (gi - 1) * rest;
      const int nr = std::min<int>(gi == 0 ? first : rest, rows_i - r0);
      if (nr <= 0) break;
      enqueue_score(c, layer, q32, g, st, r0, nr, cand);
      // the selection overwrites ring slot `slot`: the recall of layer i-kRing
      // and the copies of its outputs must be done
      if (gi == 0 && i >= (uint64_t)kRing && side != st) {
        CK(cudaStreamWaitEvent(st, c->ev_rec[slot], 0));
        if (c->cp_pending[slot]) CK(cudaStreamWaitEvent(st, c->ev_cp[slot], 0));
      }

      kc::SelectParams sp{};
      sp.logits = c->logits.as<float>();
      sp.partials = c->partials.as<float2>();
      sp.keys = c->keys.as<uint32_t>();
      sp.idx = c->idx[slot].as<uint32_t>();
      sp.w = c->w[slot].as<float>();
      sp.dropped = c->dropped[slot].as<double>();
      sp.norm = c->norm[slot].as<float>();
      sp.lstride = c->lstride;
      sp.kstride = c->kstride;
      sp.s = g.s;
      sp.nc = g.nc;
      sp.n_kv = (int)c->n_kv;
      sp.G = (int)c->G;
      sp.n_splits = g.n_splits;
      sp.max_splits = c->max_splits;
      sp.row0 = r0;
      sp.rows = nr;
      sp.force_global = c->select_global;
      sp.keep_logits = c->keep_logits;
      if (cand) {
        sp.cand = c->cand.as<uint2>();
        sp.cand_meta = c->cand_meta.as<uint2>();
        sp.fb_flags = c->fb_flags.as<uint32_t>();
        sp.chunk = g.chunk;
        sp.k = c->k_layer(layer);
        sp.q = q32;
        sp.max_seq = (int64_t)c->cfg.max_seq;
        sp.h = (int)c->h;
        sp.kdtype = c->dtype;
        sp.scale = 1.0f / std::sqrt(static_cast<float>(c->h));  // attention.hpp:15-17
        sp.force_fallback = c->cand_force_fallback;
      }
      c->timed(1, st, [&] {
        if (cand) {
          if (!kc::select_cand_launch(sp, st)) fail(KC_ECUDA, "candidate selection unavailable for this shape");
          return;
        }
        // GQA launches of more rows than SMs: select_reg needs > 1 wave of its
        // SM-wide CTAs, the cached one-row kernel holds two rows per SM (C3
        // pipelined: 41.7 -> 37.1 us per layer; the engine's 128-row groups
        // stay on select_reg, 337 vs 356 us per layer)
        if (c->G > 1 && c->select_cached && !c->select_global && nr > kc::sm_count() &&
            kc::consume_supported((int)c->G, (int)c->h)) {
          kc::ConsumeParams cp{};
          cp.logits = sp.logits;
          cp.partials = sp.partials;
          cp.idx = sp.idx;
          cp.w = sp.w;
          cp.dropped = sp.dropped;
          cp.norm = sp.norm;
          cp.lstride = sp.lstride;
          cp.s = sp.s;
          cp.nc = sp.nc;
          cp.n_kv = sp.n_kv;
          cp.G = sp.G;
          cp.n_splits = sp.n_splits;
          cp.max_splits = sp.max_splits;
          cp.row0 = sp.row0;
          cp.rows = sp.rows;
          cp.keep_logits = sp.keep_logits;
          cp.h = (int)c->h;
          if (c->consume_dbg) {
            c->cons_dbg.ensure(c->rows * 8 * sizeof(uint64_t));
            cp.dbg = c->cons_dbg.as<uint64_t>();
          }
          if (kc::select_rows_cached_launch(cp, st)) return;
        }
        kc::select_launch(sp, st);
      });
      CK(cudaEventRecord(c->ev_sel[slot], st));
      if (side != st) CK(cudaStreamWaitEvent(side, c->ev_sel[slot], 0));

      kc::RecallParams rp{};
      rp.v = c->v_layer(layer);
      rp.staged = 0;
      rp.grid = c->recall_ctas;
      rp.pipelined = c->recall_pipe < 0 ? (c->G > 1 ? 1 : 0) : c->recall_pipe;
      rp.dbg = c->recall_dbg;
      // the lean kernel shares SMs better with the next layer's scoring but
      // runs longer alone (C3: pipelined 239 -> 235 us per layer, engine
      // step 335 -> 343): multi-layer calls only by default
      rp.lean = c->recall_lean < 0 ? (n > 1 ? 1 : 0) : c->recall_lean;
      rp.tma = c->recall_tma;
      rp.idx = c->idx[slot].as<uint32_t>();
      rp.w = c->w[slot].as<float>();
      rp.norm = c->norm[slot].as<float>();
      rp.out = io_device ? o.out : c->out_tmp[slot].as<float>();
      rp.max_seq = (int64_t)c->cfg.max_seq;
      rp.nc = g.nc;
      rp.h = (int)c->h;
      rp.n_kv = (int)c->n_kv;
      rp.G = (int)c->G;
      rp.rows = nr;
      rp.renormalize = (flags & KC_RENORMALIZE) ? 1 : 0;
      rp.reverse = (flags & KC_REVERSE_ACCUM) ? 1 : 0;
      rp.row_offset = r0;
      c->timed(2, side, [&] { kc::recall_launch(rp, c->dtype, side); });
    }
    }  // stream-ordered path

    // device mode: the selection outputs depend on the selection only --
    // expand + copy them on their own stream so the side stream runs nothing
    // but recalls (the recall writes o.out itself)
    const bool dev_copies = io_device && (o.indices || o.weights || o.dropped_mass);
    cudaStream_t cst = (dev_copies && side != st) ? c->out_st : side;
    if (cst != side) CK(cudaStreamWaitEvent(cst, c->ev_sel[slot], 0));
    c->cp_pending[slot] = cst != side;
    out_used |= cst != side;
    const uint32_t* idx_slots = c->idx[slot].as<uint32_t>();
    if (io_device) {
      if (c->G > 1 && o.indices) {
        kc::expand_idx_launch(idx_slots, c->idx_exp[slot].as<uint32_t>(), (int)c->rows, (int)c->G, g.nc, cst);
        idx_slots = c->idx_exp[slot].as<uint32_t>();
      }
      if (o.indices) CK(cudaMemcpyAsync(o.indices, idx_slots, o_idx, cudaMemcpyDeviceToDevice, cst));
      if (o.weights) CK(cudaMemcpyAsync(o.weights, c->w[slot].p, o_w, cudaMemcpyDeviceToDevice, cst));
      if (o.dropped_mass)
        CK(cudaMemcpyAsync(o.dropped_mass, c->dropped[slot].p, o_dr, cudaMemcpyDeviceToDevice, cst));
      if (cst != side) CK(cudaEventRecord(c->ev_cp[slot], cst));
    } else {
      // D2H straight into pinned user buffers, else into pinned staging, on
      // their own stream: the selection outputs as soon as the selection is
      // done (GQA index expansion there too, not on the recall stream), the
      // attention output once the recall is
      cudaStream_t ost = side != st ? c->out_st : st;
      out_used |= ost == c->out_st;
      if (ost != st) CK(cudaStreamWaitEvent(ost, c->ev_sel[slot], 0));
      char* hb = (char*)c->host_out.p + i * per_layer;
      auto d2h = [&](int k, void* user, size_t off, const void* src, size_t bytes) {
        if (!user) return;
        void* dst = user_pinned(i, k, user) ? user : (void*)(hb + off);
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ost));
      };
      if (c->G > 1 && o.indices) {
        kc::expand_idx_launch(idx_slots, c->idx_exp[slot].as<uint32_t>(), (int)c->rows, (int)c->G, g.nc, ost);
        idx_slots = c->idx_exp[slot].as<uint32_t>();
      }
      d2h(1, o.indices, o_out, idx_slots, o_idx);
      d2h(2, o.weights, o_out + o_idx, c->w[slot].p, o_w);
      d2h(3, o.dropped_mass, o_out + o_idx + o_w, c->dropped[slot].p, o_dr);
      if (ost != side) {
        CK(cudaEventRecord(c->ev_out[slot], side));
        CK(cudaStreamWaitEvent(ost, c->ev_out[slot], 0));
      }
      d2h(0, o.out, 0, c->out_tmp[slot].p, o_out);
      // the ring slot is free once its outputs have left the device (the main
      // stream waits on ev_rec before reusing it)
      if (ost != side) CK(cudaEventRecord(c->ev_rec[slot], ost));
    }
    if (io_device || side == st) CK(cudaEventRecord(c->ev_rec[slot], side));
    CK(cudaGetLastError());

    // ledger: gather_v charges bytes * sum(counts) * h for offloaded layers
    // (kv_cache.cpp:181-185); GQA recalls one row set per kv head.
    o.nc = nc;
    o.h2d_bytes = 0;
    if (c->v_in_slow(layer)) {
      const uint64_t elements = checked_mul({c->rows, nc, c->h});
      o.h2d_bytes = checked_mul({c->bpe, elements});
      c->record(c->phase, layer, KC_H2D, o.h2d_bytes, elements);
    }
  }
  if (side != st && flow_call && !out_used && c->G > 1 && c->flow_join) {
    // A dataflow call without selection copies: the caller's stream joins
    // the consumer through the output stream and a marker kernel there.
    // Waiting on the consumer's (high-priority) stream directly costs the
    // next call ~100+ us before its scoring starts (measured: C3 single-layer
    // calls 437 vs 299-319 us per layer; the copies kernel of the calls that
    // return their selection had the same effect).
    CK(cudaEventRecord(c->ev_end, side));
    CK(cudaStreamWaitEvent(c->out_st, c->ev_end, 0));
    c->join_word.ensure(4);
    kc::join_mark_launch(c->join_word.as<uint32_t>(), c->out_st);
    CK(cudaEventRecord(c->ev_join, c->out_st));
    CK(cudaStreamWaitEvent(st, c->ev_join, 0));
  } else if (side != st) {
    CK(cudaEventRecord(c->ev_end, side));
    CK(cudaStreamWaitEvent(st, c->ev_end, 0));
    if (out_used) {  // host D2H / device selection copies
      CK(cudaEventRecord(c->ev_end, c->out_st));
      CK(cudaStreamWaitEvent(st, c->ev_end, 0));
    }
  }
  if (io_device) c->mark_device_work(st);
  if (!io_device) {
    CK(cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < n; ++i) {
      const char* hb = (const char*)c->host_out.p + i * per_layer;
      kc_topn_out& o = outs[i];
      auto copy = [&](int k, void* user, size_t off, size_t bytes) {
        if (user && !user_pinned(i, k, user)) std::memcpy(user, hb + off, bytes);
      };
      copy(0, o.out, 0, o_out);
      copy(1, o.indices, o_out, o_idx);
      copy(2, o.weights, o_out + o_idx, o_w);
      copy(3, o.dropped_mass, o_out + o_idx + o_w, o_dr);
    }
  }
}

}  // namespace

extern "C" {

const char* kc_last_error(void) { return g_err.c_str(); }
const char* kc_version(void) { return "kcache-b200 0.1 (sm_100a)"; }

int kc_cache_create(const kc_config* cfg, uint64_t batch, uint64_t resident_layers,
                    uint64_t bytes_per_element, int storage_dtype, int has_fast_capacity,
                    uint64_t fast_capacity_bytes, int device, int numa_node, kc_cache** out) {
  return guarded([&] {
    if (!cfg || !out) fail(KC_EARG, "kc_cache_create: null argument");
    *out = nullptr;
    // ModelConfig::validate (model.cpp:13-27) for the attention fields
    if (!cfg->n_layers || !cfg->d_model || !cfg->n_heads || !cfg->head_dim || !cfg->max_seq)
      fail(KC_ESHAPE, "ModelConfig: all counts must be >= 1");
    if (cfg->d_model != cfg->n_heads * cfg->head_dim)
      fail(KC_ESHAPE, "ModelConfig: d_model must equal n_heads * head_dim");
    const uint64_t n_kv = cfg->n_kv_heads ? cfg->n_kv_heads : cfg->n_heads;
    if (cfg->n_heads % n_kv != 0) fail(KC_ESHAPE, "ModelConfig: n_kv_heads must divide n_heads");
    // TierPlacement::validate (kv_cache.cpp:39-46)
    if (resident_layers > cfg->n_layers)
      fail(KC_ESHAPE, "TierPlacement: resident_layers must be <= n_layers");
    if (bytes_per_element == 0) fail(KC_ESHAPE, "TierPlacement: bytes_per_element must be >= 1");
    if (batch == 0) fail(KC_ESHAPE, "TieredKVCache: batch must be >= 1");
    if (cfg->n_heads / n_kv > 32) fail(KC_ESHAPE, "GQA group size > 32 unsupported");
    const size_t esz = dtype_size(storage_dtype);
    if (cfg->max_seq > (1ull << 30)) fail(KC_ESHAPE, "max_seq too large");

    auto* c = new kc_cache;
    try {
      c->cfg = *cfg;
      c->cfg.n_kv_heads = n_kv;
      c->batch = batch;
      c->L = resident_layers;
      c->bpe = bytes_per_element;
      c->dtype = storage_dtype;
      c->esz = esz;
      c->has_cap = has_fast_capacity != 0;
      c->cap = fast_capacity_bytes;
      c->device = device;
      c->n_kv = n_kv;
      c->h = cfg->head_dim;
      c->n_q = cfg->n_heads;
      c->G = cfg->n_heads / n_kv;
      c->dkv = n_kv * cfg->head_dim;
      c->rows = batch * n_kv;
      c->layers.resize(cfg->n_layers);
      set_dev(c);
      c->k_layer_bytes = checked_mul({c->rows, cfg->max_seq, c->h, esz});
      c->v_layer_bytes = c->k_layer_bytes;
      CK(cudaMalloc(&c->k_arena, checked_mul({c->k_layer_bytes, cfg->n_layers})));
      if (c->L > 0) CK(cudaMalloc(&c->v_dev, checked_mul({c->v_layer_bytes, c->L})));
      if (cfg->n_layers > c->L) {
        const uint64_t n_off = cfg->n_layers - c->L;
        const char* kind = getenv("KCACHE_V_ARENA");
        const uint64_t m = (kind && !strcmp(kind, "pinned")) ? 0 : alloc_managed_layers(c, n_off, numa_node);
        c->n_pin = n_off - m;
        if (m < n_off) {
          c->v_host_bytes = checked_mul({c->v_layer_bytes, n_off - m});
          c->v_host = alloc_pinned_arena(c->v_host_bytes, numa_node, &c->v_host_dev);
        }
      }
      // rows padded to 128 B: the selection kernel drops them from L2 by line
      c->lstride = (int64_t)((cfg->max_seq + 31) & ~31ull);
      c->kstride = c->lstride;
      c->max_splits = (int)((cfg->max_seq + 63) / 64);
      // one scoring buffer: the selection of layer i runs on the scoring
      // stream before the scoring of layer i+1
      c->logits.ensure(checked_mul({batch, c->n_q, (uint64_t)c->lstride, 4}));
      c->partials.ensure(checked_mul({batch, c->n_q, (uint64_t)c->max_splits, 8}));
      c->keys.ensure(checked_mul({c->rows, (uint64_t)c->kstride, 4}));
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithFlags(&c->main_st, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithPriority(&c->side_st, cudaStreamNonBlocking, hi));
      CK(cudaStreamCreateWithPriority(&c->cons_st, cudaStreamNonBlocking, hi));
      CK(cudaStreamCreateWithFlags(&c->out_st, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->off_st, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&c->ev_staged[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_off[k], cudaEventDisableTiming));
      }
      CK(cudaStreamCreateWithFlags(&c->in_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_q0, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_qall, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_ctr, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_end, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_stats, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_append, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_scored, cudaEventDisableTiming));
      for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&c->ev_cons[i], cudaEventDisableTiming));
      for (int i = 0; i < kRing; ++i) {
        CK(cudaEventCreateWithFlags(&c->ev_sel[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_cp[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_rec[i], cudaEventDisableTiming));
      }
    } catch (...) {
      destroy(c);
      throw;
    }
    *out = c;
  });
}

int kc_cache_destroy(kc_cache* c) {
  return guarded([&] { destroy(c); });
}

int kc_append_kv(kc_cache* c, uint64_t layer, const float* k, const float* v, uint64_t rows) {
  return guarded([&] {
    append_checks(c, layer, rows);
    set_dev(c);
    const size_t bytes = rows * c->dkv * sizeof(float);
    c->stage_k.ensure(bytes);
    c->stage_v.ensure(bytes);
    c->order_after_appends(c->main_st);
    CK(cudaMemcpyAsync(c->stage_k.p, k, bytes, cudaMemcpyHostToDevice, c->main_st));
    CK(cudaMemcpyAsync(c->stage_v.p, v, bytes, cudaMemcpyHostToDevice, c->main_st));
    enqueue_append(c, layer, c->stage_k.p, c->stage_v.p, KC_F32, rows, c->main_st);
    CK(cudaStreamSynchronize(c->main_st));
    append_account(c, layer, rows);
  });
}

int kc_append_kv_device(kc_cache* c, uint64_t layer, const void* k, const void* v, int dtype,
                        uint64_t rows, void* stream) {
  return guarded([&] {
    dtype_size(dtype);
    append_checks(c, layer, rows);
    set_dev(c);
    enqueue_append(c, layer, k, v, dtype, rows, (cudaStream_t)stream);
    // the cache's own streams (host-mode calls, k_row/v_row, gather_v) must
    // not read these rows before the caller's stream has written them
    CK(cudaEventRecord(c->ev_append, (cudaStream_t)stream));
    c->append_pending = true;
    append_account(c, layer, rows);
  });
}

int kc_offload_prefill_v(kc_cache* c, uint64_t layer) {
  return guarded([&] {
    c->check_layer(layer);
    if (layer < c->L) return;
    LayerState& st = c->layers[layer];
    if (st.offloaded)
      fail(KC_ESTATE, "offload_prefill_v: layer " + std::to_string(layer) + " already offloaded");
    const uint64_t elements = st.vfast_elems;
    if (st.stage >= 0) {
      // the staged prefill V -> its host arena: one copy-engine D2H behind the
      // layer's last append, asynchronous to the caller (readers of the layer
      // wait on ev_off: order_after_offloads)
      set_dev(c);
      const int slot = st.stage;
      const size_t pitch = (size_t)c->cfg.max_seq * c->h * c->esz;
      CK(cudaStreamWaitEvent(c->off_st, c->ev_staged[slot], 0));
      if (st.len > 0) {
        if (c->layer_managed(layer))
          kc::copy_rows_launch(c->v_stage[slot].p, c->v_arena_layer(layer), (int64_t)pitch,
                               (int64_t)(st.len * c->h * c->esz), (int)c->rows, c->stage_copy_ctas, c->off_st);
        else
          CK(cudaMemcpy2DAsync(c->v_arena_layer(layer), pitch, c->v_stage[slot].p, pitch, st.len * c->h * c->esz,
                               c->rows, cudaMemcpyDefault, c->off_st));
        CK(cudaGetLastError());
      }
      CK(cudaEventRecord(c->ev_off[slot], c->off_st));
      c->stage_copy[slot] = true;
      c->stage_owner[slot] = -1;
      c->off_pending = true;
      st.stage = -1;
    }
    st.vslow_elems += elements;
    st.vfast_elems = 0;
    st.offloaded = true;
    c->record(KC_PREFILL, layer, KC_D2H, checked_mul({c->bpe, elements}), elements);
  });
}

int kc_begin_decode(kc_cache* c) {
  return guarded([&] {
    for (uint64_t l = c->L; l < c->layers.size(); ++l)
      if (!c->layers[l].offloaded)
        fail(KC_ESTATE, "begin_decode: layer " + std::to_string(l) + " was never offloaded");
    // every prefill stage has been handed to the copy engine: once its D2H
    // lands the HBM goes back to the caller
    if (c->v_stage[0].p || c->v_stage[1].p) {
      set_dev(c);
      CK(cudaStreamSynchronize(c->off_st));
      c->v_stage[0].release();
      c->v_stage[1].release();
      c->stage_copy[0] = c->stage_copy[1] = false;
      c->off_pending = false;
    }
    c->phase = KC_DECODE;
  });
}

int kc_decode_topn(kc_cache* c, uint64_t layer, const void* q, int q_dtype, uint64_t top_n,
                   uint32_t flags, kc_topn_out* out, void* stream) {
  return guarded([&] {
    if (!out || !q) fail(KC_EARG, "kc_decode_topn: null argument");
    const void* qs[1] = {q};
    decode_topn_impl(c, 1, &layer, qs, q_dtype, top_n, flags, out, (cudaStream_t)stream);
  });
}

int kc_decode_step(kc_cache* c, uint64_t layer, const void* q, const void* k_new, const void* v_new,
                   int dtype, uint64_t top_n, uint32_t flags, float* out, void* stream) {
  return guarded([&] {
    if (!q || !k_new || !v_new || !out) fail(KC_EARG, "kc_decode_step: null argument");
    const size_t esz = dtype_size(dtype);
    if (!(flags & KC_FULL) && top_n == 0) fail(KC_EARG, "decode_attention_topn: top_n must be >= 1");
    const bool io_device = flags & KC_IO_DEVICE;
    if (!io_device && c->capture_st) fail(KC_ESTATE, "host-memory I/O inside a step graph capture");
    set_dev(c);
    cudaStream_t st = io_device ? (cudaStream_t)stream : c->main_st;
    c->order_after_appends(st);
    // engine.cpp:143 -- this step's K/V row of every batch row
    const uint64_t rows = c->batch;
    append_checks(c, layer, rows);
    const uint64_t d2h0 = c->d2h_total;
    const void* ks = k_new;
    const void* vs = v_new;
    if (!io_device) {
      const size_t bytes = rows * c->dkv * esz;
      c->stage_k.ensure(bytes);
      c->stage_v.ensure(bytes);
      CK(cudaMemcpyAsync(c->stage_k.p, k_new, bytes, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(c->stage_v.p, v_new, bytes, cudaMemcpyHostToDevice, st));
      ks = c->stage_k.p;
      vs = c->stage_v.p;
    }
    enqueue_append(c, layer, ks, vs, dtype, rows, st);
    append_account(c, layer, rows);
    c->step_host.d2h_bytes += c->d2h_total - d2h0;
    if (flags & KC_FULL) {
      const int rc = kc_decode_full(c, layer, q, dtype, flags & KC_IO_DEVICE, out, st);
      if (rc != KC_OK) fail(rc, kc_last_error());
      return;
    }
    kc_topn_out o{};
    o.out = out;
    const void* qs[1] = {q};
    decode_topn_impl(c, 1, &layer, qs, dtype, top_n, flags & (KC_RENORMALIZE | KC_IO_DEVICE), &o, st);
    // engine.cpp:146-156 on the device: ring slot 0 holds this call's
    // selection. The statistics need the selection only, so they run off the
    // critical path on the output stream (the caller's stream waits for them,
    // long done, together with the recall).
    const uint64_t slots = c->batch * c->n_q;
    cudaStream_t sst = c->pipeline ? c->out_st : st;
    if (sst != st) CK(cudaStreamWaitEvent(sst, c->ev_sel[0], 0));
    if (!c->step_dev.p) {
      c->step_dev.ensure(sizeof(kc::StepStatsDev));
      CK(cudaMemsetAsync(c->step_dev.p, 0, sizeof(kc::StepStatsDev), sst));
    }
    kc::step_stats_launch(c->idx[0].as<uint32_t>(), c->dropped[0].as<double>(), (int)c->rows, (int)c->G,
                          (int)o.nc, c->current_len(), (int)slots,
                          static_cast<kc::StepStatsDev*>(c->step_dev.p), sst);
    CK(cudaGetLastError());
    if (sst != st) {
      CK(cudaEventRecord(c->ev_stats, sst));
      CK(cudaStreamWaitEvent(st, c->ev_stats, 0));
    }
    c->step_host.h2d_bytes += o.h2d_bytes;
    c->step_host.selections += slots;
    if (io_device) c->mark_device_work(st);  // after the StepStats join
    if (!io_device) CK(cudaStreamSynchronize(st));
  });
}

// Every buffer a device-mode decode step may allocate lazily, allocated now:
// nothing may cudaMalloc while a step is being captured.
void prepare_step_buffers(kc_cache* c, uint64_t top_n, cudaStream_t st) {
  const uint64_t nc = std::min<uint64_t>(top_n, c->cfg.max_seq);
  const uint64_t slots = c->batch * c->n_q;
  for (int r = 0; r < kRing; ++r) {
    c->idx[r].ensure(c->rows * nc * 4);
    c->w[r].ensure(slots * nc * 4);
    c->dropped[r].ensure(slots * 8);
    c->norm[r].ensure(slots * 4);
    if (c->G > 1) c->idx_exp[r].ensure(slots * nc * 4);
    c->q32[r].ensure(slots * c->h * sizeof(float));
  }
  if (c->G == 1 && c->select_cand != 2) {  // candidate mode may switch on as the rows grow
    c->cand.ensure(checked_mul({c->rows, (uint64_t)c->lstride, 8}));
    c->cand_meta.ensure(checked_mul({c->rows, (uint64_t)c->max_splits, 8}));
    c->fb_flags.ensure(c->rows * 4);
  }
  if (!c->step_dev.p) {
    c->step_dev.ensure(sizeof(kc::StepStatsDev));
    CK(cudaMemsetAsync(c->step_dev.p, 0, sizeof(kc::StepStatsDev), st));
  }
  // dataflow path: both scoring slots, the row counters and the error word
  c->logits_b.ensure(c->logits.bytes);
  c->partials_b.ensure(c->partials.bytes);
  bool reset = false;
  for (DevBuf* b : {&c->row_done[0], &c->row_done[1], &c->cons_err}) {
    const size_t want = b == &c->cons_err ? 4 : c->rows * 4 * kc::kRowDoneStride;
    if (b->bytes < want) {
      b->ensure(want);
      CK(cudaMemsetAsync(b->p, 0, b->bytes, st));
      reset = true;
    }
  }
  if (reset) {  // a later dataflow consumer orders after this reset (ctr_pending)
    CK(cudaEventRecord(c->ev_ctr, st));
    c->ctr_pending = true;
  }
  if (c->L > 0) {  // full attention on the V-resident layers
    c->part_out.ensure(checked_mul({slots, (uint64_t)c->max_splits, c->h, 4}));
    c->part_ml.ensure(checked_mul({slots, (uint64_t)c->max_splits, 8}));
  }
}

int kc_step_graph_begin(kc_cache* c, uint64_t top_n, void* stream) {
  return guarded([&] {
    if (!stream) fail(KC_EARG, "kc_step_graph_begin: needs the caller's (non-default) stream");
    if (c->capture_st) fail(KC_ESTATE, "kc_step_graph_begin: a step capture is already open");
    set_dev(c);
    cudaStream_t st = (cudaStream_t)stream;
    prepare_step_buffers(c, top_n, st);
    // the cache's own streams must not hold work the captured step would
    // have to order against (their events would cross the capture boundary)
    CK(cudaStreamSynchronize(c->side_st));
    CK(cudaStreamSynchronize(c->cons_st));
    CK(cudaStreamSynchronize(c->out_st));
    // everything before the capture is complete: the dataflow slot events
    // recorded outside it must not be waited on inside it
    CK(cudaStreamSynchronize(c->main_st));
    c->cons_pending[0] = c->cons_pending[1] = false;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    c->capture_st = st;
  });
}

int kc_step_graph_launch(kc_cache* c, void* stream) {
  return guarded([&] {
    cudaStream_t st = (cudaStream_t)stream;
    if (!c->capture_st || c->capture_st != st) fail(KC_ESTATE, "kc_step_graph_launch: no capture open on this stream");
    set_dev(c);
    c->capture_st = nullptr;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamEndCapture(st, &graph));
    // kernel arguments (cache length, split counts, grids) change every step:
    // update the instantiated graph in place, re-instantiate on a topology change
    bool ok = false;
    if (c->step_exec) {
      cudaGraphExecUpdateResultInfo info{};
      ok = cudaGraphExecUpdate(c->step_exec, graph, &info) == cudaSuccess;
      if (!ok) {
        cudaGetLastError();
        cudaGraphExecDestroy(c->step_exec);
        c->step_exec = nullptr;
      }
    }
    cudaError_t e = cudaSuccess;
    if (!ok) e = cudaGraphInstantiate(&c->step_exec, graph, 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(c->step_exec, st);
    cudaGraphDestroy(graph);
    CK(e);
    // events recorded inside the capture are graph nodes: later calls order
    // after the launched graph instead (its stream), not after them
    c->cons_pending[0] = c->cons_pending[1] = false;
    c->mark_device_work(st);
  });
}

int kc_step_stats_read(kc_cache* c, kc_step_stats* out, int reset) {
  return guarded([&] {
    if (!out) fail(KC_EARG, "kc_step_stats_read: null argument");
    set_dev(c);
    CK(cudaStreamSynchronize(c->main_st));
    CK(cudaStreamSynchronize(c->side_st));
    CK(cudaDeviceSynchronize());
    kc::StepStatsDev d{};
    if (c->step_dev.p) CK(cudaMemcpy(&d, c->step_dev.p, sizeof d, cudaMemcpyDeviceToHost));
    *out = c->step_host;
    out->dropped_sum = d.dropped_sum;
    for (int i = 0; i < KC_POSITION_HISTOGRAM_BINS; ++i) out->position_histogram[i] = d.hist[i];
    if (reset) {
      c->step_host = kc_step_stats{};
      if (c->step_dev.p) CK(cudaMemset(c->step_dev.p, 0, sizeof(kc::StepStatsDev)));
    }
  });
}

int kc_decode_topn_layers(kc_cache* c, uint64_t n, const uint64_t* layers, const void* const* q,
                          int q_dtype, uint64_t top_n, uint32_t flags, kc_topn_out* outs,
                          void* stream) {
  return guarded([&] {
    if (n == 0) return;
    if (!layers || !q || !outs) fail(KC_EARG, "kc_decode_topn_layers: null argument");
    decode_topn_impl(c, n, layers, q, q_dtype, top_n, flags, outs, (cudaStream_t)stream);
  });
}

int kc_decode_full(kc_cache* c, uint64_t layer, const void* q, int q_dtype, uint32_t flags,
                   float* out, void* stream) {
  return guarded([&] {
    if (!q || !out) fail(KC_EARG, "kc_decode_full: null argument");
    dtype_size(q_dtype);
    decode_checks(c, layer);
    if (c->G * c->h > 1024) fail(KC_ESHAPE, "decode attention: group*head_dim > 1024 unsupported");
    set_dev(c);
    const bool io_device = flags & KC_IO_DEVICE;
    cudaStream_t st = io_device ? (cudaStream_t)stream : c->main_st;
    if (!io_device && c->capture_st) fail(KC_ESTATE, "host-memory I/O inside a step graph capture");
    c->order_after_appends(st);
    const StepGeom g = geom(c, 1, 1);  // fused full kernel: MHA split sizing
    const float* q32 = stage_q(c, 0, q, q_dtype, io_device, st);
    const uint64_t slots = c->batch * c->n_q;
    if (!io_device) c->out_tmp[0].ensure(slots * c->h * 4);
    float* out_dev = io_device ? out : c->out_tmp[0].as<float>();
    bool fused = false;
    if (c->h == 128 && !c->v_in_slow(layer) && c->full_fused) {
      // K and V both in HBM: one fused pass (kc_score.cu full_fast_kernel)
      c->part_out.ensure(checked_mul({slots, (uint64_t)c->max_splits, c->h, 4}));
      c->part_ml.ensure(checked_mul({slots, (uint64_t)c->max_splits, 8}));
      kc::FullParams fp{};
      fp.k = c->k_layer(layer);
      fp.v = c->v_layer(layer);
      fp.q = q32;
      fp.part_out = c->part_out.as<float>();
      fp.part_ml = c->part_ml.as<float2>();
      fp.out = out_dev;
      fp.max_seq = (int64_t)c->cfg.max_seq;
      fp.s = g.s;
      fp.n_kv = (int)c->n_kv;
      fp.G = (int)c->G;
      fp.rows = (int)c->rows;
      fp.chunk = g.chunk;
      fp.n_splits = g.n_splits;
      fp.max_splits = c->max_splits;
      fp.scale = 1.0f / std::sqrt(static_cast<float>(c->h));  // attention.hpp:15-17
      c->timed(0, st, [&] { fused = kc::full_fast_launch(fp, c->dtype, st); });
    }
    if (fused) {
      CK(cudaGetLastError());
      if (!io_device) {
        CK(cudaMemcpyAsync(out, c->out_tmp[0].p, slots * c->h * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      } else {
        c->mark_device_work(st);
      }
      return;
    }
    enqueue_score(c, layer, q32, g, st, 0, (int)c->rows);
    c->part_out.ensure(checked_mul({slots, (uint64_t)g.n_splits, c->h, 4}));
    kc::PvFullParams pp{};
    pp.v = c->v_layer(layer);
    pp.logits = c->logits.as<float>();
    pp.partials = c->partials.as<float2>();
    pp.part_out = c->part_out.as<float>();
    pp.out = out_dev;
    pp.max_seq = (int64_t)c->cfg.max_seq;
    pp.lstride = c->lstride;
    pp.s = g.s;
    pp.h = (int)c->h;
    pp.n_kv = (int)c->n_kv;
    pp.G = (int)c->G;
    pp.rows = (int)c->rows;
    pp.chunk = g.chunk;
    pp.n_splits = g.n_splits;
    pp.max_splits = c->max_splits;
    kc::pv_full_launch(pp, c->dtype, st);
    CK(cudaGetLastError());
    if (io_device) c->mark_device_work(st);
    if (!io_device) {
      CK(cudaMemcpyAsync(out, c->out_tmp[0].p, slots * c->h * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  });
}

int kc_score_probs(kc_cache* c, uint64_t layer, const void* q, int q_dtype, float* probs) {
  return guarded([&] {
    if (!q || !probs) fail(KC_EARG, "kc_score_probs: null argument");
    dtype_size(q_dtype);
    decode_checks(c, layer);
    set_dev(c);
    cudaStream_t st = c->main_st;
    c->order_after_appends(st);
    const StepGeom g = geom(c, 1);
    const float* q32 = stage_q(c, 0, q, q_dtype, false, st);
    enqueue_score(c, layer, q32, g, st, 0, (int)c->rows);
    const uint64_t slots = c->batch * c->n_q;
    c->gather_out.ensure(checked_mul({slots, (uint64_t)g.s, 4}));
    kc::SelectParams sp{};
    sp.logits = c->logits.as<float>();
    sp.partials = c->partials.as<float2>();
    sp.lstride = c->lstride;
    sp.s = g.s;
    sp.n_kv = (int)c->n_kv;
    sp.G = (int)c->G;
    sp.n_splits = g.n_splits;
    sp.max_splits = c->max_splits;
    sp.rows = (int)c->rows;
    kc::probs_launch(sp, c->gather_out.as<float>(), st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(probs, c->gather_out.p, slots * g.s * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int kc_gather_v(kc_cache* c, uint64_t layer, const uint32_t* indices, const uint64_t* counts,
                float* out, uint64_t* h2d_bytes) {
  return guarded([&] {
    c->check_layer(layer);
    const uint64_t slots = c->batch * c->n_q;
    uint64_t total = 0;
    for (uint64_t s = 0; s < slots; ++s) total += counts[s];
    std::vector<uint32_t> rows(total), pos(total);
    const uint64_t len = c->layers[layer].len;
    uint64_t e = 0;
    for (uint64_t s = 0; s < slots; ++s) {
      const uint64_t b = s / c->n_q, head = s % c->n_q;
      for (uint64_t r = 0; r < counts[s]; ++r, ++e) {
        if (indices[e] >= len)
          fail(KC_ERANGE, "gather_v: index " + std::to_string(indices[e]) + " past current length " +
                              std::to_string(len));
        rows[e] = (uint32_t)(b * c->n_kv + head / c->G);
        pos[e] = indices[e];
      }
    }
    set_dev(c);
    if (total > 0) {
      c->sel_rows.ensure(total * 4);
      c->sel_pos.ensure(total * 4);
      c->gather_out.ensure(total * c->h * 4);
      c->order_after_appends(c->main_st);
      CK(cudaMemcpyAsync(c->sel_rows.p, rows.data(), total * 4, cudaMemcpyHostToDevice, c->main_st));
      CK(cudaMemcpyAsync(c->sel_pos.p, pos.data(), total * 4, cudaMemcpyHostToDevice, c->main_st));
      kc::gather_rows_launch(c->v_layer(layer), c->dtype, c->sel_rows.as<uint32_t>(),
                             c->sel_pos.as<uint32_t>(), (int64_t)total, (int)c->h,
                             (int64_t)c->cfg.max_seq, c->gather_out.as<float>(), c->main_st);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(out, c->gather_out.p, total * c->h * 4, cudaMemcpyDeviceToHost, c->main_st));
      CK(cudaStreamSynchronize(c->main_st));
    }
    uint64_t bytes = 0;
    if (c->v_in_slow(layer)) {
      const uint64_t elements = checked_mul({total, c->h});
      bytes = checked_mul({c->bpe, elements});
      c->record(c->phase, layer, KC_H2D, bytes, elements);
    }
    if (h2d_bytes) *h2d_bytes = bytes;
  });
}

int kc_read_row(kc_cache* c, uint64_t layer, uint64_t pos, uint64_t bi, int which, float* out) {
  return guarded([&] {
    c->check_layer(layer);
    if (pos >= c->layers[layer].len || bi >= c->batch)
      fail(KC_ERANGE, std::string(which ? "v_row" : "k_row") + ": position or batch index out of range");
    set_dev(c);
    std::vector<uint32_t> rows(c->n_kv), ps(c->n_kv, (uint32_t)pos);
    for (uint64_t k = 0; k < c->n_kv; ++k) rows[k] = (uint32_t)(bi * c->n_kv + k);
    c->sel_rows.ensure(c->n_kv * 4);
    c->sel_pos.ensure(c->n_kv * 4);
    c->gather_out.ensure(c->dkv * 4);
    c->order_after_appends(c->main_st);
    CK(cudaMemcpyAsync(c->sel_rows.p, rows.data(), c->n_kv * 4, cudaMemcpyHostToDevice, c->main_st));
    CK(cudaMemcpyAsync(c->sel_pos.p, ps.data(), c->n_kv * 4, cudaMemcpyHostToDevice, c->main_st));
    kc::gather_rows_launch(which ? c->v_layer(layer) : c->k_layer(layer), c->dtype,
                           c->sel_rows.as<uint32_t>(), c->sel_pos.as<uint32_t>(), (int64_t)c->n_kv,
                           (int)c->h, (int64_t)c->cfg.max_seq, c->gather_out.as<float>(), c->main_st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, c->gather_out.p, c->dkv * 4, cudaMemcpyDeviceToHost, c->main_st));
    CK(cudaStreamSynchronize(c->main_st));
  });
}

int kc_current_len(const kc_cache* c, uint64_t* len) {
  return guarded([&] { *len = c->current_len(); });
}
int kc_phase(const kc_cache* c, int* phase) {
  return guarded([&] { *phase = c->phase; });
}
int kc_fast_bytes_used(const kc_cache* c, uint64_t* bytes) {
  return guarded([&] { *bytes = c->fast_bytes(); });
}
int kc_slow_bytes_used(const kc_cache* c, uint64_t* bytes) {
  return guarded([&] { *bytes = c->slow_bytes(); });
}
int kc_d2h_bytes_total(const kc_cache* c, uint64_t* bytes) {
  return guarded([&] { *bytes = c->d2h_total; });
}
int kc_h2d_bytes_total(const kc_cache* c, uint64_t* bytes) {
  return guarded([&] { *bytes = c->h2d_total; });
}
int kc_ledger_size(const kc_cache* c, uint64_t* n) {
  return guarded([&] { *n = c->ledger.size(); });
}
int kc_ledger_event(const kc_cache* c, uint64_t i, int* phase, uint64_t* layer, int* dir,
                    uint64_t* bytes, uint64_t* elements) {
  return guarded([&] {
    if (i >= c->ledger.size()) fail(KC_ERANGE, "ledger event index out of range");
    const LedgerEvent& e = c->ledger[i];
    *phase = e.phase;
    *layer = e.layer;
    *dir = e.dir;
    *bytes = e.bytes;
    *elements = e.elements;
  });
}
int kc_layer_storage(const kc_cache* c, uint64_t layer, void** k, void** v, int* v_on_host) {
  return guarded([&] {
    c->check_layer(layer);
    *k = c->k_layer(layer);
    *v = c->v_layer(layer);
    *v_on_host = layer >= c->L ? 1 : 0;
  });
}
int kc_v_arena_kind(const kc_cache* c, int* kind) {
  return guarded([&] {
    if (!kind) fail(KC_EARG, "kc_v_arena_kind: null argument");
    *kind = c->v_managed.empty() ? (c->v_host ? 1 : 2) : (c->v_host ? 3 : 0);
  });
}

int kc_sync(kc_cache* c) {
  return guarded([&] {
    set_dev(c);
    for (cudaStream_t s : {c->main_st, c->side_st, c->cons_st, c->out_st, c->in_st, c->off_st})
      if (s) CK(cudaStreamSynchronize(s));
    if (c->append_pending) CK(cudaEventSynchronize(c->ev_append));
  });
}
int kc_set_tuning(kc_cache* c, const char* key, int64_t value) {
  return guarded([&] {
    const std::string k = key ? key : "";
    if (k == "score_chunk") c->score_chunk = (int)value;
    else if (k == "pipeline") c->pipeline = value ? 1 : 0;
    else if (k == "select_global") c->select_global = value ? 1 : 0;
    else if (k == "score_stages") c->score_stages = (int)value;
    else if (k == "recall_ctas") c->recall_ctas = (int)value;
    else if (k == "recall_pipe") c->recall_pipe = value < 0 ? -1 : (value ? 1 : 0);
    else if (k == "side_priority") {
      // 1: the recall stream at the device's highest priority (default), 0: normal
      set_dev(c);
      CK(cudaStreamSynchronize(c->side_st));
      CK(cudaStreamDestroy(c->side_st));
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&c->side_st, cudaStreamNonBlocking, value ? hi : lo));
    }
    else if (k == "keep_logits") c->keep_logits = value ? 1 : 0;
    else if (k == "prefill_stage") c->prefill_stage = value ? 1 : 0;
    else if (k == "stage_copy_ctas") {
      if (value < 1) fail(KC_EARG, "stage_copy_ctas must be >= 1");
      c->stage_copy_ctas = (int)value;
    }
    else if (k == "group_first_pct") {
      if (value < 0 || value > 100) fail(KC_EARG, "group_first_pct: 0..100");
      c->group_first_pct = (int)value;
    }
    else if (k == "full_fused") c->full_fused = value ? 1 : 0;
    else if (k == "select_cand") {
      if (value < 0 || value > 2) fail(KC_EARG, "select_cand: 0 auto, 1 on, 2 off");
      c->select_cand = (int)value;
    }
    else if (k == "k_policy") c->k_policy = (int)value;
    else if (k == "tlb_ahead") c->tlb_ahead = (int)value;
    else if (k == "dbg_ctr_race") c->dbg_ctr_race = value ? 1 : 0;
    else if (k == "flow_join") c->flow_join = value ? 1 : 0;
    else if (k == "recall_tma") c->recall_tma = value ? 1 : 0;
    else if (k == "recall_lean") c->recall_lean = (int)std::max<int64_t>(-1, std::min<int64_t>(1, value));
    else if (k == "recall_dbg") c->recall_dbg = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
    else if (k == "tc_grid") c->tc_grid = (int)std::max<int64_t>(0, std::min<int64_t>(4, value));
    else if (k == "score_mma") c->score_mma = (int)std::max<int64_t>(0, std::min<int64_t>(3, value));
    else if (k == "cand_force_fallback") c->cand_force_fallback = value ? 1 : 0;
    else if (k == "consume") {
      if (value < 0 || value > 2) fail(KC_EARG, "consume: 0 off, 1 MHA, 2 every supported shape");
      c->consume = (int)value;
    }



    else if (k == "consume_dbg") c->consume_dbg = value ? 1 : 0;
    else if (k == "select_cached") c->select_cached = value ? 1 : 0;
    else if (k == "consume_recall") c->consume_recall = value < 0 ? -1 : (value ? 1 : 0);
    else if (k == "flow_recall_ctas") {
      if (value < 0) fail(KC_EARG, "flow_recall_ctas must be >= 0 (0 = auto)");
      c->flow_recall_ctas = (int)value;
    }
    else if (k == "consume_ctas") {
      if (value < 0) fail(KC_EARG, "consume_ctas must be >= 0 (0 = auto)");
      c->consume_ctas = (int)value;
    }
    else if (k == "score_groups") {
      if (value < 0) fail(KC_EARG, "score_groups must be >= 0 (0 = auto)");
      c->score_groups = (int)value;
    }
    else fail(KC_EARG, "unknown tuning key '" + k + "'");
  });
}

int kc_profile(kc_cache* c, int enable) {
  return guarded([&] {
    set_dev(c);
    CK(cudaStreamSynchronize(c->main_st));
    CK(cudaStreamSynchronize(c->side_st));
    c->prof_on = enable != 0;
    // enable: 1 = every kind; otherwise (enable >> 1) is a kind bit mask
    c->prof_mask = enable == 1 ? 7 : (enable >> 1) & 7;
    for (auto& v : c->prof) v.clear();
    c->prof_used = 0;
  });
}

int kc_profile_read(kc_cache* c, const char* kernel, double* total_ms, uint64_t* launches) {
  return guarded([&] {
    const std::string k = kernel ? kernel : "";
    const int kind = k == "score" ? 0 : k == "select" ? 1 : k == "recall" ? 2 : -1;
    if (kind < 0) fail(KC_EARG, "kc_profile_read: kernel must be score, select or recall");
    set_dev(c);
    double total = 0.0;
    for (auto& pr : c->prof[kind]) {
      CK(cudaEventSynchronize(pr.second));
      float ms = 0.0f;
      CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
      total += ms;
    }
    *total_ms = total;
    *launches = c->prof[kind].size();
  });
}

int kc_profile_span(kc_cache* c, const char* kernel, uint64_t i, double* t0, double* t1) {
  return guarded([&] {
    const std::string k = kernel ? kernel : "";
    const int kind = k == "score" ? 0 : k == "select" ? 1 : k == "recall" ? 2 : -1;
    if (kind < 0 || i >= c->prof[kind].size() || c->prof_pool.empty())
      fail(KC_EARG, "kc_profile_span: bad kernel or index");
    set_dev(c);
    CK(cudaEventSynchronize(c->prof[kind][i].second));
    float a = 0.0f, b = 0.0f;
    CK(cudaEventElapsedTime(&a, c->prof_pool[0], c->prof[kind][i].first));
    CK(cudaEventElapsedTime(&b, c->prof_pool[0], c->prof[kind][i].second));
    *t0 = a;
    *t1 = b;
  });
}

int kc_profile_launch(kc_cache* c, const char* kernel, uint64_t i, double* ms) {
  return guarded([&] {
    const std::string k = kernel ? kernel : "";
    const int kind = k == "score" ? 0 : k == "select" ? 1 : k == "recall" ? 2 : -1;
    if (kind < 0 || i >= c->prof[kind].size()) fail(KC_EARG, "kc_profile_launch: bad kernel or index");
    set_dev(c);
    CK(cudaEventSynchronize(c->prof[kind][i].second));
    float t = 0.0f;
    CK(cudaEventElapsedTime(&t, c->prof[kind][i].first, c->prof[kind][i].second));
    *ms = t;
  });
}

int kc_debug_read(kc_cache* c, const char* what, void* out, uint64_t bytes) {
  return guarded([&] {
    const std::string w = what ? what : "";
    const DevBuf* src = w == "consume" ? &c->cons_dbg : w == "logits0" ? &c->logits : w == "logits1" ? &c->logits_b
                         : w == "partials0" ? &c->partials : nullptr;
    if (!src || !out) fail(KC_EARG, "kc_debug_read: unknown probe");
    set_dev(c);
    CK(cudaDeviceSynchronize());
    if (!src->p) fail(KC_ESTATE, "kc_debug_read: probe buffer not allocated");
    CK(cudaMemcpy(out, src->p, std::min<uint64_t>(bytes, src->bytes), cudaMemcpyDeviceToHost));
  });
}

int kc_score_chunk_plan(uint64_t s, uint64_t rows, uint64_t group, int64_t* chunk) {
  return guarded([&] {
    if (!chunk || s == 0 || rows == 0 || group == 0) fail(KC_EARG, "kc_score_chunk_plan: bad argument");
    *chunk = kc::score_pick_chunk((int)s, (int)rows, 0, (int)group);
  });
}

int kc_prefill_attention(const float* q, const float* k, const float* v, uint64_t s, uint64_t n_heads,
                         uint64_t head_dim, float* out, int device) {
  return guarded([&] {
    if (!q || !k || !v || !out) fail(KC_EARG, "kc_prefill_attention: null argument");
    if (n_heads == 0 || head_dim == 0) fail(KC_ESHAPE, "prefill_attention: cols must divide into heads");
    if (s == 0) return;
    if (s > (1ull << 30) || n_heads * head_dim > (1ull << 20)) fail(KC_ESHAPE, "prefill_attention: too large");
    if (device >= 0) CK(cudaSetDevice(device));  // < 0: the calling thread's current device
    const size_t bytes = checked_mul({s, n_heads, head_dim, 4});
    float* buf = nullptr;
    CK(cudaMalloc(&buf, 4 * bytes));
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemcpyAsync(buf, q, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)buf + bytes, k, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)buf + 2 * bytes, v, bytes, cudaMemcpyHostToDevice, st);
    float* dout = (float*)((char*)buf + 3 * bytes);
    if (e == cudaSuccess &&
        !kc::prefill_attention_launch(buf, (float*)((char*)buf + bytes), (float*)((char*)buf + 2 * bytes), dout,
                                      (int)s, (int)n_heads, (int)head_dim, st))
      e = cudaErrorInvalidValue;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (st) cudaStreamDestroy(st);
    cudaFree(buf);
    if (e != cudaSuccess) fail(KC_ECUDA, std::string("prefill_attention: ") + cudaGetErrorString(e));
  });
}

int kc_prefill_attention_device(const float* q, const float* k, const float* v, uint64_t s, uint64_t n_heads,
                                uint64_t head_dim, float* out, void* stream) {
  return guarded([&] {
    if (!q || !k || !v || !out) fail(KC_EARG, "kc_prefill_attention_device: null argument");
    if (n_heads == 0 || head_dim == 0) fail(KC_ESHAPE, "prefill_attention: cols must divide into heads");
    if (s == 0) return;
    if (s > (1ull << 30) || n_heads * head_dim > (1ull << 20)) fail(KC_ESHAPE, "prefill_attention: too large");
    if (!kc::prefill_attention_launch(q, k, v, out, (int)s, (int)n_heads, (int)head_dim, (cudaStream_t)stream))
      fail(KC_ESHAPE, "prefill_attention: head_dim too large for the shared-memory tiles");
    CK(cudaGetLastError());
  });
}

int kc_arg_topk(const float* values, uint64_t n, uint64_t k, uint32_t* out, uint64_t* count) {
  return guarded([&] {
    if (k == 0) fail(KC_EARG, "arg_topk: k must be >= 1");
    const uint64_t m = std::min(k, n);
    if (count) *count = m;
    if (n == 0) return;
    if (n > (1ull << 31)) fail(KC_EARG, "arg_topk: too many values");
    float* dv = nullptr;
    uint32_t *dk = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dv, n * 4));
    CK(cudaMalloc(&dk, n * 4));
    CK(cudaMalloc(&dout, m * 4));
    CK(cudaMemcpy(dv, values, n * 4, cudaMemcpyHostToDevice));
    kc::arg_topk_launch(dv, (int)n, (int)m, dk, dout, nullptr);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, m * 4, cudaMemcpyDeviceToHost);
    cudaFree(dv);
    cudaFree(dk);
    cudaFree(dout);
    if (e != cudaSuccess) fail(KC_ECUDA, std::string("arg_topk: ") + cudaGetErrorString(e));
  });
}

int kc_fill_uniform(void* dst, int dtype, uint64_t n, uint64_t seed, uint64_t offset, float lo,
                    float hi, void* stream) {
  return guarded([&] {
    dtype_size(dtype);
    if (n == 0) return;
    kc::fill_uniform_launch(dst, dtype, n, seed, offset, lo, hi, (cudaStream_t)stream);
    CK(cudaGetLastError());
  });
}

}  // extern "C"

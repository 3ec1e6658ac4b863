// perf_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference cost model
// (proj/core/src/perf_model.cpp, proj/core/include/kcache/perf_model.hpp),
// compiled in place from /root/reference by oracle/Makefile into
// oracle/_ref/libkcache_perf.so. tests/test_perf_model_cpu.py loads the
// measured B200 profile (profiles/b200_profile.json, written by
// tools/b200_profile.py in the reference's load_profile format) through the
// reference's own load_profile and checks decode_transfer_check /
// project_run against the measured C5 crossover and prefill_overlap_check
// against the measured prefill V offload. No reference source is
// copied into this repository.
#include <cstring>
#include <exception>
#include <string>

#include "kcache/perf_model.hpp"

using namespace kcache;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* ref_perf_last_error() { return g_err.c_str(); }

// profile fields out: flops, bw_gpu, bw_h2d, bw_d2h, fast_capacity
int ref_perf_load_profile(const char* name_or_path, double* fields) {
  try {
    const HardwareProfile p = resolve_profile(name_or_path);
    fields[0] = p.flops;
    fields[1] = p.bw_gpu;
    fields[2] = p.bw_h2d;
    fields[3] = p.bw_d2h;
    fields[4] = p.fast_capacity;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// decode_transfer_check (perf_model.hpp:98): out = {beneficial, ratio, threshold}
int ref_perf_transfer_check(const char* profile, unsigned long long s, unsigned long long top_n, double* out) {
  try {
    const TransferCheck c = decode_transfer_check(s, top_n, resolve_profile(profile));
    out[0] = c.beneficial ? 1.0 : 0.0;
    out[1] = c.ratio;
    out[2] = c.threshold;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// prefill_overlap_check (perf_model.hpp:87-89, perf_model.cpp:147-162, the
// paper's Eq. 1-2): out = {holds, compute_time, transfer_time, lhs, rhs}
int ref_perf_prefill_check(const char* profile, unsigned long long s, unsigned long long d, unsigned long long b,
                           unsigned long long bytes, double* out) {
  try {
    const OverlapCheck c = prefill_overlap_check(s, d, b, bytes, resolve_profile(profile));
    out[0] = c.holds ? 1.0 : 0.0;
    out[1] = c.compute_time;
    out[2] = c.transfer_time;
    out[3] = c.lhs;
    out[4] = c.rhs;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// project_run (perf_model.hpp:130-133): out = {baseline_step, kcache_step,
// baseline_tok/s, kcache_tok/s, speedup, h2d_time_per_offloaded_layer}
int ref_perf_project_run(const char* profile, unsigned long long batch, unsigned long long seq_len,
                         unsigned long long d_model, unsigned long long n_heads, unsigned long long head_dim,
                         unsigned long long n_layers, unsigned long long ffn_hidden, unsigned long long top_n,
                         unsigned long long resident, int overlap_h2d, double* out) {
  try {
    ProjectShape shape;
    shape.decode.batch = batch;
    shape.decode.seq_len = seq_len;
    shape.decode.d_model = d_model;
    shape.decode.n_heads = n_heads;
    shape.decode.head_dim = head_dim;
    shape.decode.bytes_per_element = 2;
    shape.n_layers = n_layers;
    shape.ffn_hidden = ffn_hidden;
    const RunProjection r = project_run(shape, top_n, resident, resolve_profile(profile), overlap_h2d != 0);
    out[0] = r.baseline_step_time;
    out[1] = r.kcache_step_time;
    out[2] = r.baseline_tokens_per_s;
    out[3] = r.kcache_tokens_per_s;
    out[4] = r.speedup;
    out[5] = r.h2d_time_per_offloaded_layer;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"

// kc_gather.hpp -- host-side V recall for offloaded layers: a worker pool
// that compacts the selected V rows out of the pinned host arena into a
// contiguous pinned staging block, which one cudaMemcpyAsync then moves to
// HBM at full DMA rate.
//
// Why it exists: zero-copy SM loads of scattered 256-B rows cost one GPU
// page walk per row (tools/tlb_probe.cu), while a
// contiguous DMA needs none. This is the reference's gather_v
// (proj/core/src/kv_cache.cpp:150-187) done where the slow tier lives.
// Measured on the 16-vCPU box the host side is the limit (20-26 GB/s), so it
// is an option (recall_mode 2 / 3), not the default.
#pragma once

#include <immintrin.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace kc {

class GatherPool {
 public:
  explicit GatherPool(int n_workers) {
    for (int i = 0; i < n_workers; ++i) threads_.emplace_back([this, i] { worker(i); });
  }
  ~GatherPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return (int)threads_.size() + 1; }

  // Run fn(part, parts) on every worker plus the calling thread; returns when
  // all parts are done.
  void run(const std::function<void(int, int)>& fn) {
    const int parts = size();
    job_ = &fn;
    done_.store(0);
    {
      std::lock_guard<std::mutex> lk(m_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    fn(parts - 1, parts);
    while (done_.load(std::memory_order_acquire) < parts - 1) _mm_pause();
  }

 private:
  void worker(int i) {
    uint64_t seen = 0;
    for (;;) {
      // spin briefly (layers arrive every few hundred us), then block
      int spins = 0;
      while (gen_.load(std::memory_order_acquire) == seen && spins < 20000) {
        _mm_pause();
        ++spins;
      }
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load();
      if (stop_) return;
      (*job_)(i, (int)threads_.size() + 1);
      done_.fetch_add(1, std::memory_order_release);
    }
  }

  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> done_{0};
  const std::function<void(int, int)>* job_ = nullptr;
  bool stop_ = false;
};

// One layer's compaction: for slot row r and entry j, copy row_bytes from
// src + r*slot_bytes + idx[r*nc + j]*row_bytes to dst + (r*nc + j)*row_bytes.
struct GatherJob {
  GatherPool* pool;
  const char* src;
  size_t slot_bytes;
  size_t row_bytes;
  const uint32_t* idx;  // pinned host copy of the selection
  uint64_t rows;
  uint64_t nc;
  char* dst;            // pinned host staging
};

inline void gather_rows_host(const GatherJob& j, int part, int parts) {
  const uint64_t total = j.rows * j.nc;
  const uint64_t per = (total + parts - 1) / parts;
  const uint64_t e0 = per * part;
  const uint64_t e1 = e0 + per < total ? e0 + per : total;
  constexpr uint64_t kAhead = 8;
  for (uint64_t e = e0; e < e1; ++e) {
    if (e + kAhead < e1) {
      const uint64_t f = e + kAhead;
      const char* p = j.src + (f / j.nc) * j.slot_bytes + (size_t)j.idx[f] * j.row_bytes;
      for (size_t off = 0; off < j.row_bytes; off += 64) _mm_prefetch(p + off, _MM_HINT_T0);
    }
    const uint64_t r = e / j.nc;
    std::memcpy(j.dst + e * j.row_bytes, j.src + r * j.slot_bytes + (size_t)j.idx[e] * j.row_bytes,
                j.row_bytes);
  }
}

// cudaLaunchHostFunc entry: owns and frees the job.
inline void gather_host_fn(void* p) {
  GatherJob* j = static_cast<GatherJob*>(p);
  const GatherJob job = *j;
  delete j;
  job.pool->run([&](int part, int parts) { gather_rows_host(job, part, parts); });
}

}  // namespace kc

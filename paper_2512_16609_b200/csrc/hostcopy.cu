// Host-side memcpy over a persistent worker pool (no device code).
//
// process_stream (reference pipeline.py:232-308) hands every frame to the pipeline as a
// separate host array: its bytes are copied into pinned staging before the H2D copy,
// and every output frame is copied out of pinned staging into a fresh array for the
// sink.  One memcpy per 1080p frame (6.2 MB) runs at a single core's copy bandwidth,
// which bounds the stream at ~1,400 fps; Python thread-pool dispatch per frame costs
// more than it saves at that size.  dhz_host_copy splits a copy over a pool of native
// threads that stay parked between calls (a call costs a wake-up, not a thread start).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/dehaze_b200.h"

namespace {

class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }

  int workers() const { return (int)threads_.size(); }

  void copy(char* dst, const char* src, size_t bytes, int parts) {
    std::lock_guard<std::mutex> call(call_);  // one job at a time
    {
      std::unique_lock<std::mutex> g(m_);
      done_.wait(g, [&] { return busy_ == 0; });  // no worker still inside the last job
      dst_ = dst;
      src_ = src;
      bytes_ = bytes;
      parts_ = parts;
      next_.store(0);
      left_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    const int mine = run_parts();  // the caller takes parts too
    std::unique_lock<std::mutex> g(m_);
    left_ -= mine;
    done_.wait(g, [&] { return left_ == 0 && busy_ == 0; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int n = (int)std::min(15u, hw > 1 ? hw - 1 : 0u);
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }

  // parts of the current job (fields stable while busy_ > 0 or the caller runs)
  int run_parts() {
    int done = 0;
    for (;;) {
      const int p = next_.fetch_add(1);
      if (p >= parts_) break;
      const size_t a = bytes_ * (size_t)p / (size_t)parts_, b = bytes_ * (size_t)(p + 1) / (size_t)parts_;
      std::memcpy(dst_ + a, src_ + a, b - a);
      ++done;
    }
    return done;
  }

  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        ++busy_;
      }
      const int done = run_parts();
      {
        std::lock_guard<std::mutex> g(m_);
        left_ -= done;
        --busy_;
      }
      done_.notify_all();
    }
  }

  std::vector<std::thread> threads_;
  std::mutex call_, m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int parts_ = 0;
  std::atomic<int> next_{0};
  int left_ = 0;
  int busy_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

}  // namespace

extern "C" {

int dhz_host_copy(void* dst, const void* src, size_t bytes, int nthreads) {
  if (bytes == 0) return DHZ_OK;
  if (!dst || !src) return DHZ_E_INVALID;
  CopyPool& pool = CopyPool::get();
  // >= 1 MiB per part; never more parts than threads (workers + the caller)
  const size_t by_size = std::max<size_t>(1, bytes >> 20);
  int parts = (int)std::min<size_t>(by_size, (size_t)std::max(1, nthreads));
  parts = std::min(parts, pool.workers() + 1);
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return DHZ_OK;
  }
  pool.copy(static_cast<char*>(dst), static_cast<const char*>(src), bytes, parts);
  return DHZ_OK;
}

}  // extern "C"

// fn(i) for i < n on the host's threads (chunks of up to 64 indices; one
// thread when n < 2 x minPerThread).  Host-side data parallelism of the sweep pipeline
// (speculated configurations, batch staging, merges).  The worker threads
// persist for the process (thread creation would cost more than a sweep's
// host phases); a call that finds the pool busy (another thread's
// parallelFor) runs inline.
//
// Wake-ups go through a futex on the generation word, not a condition
// variable: with the condvar broadcast the sleepers woke only once the
// caller had finished every chunk alone (measured here: a 229-job sweep
// report ran 2.4 ms on one thread of eight).  Workers also spin briefly on
// the word after a run, so the back-to-back parallel phases of a sweep find
// them awake.
#pragma once

#include <linux/futex.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace hgrdgpu {

class HostPool {
public:
  static HostPool &get() {
    static HostPool pool;
    return pool;
  }
  size_t threads() const { return workers_.size() + 1; }

  // Runs body(i) for i < n with the workers; false when the pool is busy.
  bool run(size_t n, const std::function<void(size_t)> &body) {
    std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
    if (!busy.owns_lock())
      return false;
    body_ = &body;
    n_ = n;
    // chunks small enough for every thread to get several
    chunk_ = std::max<size_t>(1, std::min<size_t>(64, n / (4 * threads())));
    next_.store(0, std::memory_order_relaxed);
    active_.store(static_cast<int>(workers_.size()), std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    futex(FUTEX_WAKE_PRIVATE, 0x7fffffff);
    drain();
    // every worker has seen this generation before body goes out of scope
    for (int spin = 0; active_.load(std::memory_order_acquire) != 0; ++spin)
      if (spin > 64)
        std::this_thread::yield();
    body_ = nullptr;
    return true;
  }

private:
  HostPool() {
    const size_t hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    for (size_t t = 1; t < hw; ++t)
      workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    stop_.store(true, std::memory_order_release);
    gen_.fetch_add(1, std::memory_order_release);
    futex(FUTEX_WAKE_PRIVATE, 0x7fffffff);
    for (auto &t : workers_)
      t.join();
  }
  long futex(int op, uint32_t val) {
    return syscall(SYS_futex, reinterpret_cast<uint32_t *>(&gen_), op, val, nullptr, nullptr, 0);
  }
  void drain() {
    for (size_t b; (b = next_.fetch_add(chunk_)) < n_;)
      for (size_t i = b; i < std::min(n_, b + chunk_); ++i)
        (*body_)(i);
  }
  void loop() {
    uint32_t seen = 0;
    for (;;) {
      uint32_t g;
      // spin briefly after a run (the sweep's next phase), then sleep
      for (int spin = 0; (g = gen_.load(std::memory_order_acquire)) == seen; ++spin) {
        if (spin < 2000)
          std::this_thread::yield();
        else
          futex(FUTEX_WAIT_PRIVATE, seen);
      }
      seen = g;
      if (stop_.load(std::memory_order_acquire))
        return;
      drain();
      active_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }

  std::vector<std::thread> workers_;
  std::mutex busy_;
  std::atomic<uint32_t> gen_{0};
  std::atomic<bool> stop_{false};
  const std::function<void(size_t)> *body_ = nullptr;
  size_t n_ = 0, chunk_ = 64;
  std::atomic<size_t> next_{0};
  std::atomic<int> active_{0};
};

template <class F> void parallelFor(size_t n, F &&fn, size_t minPerThread = 256) {
  if (n < 2 * minPerThread || std::thread::hardware_concurrency() <= 1) {
    for (size_t i = 0; i < n; ++i)
      fn(i);
    return;
  }
  const std::function<void(size_t)> body = [&](size_t i) { fn(i); };
  if (!HostPool::get().run(n, body))
    for (size_t i = 0; i < n; ++i)
      fn(i);
}

} // namespace hgrdgpu

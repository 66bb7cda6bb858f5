// fn(i) for i < n on the host's threads (chunks of up to 64 indices; one
// thread when n < 2 x minPerThread).  Host-side data parallelism of the sweep pipeline
// (speculated configurations, batch staging, merges).  The worker threads
// persist for the process (thread creation would cost more than a sweep's
// host phases); a call that finds the pool busy (another thread's
// parallelFor) runs inline.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstddef>
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
    {
      std::lock_guard<std::mutex> lk(mu_);
      body_ = &body;
      n_ = n;
      // chunks small enough for every thread to get several
      chunk_ = std::max<size_t>(1, std::min<size_t>(64, n / (4 * threads())));
      next_ = 0;
      active_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return active_ == 0; });
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
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto &t : workers_)
      t.join();
  }
  void drain() {
    for (size_t b; (b = next_.fetch_add(chunk_)) < n_;)
      for (size_t i = b; i < std::min(n_, b + chunk_); ++i)
        (*body_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_)
          return;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0)
        done_.notify_one();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex busy_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t)> *body_ = nullptr;
  size_t n_ = 0, chunk_ = 64;
  std::atomic<size_t> next_{0};
  size_t active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
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

// fn(i) for i < n on up to the hardware's threads (chunks of 64 indices,
// one thread when n is small).  Host-side data parallelism of the sweep
// pipeline (speculated configurations, batch staging, merges).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <thread>
#include <vector>

namespace hgrdgpu {

template <class F> void parallelFor(size_t n, F &&fn, size_t minPerThread = 256) {
  const size_t hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const size_t nt = std::min(hw, (n + minPerThread - 1) / minPerThread);
  if (nt <= 1) {
    for (size_t i = 0; i < n; ++i)
      fn(i);
    return;
  }
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t b; (b = next.fetch_add(64)) < n;)
      for (size_t i = b; i < std::min(n, b + 64); ++i)
        fn(i);
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nt; ++t)
    pool.emplace_back(work);
  work();
  for (auto &t : pool)
    t.join();
}

} // namespace hgrdgpu

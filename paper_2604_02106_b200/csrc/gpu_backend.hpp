// The product's LaunchBackend: the host front end (csrc/host) driving the
// B200 race-check stage of one context through the C ABI, plus the pool of
// worker contexts a sweep spreads its configurations over.
#pragma once

#include "hgrd_gpu.h"
#include "host.hpp"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace hgrdgpu {

hgrd_gpu_ctx *sweepWorker(hgrd_gpu_ctx *c, int i); // ctx.cu
bool setTiming(hgrd_gpu_ctx *c, bool on);            // ctx.cu
void setError(hgrd_gpu_ctx *c, const std::string &m); // ctx.cu (hgrd_gpu_last_error)

class GpuBackend final : public LaunchBackend {
public:
  explicit GpuBackend(hgrd_gpu_ctx *c) : c_(c) {}
  int reset() override { return hgrd_gpu_buffers_reset(c_); }
  int alloc(int64_t elems, int32_t *handle) override {
    return hgrd_gpu_buffer_alloc(c_, elems, handle);
  }
  int write(int32_t h, int64_t off, int64_t n, const int64_t *src) override {
    return hgrd_gpu_buffer_write(c_, h, off, n, src);
  }
  int read(int32_t h, int64_t off, int64_t n, int64_t *dst) override {
    return hgrd_gpu_buffer_read(c_, h, off, n, dst);
  }
  int checkLaunch(const hgrd_gpu_launch &l, hgrd_gpu_result &r) override {
    return hgrd_gpu_check_launch(c_, &l, &r);
  }
  int checkBatch(const hgrd_gpu_batch_launch *b, uint32_t n, hgrd_gpu_result *r) override {
    return hgrd_gpu_check_batch(c_, b, n, r);
  }
  bool hasBatch() const override { return batch_; }
  void setBatch(bool on) { batch_ = on; }
  std::string lastError() override { return hgrd_gpu_last_error(c_); }

private:
  hgrd_gpu_ctx *c_;
  bool batch_ = true;
};

// Sweeps check their configurations' launches in batches (one GPU round
// trip per batch) unless HGRD_SWEEP_BATCH=0 selects the per-launch path
// spread over worker contexts.
inline bool sweepBatched() {
  const char *e = std::getenv("HGRD_SWEEP_BATCH");
  return !e || std::atoi(e) != 0;
}

// Configurations of a sweep are independent runs: they are spread over
// worker contexts (own streams and buffers on the same GPU, one host thread
// each) so the small launches of a sweep overlap instead of queueing behind
// each other's host round trips (HGRD_SWEEP_WORKERS, default 8).  Per-check
// event timing is off while the pool lives.
struct SweepWorkers {
  hgrd_gpu_ctx *ctx;
  int n;
  bool timing;
  std::vector<std::unique_ptr<GpuBackend>> bes;

  explicit SweepWorkers(hgrd_gpu_ctx *c) : ctx(c) {
    const char *env = std::getenv("HGRD_SWEEP_WORKERS");
    n = std::max(1, env ? std::atoi(env) : 8);
    bes.resize(static_cast<size_t>(n));
    timing = setTiming(ctx, false);
  }
  ~SweepWorkers() { setTiming(ctx, timing); }
  SweepWorkers(const SweepWorkers &) = delete;
  SweepWorkers &operator=(const SweepWorkers &) = delete;

  LaunchBackend *get(int i) {
    if (i < 0 || i >= n)
      return nullptr;
    hgrd_gpu_ctx *w = sweepWorker(ctx, i);
    if (!w)
      return nullptr;
    if (i > 0)
      setTiming(w, false); // worker contexts only run sweeps
    if (!bes[static_cast<size_t>(i)]) {
      bes[static_cast<size_t>(i)] = std::make_unique<GpuBackend>(w);
      bes[static_cast<size_t>(i)]->setBatch(sweepBatched());
    }
    return bes[static_cast<size_t>(i)].get();
  }
  std::function<LaunchBackend *(int)> getter() {
    return [this](int i) { return get(i); };
  }
};

} // namespace hgrdgpu

// Block-private partition proof (see affine.cpp).
#pragma once

#include "hgrd_gpu.h"

#include <cstdint>
#include <vector>

namespace hgrdgpu {

// Per site: 1 when no element its buffer holds can be reached from two
// MiniCU blocks of this launch (so INTER-BLOCK pairs on it are impossible).
std::vector<uint8_t> blockPrivateSites(const hgrd_gpu_launch &L);

// Per site: c when the site is a load whose index is always the thread's
// dense id plus the constant c (t = blockLin * tpb + threadLin, reference
// src/oracle.cpp:443-460) — one contiguous stream per fused iteration,
// staged into shared memory by bulk copies; kNoStream otherwise.
constexpr int64_t kNoStream = INT64_MIN;
std::vector<int64_t> streamSites(const hgrd_gpu_launch &L);

} // namespace hgrdgpu

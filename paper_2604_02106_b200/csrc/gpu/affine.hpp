// Block-private partition proof (see affine.cpp).
#pragma once

#include "hgrd_gpu.h"

#include <cstdint>
#include <vector>

namespace hgrdgpu {

// Per site: 1 when no element its buffer holds can be reached from two
// MiniCU blocks of this launch (so INTER-BLOCK pairs on it are impossible).
std::vector<uint8_t> blockPrivateSites(const hgrd_gpu_launch &L);

} // namespace hgrdgpu

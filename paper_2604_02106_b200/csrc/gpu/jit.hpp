// NVRTC specialisation of the race-check kernels (see jit.cpp).
#pragma once

#include "hgrd_gpu.h"

#include <map>
#include <string>
#include <vector>

namespace hgrdgpu {
namespace jit {

// k_expand_par, k_fused<256,4> / <256,16> / <256,8>, k_expand_seq, k_fused<256,12>
enum Variant {
  kExpandPar = 0,
  kFusedNarrow = 1,
  kFusedWide = 2,
  kFusedMid = 3,
  kExpandSeq = 4,
  kFused12 = 5,
  kVariants = 6
};

// Per kernel parameter: its buffer's element count (0: none, every access
// traps) and global element base, folded into the generated accesses.
struct JitParam {
  int64_t size;
  uint64_t base;
};

struct Cache;
Cache *create();
void destroy(Cache *c);
// The specialised kernel `v` for this launch's code and constants (compiled
// on first use, cached).  Returns nullptr (and err) when NVRTC is
// unavailable or the compile fails; callers then use the interpreter.
// `rec[s]`: bit 0: site s produces race-check records (written buffer);
// bit 1: its buffer may be reached from two blocks (ownership exchange);
// bit 2: a streamed load (affine.hpp streamSites; k_fused stages its values).
const void *get(Cache *c, const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                const std::vector<JitParam> &params, Variant v, std::string &err);
// lowOccupancy: the k_fused variant keeps at most two CTAs per SM (x12, x16)
std::string generate(const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                     const std::vector<JitParam> &params, bool seq = false,
                     bool lowOccupancy = false);
// Compile without loading (no GPU needed): cubin size, 0 and err on failure.
size_t compileOnly(const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                   const std::vector<JitParam> &params, Variant v, std::string &err);
double compileMs(const Cache *c);
int compiles(const Cache *c);

} // namespace jit
} // namespace hgrdgpu

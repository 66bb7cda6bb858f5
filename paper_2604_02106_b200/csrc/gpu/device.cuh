// Device-side data layout of the race-check stage (sm_100a).
//
// HBM layout per launch (all device-resident, owned by hgrd_gpu_ctx):
//   buffers      int64[elems] per allocation (reference buffers_, :789)
//   blob         code | sites | params | reg_init | conflict masks  (one H2D)
//   keys/vals    packed access records: u64 key + u32 (site,seq)
//   keySeg       u32 per race key (locA, locB, kind): first segment start
//   races        hgrd_gpu_race[] output
//
// Packed record key (high -> low bits), widths chosen per launch:
//   element | block | blockPhase | warp | warpPhase | lane
// element = flat index over the buffers the launch writes (handle order,
// so element order == reference (handle, index) order).  Sorting by the
// key makes the reference's element groups contiguous (:733-735) and,
// inside them, the (block, blockPhase) and (block, blockPhase, warp,
// warpPhase) groups on which the pair rule (:750-769) reduces to
// "two distinct ids at the right level" — see detect.cuh.
#pragma once

#include "hgrd_gpu.h"

#if !defined(__CUDACC_RTC__)
#include <cstdint>
#endif

namespace hgrdgpu {
namespace dev {

constexpr int kMaxRegs = 64;    // PARALLEL per-lane register file
constexpr int kMaxSites = 64;   // summary detector site masks (u64)
constexpr int kLaneBuf = 16;    // records buffered per lane per batch
constexpr uint32_t kChunk = 4096; // records reserved per warp refill
// fused records (r0 seq field) and their thread << 20 | seq orders; the
// general path's record values are site << KeyLayout::bS | seq instead
constexpr int kSeqBits = 20;
constexpr uint32_t kSeqMask = (1u << kSeqBits) - 1;
constexpr int kMaxSiteId = 4095;

enum CounterFlags : uint32_t {
  kFlagCapacity = 1u,   // record buffer too small
  kFlagPhase = 2u,      // a phase counter exceeded its key field
  kFlagSeqSite = 4u,    // seq >= 2^KeyLayout::bS
  kFlagAbort = 8u,      // step budget exhausted
  kFlagLockSet = 16u,   // lock-set scratch overflow (pairwise)
  kFlagSegment = 32u,   // pairwise: 2^32 or more events
  kFlagOps = 64u        // sync-op buffer too small
};

struct ParamDev {
  int64_t *ptr;      // device buffer base (nullptr: scalar / unallocated)
  int64_t size;      // elements
  int32_t handle;    // -1 when unbound
  int32_t written;   // 1 + index among the buffers the launch writes, 0 if read-only
  uint64_t elemBase; // flat element base (written buffers only)
};

struct SiteDev {
  int32_t param;
  int32_t loc;
  uint8_t kind, aop, scope, record; // record: access lands in a written buffer
  uint8_t own;  // fused path: the buffer may be reached from two blocks (ownership exchange)
  uint8_t pad0, pad1, pad2;
};

struct KeyLayout {
  int bL, bQ, bW, bP, bB, bE;
  int bS; // record value = site << bS | seq (32 - bits of the site count)
  int shQ, shW, shP, shB, shE;
  int total;
  uint64_t sentinel; // all-ones in `total` bits: never a valid key
};

struct Counters {
  unsigned long long steps;
  unsigned long long instances;
  unsigned long long records;   // real records written (no sentinels)
  unsigned long long traps;
  unsigned long long cursor;    // record slots handed out (incl. padding)
  unsigned long long nOps;
  unsigned int maxBp, maxWp;
  unsigned int flags;
  int abortStmt;
  unsigned int nRaces;
  unsigned int candCount;
  unsigned int doneCtas; // fused kernel: CTAs finished (last one finalises)
  unsigned int pad;
};

// Division by a launch-invariant 32-bit divisor: one mul.hi + shifts
// (Granlund-Montgomery); exact for every 32-bit dividend.
struct FastDiv {
  uint32_t d = 1, m = 1;
  int s1 = 0, s2 = 0;
#if !defined(__CUDACC_RTC__)
  static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d;
    int l = 0;
    while ((uint64_t(1) << l) < d)
      ++l;
    f.m = static_cast<uint32_t>(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
    f.s1 = l < 1 ? l : 1;
    f.s2 = l > 1 ? l - 1 : 0;
    return f;
  }
#endif
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#if defined(__CUDA_ARCH__)
    const uint32_t t = __umulhi(m, n);
#else
    const uint32_t t = static_cast<uint32_t>((uint64_t(m) * n) >> 32);
#endif
    return (t + ((n - t) >> s1)) >> s2;
  }
};

struct LaunchDev {
  const hgrd_gpu_insn *code;
  const SiteDev *sites;
  const ParamDev *params;
  const int64_t *regInit;
  const uint64_t *confInter; // per site: sites it can race with across blocks
  const uint64_t *confIntra; // ... within a block
  const uint64_t *locMask;   // per loc id: sites at that loc
  int nCode, nRegs, nSites, nParams, nLocs;
  int64_t grid[3], block[3];
  int64_t ws, tpb, nThreads, nBlocks;
  int64_t stepBudget;
  KeyLayout kl;
  uint64_t *keys;
  uint32_t *vals;
  uint64_t capacity;
  uint32_t chunk;             // records reserved per warp refill
  Counters *ctr;
  // SEQUENTIAL extras
  int64_t *seqRegs;          // nRegs scratch
  hgrd_gpu_trap *traps;      // first trapCap traps
  uint32_t trapCap;
  // lock idioms (pairwise): per-thread sync ops
  int64_t *opIndex;          // per op: element index
  int32_t *opMeta;           // per op: kind | scope << 4 | handle << 8
  int32_t *opSeq;
  uint64_t opCap;
  uint64_t *opStart;         // nThreads + 1
  uint32_t opStride;         // PARALLEL lock launches: ops at thread * opStride (no opStart)
  // pass 2 of the fused path: only elements the ownership table marks MULTI
  const uint32_t *ownerFilter;
  uint32_t ownerMultiTag;
  uint32_t *interTab;        // INTER summary mode: (element, site) block sets
  int nSitesTab;
  uint32_t *interLo, *interHi; // sharded INTER summary: (element, site) min / max block + 1
  int64_t threadBase, threadEnd; // k_expand_par: dense thread range (a shard of the launch)
  const uint64_t *targets;   // witness mode: only these elements
  int nTargets;
  // 32-bit thread identity (nThreads < 2^32): tpb, bx, bx*by, gx, gx*gy, ws
  bool small;
  FastDiv dTpb, dBx, dBxBy, dGx, dGxGy, dWs;
};

__host__ __device__ inline int64_t wrapAdd(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}

// reference applyBinOp, src/oracle.cpp:179-209, over wrapping int64
__device__ __forceinline__ int64_t applyBin(int op, int64_t l, int64_t r) {
  switch (op) {
  case HGRD_ADD:
    return wrapAdd(l, r);
  case HGRD_SUB:
    return static_cast<int64_t>(static_cast<uint64_t>(l) - static_cast<uint64_t>(r));
  case HGRD_MUL:
    return static_cast<int64_t>(static_cast<uint64_t>(l) * static_cast<uint64_t>(r));
  case HGRD_DIV:
    return r == 0 ? 0 : (r == -1 ? -l : l / r);
  case HGRD_MOD:
    return (r == 0 || r == -1) ? 0 : l % r;
  case HGRD_LT:
    return l < r;
  case HGRD_LE:
    return l <= r;
  case HGRD_GT:
    return l > r;
  case HGRD_GE:
    return l >= r;
  case HGRD_EQ:
    return l == r;
  case HGRD_NE:
    return l != r;
  case HGRD_AND:
    return (l != 0 && r != 0) ? 1 : 0;
  case HGRD_OR:
    return (l != 0 || r != 0) ? 1 : 0;
  }
  return 0;
}

__device__ __forceinline__ uint64_t packKey(const KeyLayout &k, uint64_t elem,
                                            uint64_t block, uint64_t bp,
                                            uint64_t warp, uint64_t wp,
                                            uint64_t lane) {
  return (elem << k.shE) | (block << k.shB) | (bp << k.shP) | (warp << k.shW) |
         (wp << k.shQ) | lane;
}

__device__ __forceinline__ int bitsForDev(uint64_t n) { // bits to hold 0 .. n-1
  return n <= 1 ? 0 : 64 - __clzll(static_cast<long long>(n - 1));
}

__device__ __forceinline__ uint64_t fieldMask(int bits) {
  return bits >= 64 ? ~0ull : ((1ull << bits) - 1);
}

__host__ __device__ __forceinline__ uint32_t seqMask(const KeyLayout &kl) {
  return (1u << kl.bS) - 1;
}

constexpr uint32_t kOwnerMulti = 0xFFFFFu; // filter-tag marker of the bit-map layout

// Ownership table (the fused path's INTER-BLOCK filter), two layouts:
// * bit map (two bits per element, 16 elements per word): the block's first
//   record of element e ORs e's "touched" bit; finding it already set means
//   another block touched e (each block records e's first access once:
//   k_fused's `first`), and the thread then ORs e's MULTI bit.  2 bits per
//   element keep a 2^27-element table at 32 MiB, resident in L2 (the
//   32-bit exchange table it replaced was 512 MiB of random DRAM
//   read-modify-writes).  Cleared per launch (a memset of n / 4 bytes).  A
//   block that records e twice (a chain walk cut short by radix mode) can
//   only add a false MULTI, which pass 2 — exact on any superset of the
//   shared elements — filters out.
// * reduction (two words per element): hi = max(epoch | block+1) and
//   lo = max(epoch | (0xFFFFF - (block+1))) — max and (complemented) min
//   block, fire-and-forget RED.MAX with no round trip on the thread's
//   critical path; MULTI iff both words carry the epoch and min != max.
//   Epoch tags: no memset between launches.
// Tables up to 4 Mi elements use reductions, larger ones the bit map.  The
// filter tag tells the layouts apart: kOwnerMulti (bit map) or epoch << 20
// (reduction).
__device__ __forceinline__ void ownerJoin(uint32_t *owner, uint64_t e, uint32_t epochTag,
                                          uint32_t blockPlus1) {
  atomicMax(&owner[2 * e], epochTag | blockPlus1);
  atomicMax(&owner[2 * e + 1], epochTag | (kOwnerMulti - blockPlus1));
}
__device__ __forceinline__ bool ownerIsMulti(const uint32_t *owner, uint64_t e,
                                             uint32_t filterTag) {
  if (filterTag & kOwnerMulti)
    return (owner[e >> 4] >> (2 * (e & 15) + 1)) & 1u;
  const uint2 w = *reinterpret_cast<const uint2 *>(owner + 2 * e);
  return (w.x >> 20) == (filterTag >> 20) && (w.y >> 20) == (filterTag >> 20) &&
         (w.x & kOwnerMulti) != kOwnerMulti - (w.y & kOwnerMulti);
}

} // namespace dev
} // namespace hgrdgpu

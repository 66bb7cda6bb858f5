// K-fused: block-local race check (PARALLEL launches without lock idioms).
//
// One CTA iteration takes one or more whole MiniCU blocks.  Every
// INTRA-BLOCK / INTRA-WARP pair lies inside one MiniCU block
// (reference src/oracle.cpp:754-769), so they are found entirely on chip:
//   1. expansion into shared memory (two-word records, see packR0/packR1);
//      each record is pushed onto the chain of its element's hash slot
//      (2x-oversized table, lock-free acq_rel CAS) and at that moment paired
//      with the earlier records of its element on the chain: realised INTRA
//      keys and, per key, the minimum element.  A chain longer than
//      kSmallGroup (a hot element) switches the iteration to a CUB block
//      radix sort of element | block | bp | warp | wp | lane with per-group
//      summaries instead,
//   2. per realised key: the first (x, y) pair of the reference's order
//      inside that element, published as a candidate (global element via
//      atomicMin, candidates filtered by it; the last CTA keeps the
//      lexicographically first pair of the minimum element).
// INTER-BLOCK pairs need a second block: every (element, block) also joins
// the element in the ownership table (device.cuh); an element reached from
// two blocks becomes MULTI and only MULTI elements go through pass 2
// (ctx.cu).
#pragma once

#include "detect.cuh"
#include "device.cuh"
#include "expand.cuh"

#include <cub/block/block_radix_sort.cuh>

namespace hgrdgpu {
namespace dev {

constexpr int kMaxWritten = 8;
constexpr int kSmallGroup = 32; // hash slots up to this size, radix grouping above
constexpr int kMaxIterBlocks = 256; // MiniCU blocks per iteration: the 8-bit blk field of r1
constexpr uint64_t kKnownMax = 1u << 17; // elements of a CTA's known-MULTI map (16 KB)

enum FusedFlags : uint32_t {
  kFlagShared = 128u,   // an element is accessed by two blocks (pass 2 needed)
  kFlagFusedOverflow = 256u, // records / key bits / candidates did not fit
};

struct Candidate {
  int32_t key;
  int32_t siteX, siteY;
  int32_t pad;
  uint64_t elem;
  uint64_t xOrd, yOrd;
};

struct FusedArgs {
  LaunchDev L;
  int nLocs, nKeys;
  int bpi;              // whole MiniCU blocks per iteration
  int64_t blockBase, blockEnd; // dense MiniCU block range of this launch (or shard)
  int interOnChip; // the whole launch is one iteration: INTER-BLOCK pairs found on chip too
  uint32_t R;           // records per MiniCU thread when static (0: allocate)
  int64_t nIters;
  uint32_t *owner; // per element ownership word(s) (device.cuh)
  uint32_t epoch;
  int ownerRed;    // reduction layout (two words per element), else the bit map
  unsigned long long *keyElem;
  Candidate *cand;
  uint32_t candCap;
  unsigned int *candCount;
  int nW;
  hgrd_gpu_race *races;     // INTRA races are finalised by the last CTA
  const uint64_t *wBase;    // element -> (handle, index)
  const int32_t *wHandle;
  int ablate; // profiling knob (HGRD_FUSED_ABLATE): 1 skip the post-expansion phases,
              // 4 skip ownership exchanges, 8 skip expansion
  // streamed load (affine.hpp streamSites; JIT bodies' loadS): index = dense
  // thread + streamOff into `stream` (streamSize elements); each iteration's
  // values arrive in shared memory by a TMA bulk copy issued one iteration
  // ahead (double-buffered, mbarrier-completed); nullptr: no stream
  const int64_t *stream;
  int64_t streamOff, streamSize;
  int stageCap; // elements per staging buffer
  // reduction layout, small tables: words of the CTA's shared bit map of
  // elements it has seen become MULTI (their joins are skipped), else 0
  uint32_t knownWords;
  // sharded checks: the shard's per-(element, site) min / max block + 1
  // (parallel.py's INTER summary), filled from the records (nullptr: none)
  uint32_t *shardLo, *shardHi;
  int nSitesTab;
};

// TMA bulk copies (cp.async.bulk -> UBLKCP) completing on an mbarrier
__device__ __forceinline__ uint32_t smemAddr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbarInit(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smemAddr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbarArriveTx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemAddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbarArrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smemAddr(bar)) : "memory");
}
__device__ __forceinline__ void mbarWait(uint64_t *bar, unsigned parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT_%=;\n\t}" ::"r"(smemAddr(bar)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void bulkToShared(void *dst, const void *src, unsigned bytes,
                                             uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
               "%2, [%3];" ::"r"(smemAddr(dst)),
               "l"(src), "r"(bytes), "r"(smemAddr(bar))
               : "memory");
}

// Stage iteration `it`'s streamed values: elements [first + off, first +
// off + n) clamped to the buffer, widened to 16-byte alignment (buffers are
// 256-byte aligned and padded); one elected thread.  Returns the first
// staged element index.
__device__ __forceinline__ int64_t stageIssue(const FusedArgs &F, int64_t it, int64_t *buf,
                                              uint64_t *bar) {
  const int64_t first = (F.blockBase + it * F.bpi) * F.L.tpb;
  const int64_t n = (min(static_cast<int64_t>(F.bpi), F.blockEnd - (F.blockBase + it * F.bpi))) *
                    F.L.tpb;
  const int64_t lo = max(first + F.streamOff, static_cast<int64_t>(0));
  const int64_t hi = min(first + F.streamOff + n, F.streamSize);
  if (hi <= lo) {
    mbarArrive(bar); // nothing in bounds: complete the phase without data
    return 0;
  }
  const int64_t a = (lo * 8) & ~int64_t(15), b = (hi * 8 + 15) & ~int64_t(15);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // generic reads before TMA writes
  mbarArriveTx(bar, static_cast<unsigned>(b - a));
  bulkToShared(buf, reinterpret_cast<const char *>(F.stream) + a, static_cast<unsigned>(b - a), bar);
  return a / 8;
}

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// Records are two words (elements < 2^32 - 1 on this path):
//   r0 = site:12 | seq:20 | elem:32
//   r1 = tli:16 | blk:8 | bp:8 | wp:8 | warp:16 | 0:8
// tli = thread within the iteration, blk = MiniCU block within the
// iteration, warp = warp within the MiniCU block; the pair rule reads
// XORs of r1 words (no divisions).
constexpr uint64_t kNoRec = ~0ull; // fixed-slot mode: a slot its thread did not fill

__device__ __forceinline__ uint64_t packR0(int site, uint32_t seq, uint32_t e) {
  return (static_cast<uint64_t>(site & 4095) << 52) |
         (static_cast<uint64_t>(seq & kSeqMask) << 32) | e;
}
__device__ __forceinline__ uint64_t packR1(uint32_t tli, uint32_t blk, uint32_t bp, uint32_t wp,
                                           uint32_t warp) {
  return (static_cast<uint64_t>(tli) << 48) | (static_cast<uint64_t>(blk & 255) << 40) |
         (static_cast<uint64_t>(bp & 255) << 32) | (static_cast<uint64_t>(wp & 255) << 24) |
         (static_cast<uint64_t>(warp & 0xFFFF) << 8);
}
__device__ __forceinline__ uint32_t rElem(uint64_t r0) { return static_cast<uint32_t>(r0); }
__device__ __forceinline__ int rSite(uint64_t r0) { return static_cast<int>(r0 >> 52); }
__device__ __forceinline__ uint32_t rSeq(uint64_t r0) {
  return static_cast<uint32_t>(r0 >> 32) & kSeqMask;
}
__device__ __forceinline__ uint32_t rTli(uint64_t r1) { return static_cast<uint32_t>(r1 >> 48); }
__device__ __forceinline__ uint32_t rBlk(uint64_t r1) { return (r1 >> 40) & 255; }
__device__ __forceinline__ uint32_t rBp(uint64_t r1) { return (r1 >> 32) & 255; }
__device__ __forceinline__ uint32_t rWp(uint64_t r1) { return (r1 >> 24) & 255; }
__device__ __forceinline__ uint32_t rWarp(uint64_t r1) { return (r1 >> 8) & 0xFFFF; }

// The reference pair rule (:750-769) for two records of one element, given
// that their sites conflict statically (confIntra covers "a write" and "not
// two covering atomics"): -1 when the pair is excluded or INTER-BLOCK, else
// 1 (INTRA-BLOCK) or 2 (INTRA-WARP).
__device__ __forceinline__ int intraRule(uint64_t a1, uint64_t b1) {
  const uint64_t x = a1 ^ b1;
  if ((x >> 48) == 0)
    return -1; // same thread
  if ((x >> 32) & 0xFFFF)
    return -1; // other MiniCU block (INTER) or other barrier phase
  if ((x >> 8) & 0xFFFF)
    return 1; // other warp
  return ((x >> 24) & 255) ? -1 : 2; // same warp: same warp phase only
}

// After k_fused: whether any element is MULTI (then pass 2 runs); read with
// the counters, so no extra round trip.
__global__ void k_owner_any(const uint32_t *owner, uint64_t nElems, uint32_t epochTag,
                            Counters *ctr) {
  bool any = false;
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nElems;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    any |= ownerIsMulti(owner, e, epochTag);
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0)
    atomicOr(&ctr->flags, static_cast<unsigned>(kFlagShared));
}

// A thread's ownership atomic in flight: its old word is examined when the
// thread issues its next one or at the kernel's end, so the L2 round trip
// overlaps the next MiniCU thread's expansion instead of stalling this one.
// * bit map (device.cuh): the touched bit was already set -> the thread
//   sets e's MULTI bit (a late MULTI bit is still set before the kernel
//   ends, and only pass 2 reads it);
// * reduction layout with the CTA's known-MULTI map (`known`): the previous
//   max(epoch | block+1) was another block's -> e is MULTI, and the CTA's
//   later joins of e are skipped (MULTI is final within the launch: the
//   joins already made keep min != max).
struct OwnerPend {
  uint32_t *addr = nullptr;
  uint32_t old = 0, aux = 0, mine = 0; // aux: bit-pair offset, or the element
  __device__ __forceinline__ void settle(unsigned &flags, uint32_t *known, uint32_t epochTag) {
    if (addr) {
      if (known) {
        if ((old >> 20) == (epochTag >> 20) && (old & kOwnerMulti) != mine)
          atomicOr(&known[aux >> 5], 1u << (aux & 31));
      } else if ((old >> aux) & 1u) { // touched before by another block
        if (!((old >> aux) & 2u))
          atomicOr(addr, 2u << aux);
        flags |= kFlagShared;
      }
      addr = nullptr;
    }
  }
};

// NT threads x IPT records per thread of shared-memory record capacity.
template <int NT, int IPT> struct FusedSmem {
  static constexpr int kThreads = NT;
  static constexpr int kCap = NT * IPT;
  static constexpr int kTable = 2 * kCap; // hash slots (power of two)
  static constexpr int kLogTable = ilog2(kTable);
  static constexpr uint32_t kEnd = 0xffffffffu;
  using Sort = cub::BlockRadixSort<uint64_t, NT, IPT, uint32_t, 5>;
  union {
    typename Sort::TempStorage sortTmp;
    struct {
      uint32_t head[kTable]; // per hash slot: most recent record (chain head)
      uint32_t next[kCap];   // per record: previous record of its slot
    } ch;
    struct {
      uint64_t skey[kCap];  // radix mode: sorted keys
      uint32_t sidx[kCap];  // sorted position -> record index
    } rx;
  } u;
  // records by index, {r0, r1} interleaved so a record is one 16-byte
  // shared-memory store: r0 = site | seq | elem, r1 = tli | blk | bp | wp | warp
  ulonglong2 rec[kCap];
  uint32_t minE[kMaxWritten], maxE[kMaxWritten];
  unsigned int count, maxBp, maxWp, nReal, flags, hot;
  // radix mode: field start bits of the key  w|off|blk|bp|warp|wp|lane
  int fWp, fWarp, fBp, fBlk, fOff, fW, total;
};

template <class Smem> __device__ __forceinline__ uint32_t hashSlot(uint32_t e) {
  return (e * 0x9E3779B1u) >> (32 - Smem::kLogTable);
}

__device__ __forceinline__ int keyIndex(const SiteDev *sites, int nLocs, int sa, int sb, int kind) {
  int la = sites[sa].loc, lb = sites[sb].loc;
  if (lb < la) {
    int t = la;
    la = lb;
    lb = t;
  }
  return (la * nLocs + lb) * 3 + kind;
}

// Keep the minimum `v` (element in hash mode, sorted position in radix
// mode) per key; the first setter appends the key to the realised list.
template <class Smem>
__device__ __forceinline__ void noteKey(Smem &S, uint32_t *sKeyMin, uint32_t *sReal, int K,
                                        uint32_t v) {
  if (sKeyMin[K] <= v)
    return;
  const uint32_t old = atomicMin(&sKeyMin[K], v);
  if (old == ~0u) {
    const unsigned slot = atomicAdd(&S.nReal, 1u);
    sReal[slot] = static_cast<uint32_t>(K);
  }
}

// Lock-free push of record `pos` onto a hash slot's chain.  acq_rel: the
// record's words (written before) are visible to whoever later reads the
// chain through the slot, and this thread sees the words of every record
// pushed before it.
__device__ __forceinline__ uint32_t casAcqRel(uint32_t *p, uint32_t cmp, uint32_t val) {
  uint32_t old;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("atom.acq_rel.cta.shared::cta.cas.b32 %0, [%1], %2, %3;"
               : "=r"(old)
               : "r"(a), "r"(cmp), "r"(val)
               : "memory");
  return old;
}

// PARALLEL sink of the fused kernel: records into shared memory, each
// pushed onto the chain of its element's hash slot and, at that moment,
// paired with the records of its element pushed before it (every pair is
// seen exactly once: by whichever of the two was pushed second).  The
// block's first record of an element also joins the element's block range
// in the ownership table (the INTER-BLOCK filter, device.cuh): an OR into
// the bit map, or two fire-and-forget max reductions when the table fits
// L2.  Sites whose parameter is provably block-private (host affine
// analysis, `own` = false) skip it: no other block can reach their elements.
template <class Smem> struct FusedSink : ParState {
  Smem *S;
  uint32_t tli;      // thread index within the iteration
  uint32_t stride;   // fixed-slot mode: threads in the iteration
  uint32_t nrec = 0; // records produced by this thread
  uint32_t R;        // fixed-slot mode: slots per thread (0: allocate)
  uint32_t myBlk;    // MiniCU block within the iteration
  int nLocs;
  uint32_t *keyMin;  // per key: minimum element realised in the iteration
  uint32_t *real;    // realised keys
  const uint64_t *conf;  // per site: statically conflicting sites within a block (bit mask)
  const uint64_t *confX; // ... across blocks (interOnChip)
  bool interOnChip;
  uint32_t *owner;      // per element ownership words (nullptr: ablated)
  uint32_t epochTag;    // epoch << 20
  uint32_t mine;        // this thread's block + 1
  bool ownerRed = false; // reduction layout of the ownership table (else the bit map)
  OwnerPend *pend = nullptr; // the thread's ownership atomic in flight
  uint32_t *known = nullptr;  // the CTA's known-MULTI elements (reduction layout)
  uint32_t *shardLo = nullptr, *shardHi = nullptr; // sharded: (element, site) block min / max
  int nSitesTab = 0;
  // k_batch: every trap of the launch, keyed thread << 20 | n-th trap of the
  // thread (canonical order once sorted); nullptr in k_fused (any trap sends
  // the launch to the ordered path there)
  uint64_t *trapKey = nullptr;
  uint32_t *trapSite = nullptr; // site << 1 | unallocated
  unsigned *trapCount = nullptr;
  unsigned trapCap = 0;
  uint32_t myTraps = 0;

  __device__ __forceinline__ void noteTrap(int site, int param) {
    if (!trapKey)
      return;
    const ParamDev *P = param >= 0 ? &params[param] : nullptr;
    const bool unalloc = !P || P->handle < 0;
    const unsigned i = atomicAdd(trapCount, 1u);
    if (i < trapCap) {
      trapKey[i] = (static_cast<uint64_t>(tli) << 20) | myTraps;
      trapSite[i] = (static_cast<uint32_t>(site) << 1) | (unalloc ? 1u : 0u);
    }
    ++myTraps;
  }

  __device__ __forceinline__ void pairWithEarlier(uint32_t e, uint64_t r1, int site, uint32_t q,
                                                  bool own) {
    bool first = true;
    int len = 0;
    const int myLoc = sites[site].loc;
    for (; q != Smem::kEnd; q = S->u.ch.next[q]) {
      if (++len > kSmallGroup) { // a hot element: radix grouping instead
        S->hot = 1;
        break;
      }
      const uint64_t q0 = S->rec[q].x;
      if (rElem(q0) != e)
        continue;
      const uint64_t q1 = S->rec[q].y;
      const uint64_t *cf = conf;
      int kind;
      if (rBlk(q1) == myBlk) {
        first = false;
        kind = intraRule(q1, r1);
      } else if (interOnChip) { // another block of this one-iteration launch
        kind = 0;
        cf = confX;
      } else {
        continue; // INTER: the ownership table and pass 2
      }
      if (kind < 0)
        continue;
      const int sq = rSite(q0);
      if (!((cf[sq] >> site) & 1ull))
        continue;
      int la = sites[sq].loc, lb = myLoc;
      if (lb < la) {
        const int t = la;
        la = lb;
        lb = t;
      }
      noteKey(*S, keyMin, real, (la * nLocs + lb) * 3 + kind, e);
    }
    if (own && shardLo) { // sharded check: the block joins (e, site)'s block range
      const uint64_t i = static_cast<uint64_t>(e) * nSitesTab + site;
      atomicMin(&shardLo[i], mine);
      atomicMax(&shardHi[i], mine);
    }
    if (own && first && owner) { // the block's first record of e (device.cuh ownership)
      if (!ownerRed) {
        pend->settle(flags, nullptr, epochTag);
        pend->addr = &owner[e >> 4];
        pend->aux = 2 * (e & 15);
        pend->old = atomicOr(pend->addr, 1u << pend->aux);
      } else if (!known) {
        ownerJoin(owner, e, epochTag, mine);
      } else if (!((known[e >> 5] >> (e & 31)) & 1u)) { // (known MULTI: nothing to add)
        pend->settle(flags, known, epochTag);
        atomicMax(&owner[2 * e + 1], epochTag | (kOwnerMulti - mine));
        pend->addr = &owner[2 * e];
        pend->aux = e;
        pend->mine = mine;
        pend->old = atomicMax(pend->addr, epochTag | mine);
      }
    }
  }

  __device__ __forceinline__ void record(int site, const ParamDev *P, int64_t idx, bool own) {
    recordE(site, P->elemBase + static_cast<uint64_t>(idx), own);
  }
  __device__ __forceinline__ void recordE(int site, uint64_t elem, bool own) {
    if (bp > 255 || wp > 255 || seq > kSeqMask || site > kMaxSiteId)
      flags |= kFlagFusedOverflow;
    unsigned pos;
    if (R) { // static record count per thread: slot k of thread t at k * stride + t
      // (column-major, so a warp's k-th records are adjacent), no atomics
      pos = nrec < R ? nrec * stride + tli : 0xffffffffu;
    } else { // warp-aggregated allocation (one shared atomic per converged group)
      const unsigned act = __activemask();
      const int ln = threadIdx.x & 31;
      const int leader = __ffs(act) - 1;
      unsigned base = 0;
      if (ln == leader)
        base = atomicAdd(&S->count, static_cast<unsigned>(__popc(act)));
      base = __shfl_sync(act, base, leader);
      pos = base + __popc(act & ((1u << ln) - 1));
    }
    ++nrec;
    if (pos < static_cast<unsigned>(Smem::kCap)) {
      const uint32_t e = static_cast<uint32_t>(elem);
      const uint64_t r1 = packR1(tli, myBlk, bp, wp, static_cast<uint32_t>(warp));
      S->rec[pos] = make_ulonglong2(packR0(site, seq, e), r1); // one STS.128
      uint32_t *head = &S->u.ch.head[hashSlot<Smem>(e)];
      uint32_t h = *reinterpret_cast<volatile uint32_t *>(head);
      for (;;) {
        S->u.ch.next[pos] = h;
        const uint32_t o = casAcqRel(head, h, pos);
        if (o == h)
          break;
        h = o;
      }
      pairWithEarlier(e, r1, site, h, own);
    } else {
      flags |= kFlagFusedOverflow;
    }
    ++recs;
  }
  // C variants (JIT bodies): the site's parameter, flags, buffer size and
  // element base as constants (size 0: unallocated parameter, always traps)
  // (I: int64_t, or int32_t when the index and the buffer size fit 32 bits)
  template <class I>
  __device__ __forceinline__ int64_t loadC(int site, int param, bool rec, bool own, I idx,
                                           bool need, int64_t size, uint64_t base) {
    if (outOfRange(idx, size)) {
      ++traps;
      return 0;
    }
    ++inst;
    if (rec)
      recordE(site, elementAt(base, idx), own);
    ++seq;
    return need ? __ldg(params[param].ptr + idx) : 0;
  }
  // The value half of a value-needed loadC (JitBody::run2 issues both
  // threads' fetches before either records): 0 when out of range, as loadC.
  template <class I>
  __device__ __forceinline__ int64_t fetchC(int param, I idx, int64_t size) const {
    return outOfRange(idx, size) ? 0 : __ldg(params[param].ptr + idx);
  }
  // S variant: a streamed load (affine.hpp streamSites): idx is the MiniCU
  // thread's dense id plus a constant, so the iteration's values were staged
  // in shared memory by a bulk copy (k_fused) — no global load latency on the
  // thread's critical path
  const int64_t *stage = nullptr; // staged values, element stageBase first
  int64_t stageBase = 0;
  template <class I>
  __device__ __forceinline__ int64_t loadS(int site, int param, bool rec, bool own, I idx,
                                           int64_t size, uint64_t base) {
    if (!stage)
      return loadC(site, param, rec, own, idx, true, size, base);
    if (outOfRange(idx, size)) {
      ++traps;
      return 0;
    }
    ++inst;
    if (rec)
      recordE(site, elementAt(base, idx), own);
    ++seq;
    return stage[static_cast<int64_t>(idx) - stageBase];
  }
  template <class I>
  __device__ __forceinline__ void storeC(int site, int param, bool rec, bool own, I idx, int64_t,
                                         int64_t size, uint64_t base) {
    loadC(site, param, rec, own, idx, false, size, base);
  }
  template <class I>
  __device__ __forceinline__ void atomicC(int site, int param, bool rec, bool own, I idx,
                                          int64_t, int64_t, int64_t size, uint64_t base) {
    loadC(site, param, rec, own, idx, false, size, base);
  }
  // K variants: the site's parameter, record and ownership flags as (JIT)
  // constants
  __device__ __forceinline__ int64_t loadK(int site, int param, bool rec, bool own, int64_t idx,
                                           bool need) {
    const ParamDev *P = checkK(param, idx);
    if (!P) {
      noteTrap(site, param);
      return 0;
    }
    if (rec)
      record(site, P, idx, own);
    ++seq;
    return need ? __ldg(P->ptr + idx) : 0;
  }
  __device__ __forceinline__ void storeK(int site, int param, bool rec, bool own, int64_t idx,
                                         int64_t) {
    const ParamDev *P = checkK(param, idx);
    if (!P) {
      noteTrap(site, param);
      return;
    }
    if (rec)
      record(site, P, idx, own);
    ++seq;
  }
  __device__ __forceinline__ void atomicK(int site, int param, bool rec, bool own, int64_t idx,
                                          int64_t, int64_t) {
    storeK(site, param, rec, own, idx, 0);
  }
  __device__ __forceinline__ int64_t load(int site, int64_t idx, bool need) {
    const SiteDev &S_ = sites[site];
    return loadK(site, S_.param, S_.record, S_.own, idx, need);
  }
  __device__ __forceinline__ void store(int site, int64_t idx, int64_t v) {
    const SiteDev &S_ = sites[site];
    storeK(site, S_.param, S_.record, S_.own, idx, v);
  }
  __device__ __forceinline__ void atomic(int site, int64_t idx, int64_t v, int64_t c) {
    const SiteDev &S_ = sites[site];
    atomicK(site, S_.param, S_.record, S_.own, idx, v, c);
  }
};

#ifndef HGRD_FUSED_MINB
#define HGRD_FUSED_MINB 3
#endif
// NT = 128 or 256 threads per CTA; IPT records per thread of capacity.
template <int NT, int IPT, class Body>
__global__ void __launch_bounds__(NT, NT == 128 ? 6 : HGRD_FUSED_MINB) k_fused(FusedArgs F) {
  using Smem = FusedSmem<NT, IPT>;
  constexpr int kFusedThreads = NT;
  extern __shared__ __align__(16) unsigned char dyn[];
  Smem &S = *reinterpret_cast<Smem *>(dyn);
  unsigned char *after = dyn + ((sizeof(Smem) + 15) & ~size_t(15));
  const int nKeysPad = (F.nKeys + 3) & ~3;
  uint32_t *sKeyMin = reinterpret_cast<uint32_t *>(after);
  uint32_t *sReal = reinterpret_cast<uint32_t *>(sKeyMin + nKeysPad);
  // per key: an upper bound of the global minimum element F.keyElem[K]
  // (it only decreases), so later iterations skip most global reads
  uint32_t *sKeyBound = sReal + nKeysPad;
  hgrd_gpu_insn *sCode = reinterpret_cast<hgrd_gpu_insn *>(sKeyBound + nKeysPad);
  SiteDev *sSites = reinterpret_cast<SiteDev *>(sCode + F.L.nCode);
  ParamDev *sParams = reinterpret_cast<ParamDev *>(sSites + F.L.nSites);
  uint64_t *sConf = reinterpret_cast<uint64_t *>(sParams + F.L.nParams);
  uint64_t *sConfX = sConf + F.L.nSites;
  int64_t *sStage = reinterpret_cast<int64_t *>(
      (reinterpret_cast<uintptr_t>(sConfX + F.L.nSites) + 15) & ~uintptr_t(15));
  uint32_t *sKnown = F.knownWords ? reinterpret_cast<uint32_t *>(
                                         sStage + (F.stream ? 2 * F.stageCap + 2 : 0))
                                   : nullptr;
  // dynamic shared memory layout mirrored by fusedSmemBytes() in ctx.cu
  __shared__ __align__(8) uint64_t sBar[2];
  __shared__ int64_t sStageBase[2];
  const bool streamed = F.stream != nullptr;
  const LaunchDev &L = F.L;
  const int tid = threadIdx.x;
  for (int i = tid; i < L.nCode; i += kFusedThreads)
    sCode[i] = L.code[i];
  for (int i = tid; i < L.nSites; i += kFusedThreads) {
    sSites[i] = L.sites[i];
    sConf[i] = L.confIntra[i];
    sConfX[i] = L.confInter[i];
  }
  for (int i = tid; i < L.nParams; i += kFusedThreads)
    sParams[i] = L.params[i];
  for (uint32_t i = tid; i < F.knownWords; i += kFusedThreads)
    sKnown[i] = 0;
  for (int i = tid; i < F.nKeys; i += kFusedThreads) {
    sKeyMin[i] = ~0u;
    sKeyBound[i] = ~0u;
  }
  if (tid == 0) {
    S.nReal = 0;
    S.flags = 0;
  }
  const uint32_t tpb = static_cast<uint32_t>(L.tpb);
  const int64_t ws = L.ws;
  // records per thread (fixed slots) — a compile-time constant in JIT bodies
  const uint32_t fixedR = Body::kFixedR >= 0 ? static_cast<uint32_t>(Body::kFixedR) : F.R;
  LaneTally tally;
  unsigned myFlags = 0;
  bool wroteCand = false; // this thread stored a candidate (released before the done count)
  int64_t regs[kMaxRegs];
  OwnerPend pend, pend2; // (pend2: the second thread of a JitBody::run2 pair)
  if (streamed && tid == 0) {
    mbarInit(&sBar[0], 1);
    mbarInit(&sBar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (static_cast<int64_t>(blockIdx.x) < F.nIters)
      sStageBase[0] = stageIssue(F, blockIdx.x, sStage, &sBar[0]);
  }

  int64_t k = 0; // this CTA's iteration count (staging buffer k & 1)
  for (int64_t it = blockIdx.x; it < F.nIters; it += gridDim.x, ++k) {
    const int64_t firstBlock = F.blockBase + it * F.bpi;
    const int64_t nb = min(static_cast<int64_t>(F.bpi), F.blockEnd - firstBlock);
    __syncthreads();
    const int sb = static_cast<int>(k & 1);
    if (streamed) { // prefetch the next iteration's values, then wait for this one's
      if (tid == 0 && it + gridDim.x < F.nIters)
        sStageBase[sb ^ 1] =
            stageIssue(F, it + gridDim.x, sStage + (sb ^ 1) * F.stageCap, &sBar[sb ^ 1]);
      mbarWait(&sBar[sb], static_cast<unsigned>((k >> 1) & 1));
    }
    if (tid == 0) {
      S.count = fixedR ? static_cast<unsigned>(nb * L.tpb) * fixedR : 0;
      S.maxBp = 0;
      S.maxWp = 0;
      S.hot = 0;
      S.nReal = 0; // (every thread read it after the previous iteration's barrier)
    }
    static_assert(Smem::kTable % 4 == 0, "chain heads are reset 16 bytes at a time");
    for (int i = tid; i < Smem::kTable / 4; i += kFusedThreads) // (S: 16-byte aligned)
      reinterpret_cast<uint4 *>(S.u.ch.head)[i] =
          make_uint4(Smem::kEnd, Smem::kEnd, Smem::kEnd, Smem::kEnd);
    __syncthreads();
    // 1. expansion of the iteration's whole MiniCU blocks: records pushed
    //    per hash slot and paired as they are produced (FusedSink)
    if (!(F.ablate & 8)) {
      unsigned myBp = 0, myWp = 0;
      // (iteration invariants hoisted; an iteration holds < 2^16 MiniCU threads)
      const uint32_t nT = static_cast<uint32_t>(nb * L.tpb);
      const int64_t *stageBuf = streamed ? sStage + sb * F.stageCap : nullptr;
      const int64_t stageB = streamed ? sStageBase[sb] : 0;
      const int64_t firstThread = firstBlock * L.tpb;
      auto begin = [&](FusedSink<Smem> &s, uint32_t tl, OwnerPend *pd, Builtins &bi) {
        s.L = &L;
        s.sites = sSites;
        s.params = sParams;
        s.S = &S;
        s.tli = static_cast<uint32_t>(tl);
        s.R = fixedR;
        s.stride = nT;
        s.myBlk = L.dTpb.div(tl);
        s.nLocs = F.nLocs;
        s.keyMin = sKeyMin;
        s.real = sReal;
        s.conf = sConf;
        s.confX = sConfX;
        s.interOnChip = F.interOnChip != 0;
        s.owner = (F.ablate & 4) ? nullptr : F.owner;
        s.epochTag = F.epoch << 20;
        s.ownerRed = F.ownerRed != 0;
        s.pend = pd;
        s.known = sKnown;
        s.shardLo = F.shardLo;
        s.shardHi = F.shardHi;
        s.nSitesTab = F.nSitesTab;
        s.mine = static_cast<uint32_t>(firstBlock + s.myBlk + 1);
        s.stage = stageBuf;
        s.stageBase = stageB;
        Body::identity(L, firstThread + tl, bi, s.block, s.warp, s.lane);
      };
      auto finish = [&](FusedSink<Smem> &s) {
        for (uint32_t j = s.nrec; j < s.R; ++j)
          if (j * s.stride + s.tli < static_cast<uint32_t>(Smem::kCap))
            S.rec[j * s.stride + s.tli].x = kNoRec;
        tally.add(s);
        myBp = max(myBp, s.bp);
        myWp = max(myWp, s.wp);
      };
      if constexpr (Body::kPair) { // MiniCU threads tl and tl + NT together (JitBody::run2)
        for (uint32_t tl = tid; tl < nT; tl += 2 * kFusedThreads) {
          FusedSink<Smem> s0, s1;
          Builtins b0, b1;
          begin(s0, tl, &pend, b0);
          if (tl + kFusedThreads < nT) {
            begin(s1, tl + kFusedThreads, &pend2, b1);
            Body::run2(b0, s0, b1, s1);
            finish(s0);
            finish(s1);
          } else {
            Body::run(L, sCode, b0, s0, regs);
            finish(s0);
          }
        }
      } else {
        for (uint32_t tl = tid; tl < nT; tl += kFusedThreads) {
          FusedSink<Smem> s;
          Builtins bi;
          begin(s, tl, &pend, bi);
          Body::run(L, sCode, bi, s, regs);
          finish(s);
        }
      }
      if (__any_sync(0xffffffffu, myBp | myWp)) { // (barrier-free bodies: one vote)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          myBp = max(myBp, __shfl_down_sync(0xffffffffu, myBp, o));
          myWp = max(myWp, __shfl_down_sync(0xffffffffu, myWp, o));
        }
        if ((tid & 31) == 0) {
          atomicMax(&S.maxBp, myBp);
          atomicMax(&S.maxWp, myWp);
        }
      }
    }
    __syncthreads();
    const unsigned n = min(S.count, static_cast<unsigned>(Smem::kCap));
    if (S.count > static_cast<unsigned>(Smem::kCap))
      myFlags |= kFlagFusedOverflow;
    if (n == 0)
      continue;
    if (F.ablate & 1)
      continue;
    const bool hashed = S.hot == 0;
    if (!hashed && F.interOnChip) { // radix grouping has no INTER level: general path
      myFlags |= kFlagFusedOverflow;
      continue;
    }
    if (!hashed) {
      // radix mode for this iteration: drop the hash-mode keys, sort by
      // w | off | blk | bp | warp | wp | lane and summarise per group
      for (unsigned r = tid; r < S.nReal; r += kFusedThreads)
        sKeyMin[sReal[r]] = ~0u;
      if (tid < kMaxWritten) {
        S.minE[tid] = ~0u;
        S.maxE[tid] = 0;
      }
      __syncthreads();
      if (tid == 0)
        S.nReal = 0;
      for (unsigned i = tid; i < n; i += kFusedThreads) {
        const uint64_t r0 = S.rec[i].x;
        if (r0 == kNoRec)
          continue;
        const int w = sParams[sSites[rSite(r0)].param].written - 1;
        atomicMin(&S.minE[w], rElem(r0));
        atomicMax(&S.maxE[w], rElem(r0));
      }
      __syncthreads();
      if (tid == 0) {
        uint64_t span = 1;
        for (int w = 0; w < F.nW && w < kMaxWritten; ++w)
          if (S.minE[w] <= S.maxE[w])
            span = max(span, static_cast<uint64_t>(S.maxE[w] - S.minE[w]) + 1);
        const int bL = bitsForDev(static_cast<uint64_t>(ws < L.tpb ? ws : L.tpb));
        const int bW = bitsForDev(static_cast<uint64_t>((L.tpb + ws - 1) / ws));
        const int bQ = bitsForDev(uint64_t(S.maxWp) + 1);
        const int bP = bitsForDev(uint64_t(S.maxBp) + 1);
        const int bBk = bitsForDev(static_cast<uint64_t>(F.bpi));
        const int bO = bitsForDev(span);
        const int bWr = bitsForDev(static_cast<uint64_t>(F.nW));
        S.fWp = bL;
        S.fWarp = S.fWp + bQ;
        S.fBp = S.fWarp + bW;
        S.fBlk = S.fBp + bP;
        S.fOff = S.fBlk + bBk;
        S.fW = S.fOff + bO;
        S.total = S.fW + bWr;
        if (S.total > 64)
          S.flags |= kFlagFusedOverflow;
      }
      __syncthreads();
      if (S.total > 64)
        continue;
      uint64_t keys[IPT];
      uint32_t vals[IPT];
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const unsigned i = static_cast<unsigned>(tid * IPT + j);
        vals[j] = i;
        const uint64_t r0 = i < n ? S.rec[i].x : kNoRec;
        if (r0 != kNoRec) {
          const uint64_t r1 = S.rec[i].y;
          const uint32_t blk = rBlk(r1), warp = rWarp(r1);
          const uint32_t tl = rTli(r1) - blk * tpb;
          const uint32_t lane = tl - warp * static_cast<uint32_t>(ws);
          const int w = sParams[sSites[rSite(r0)].param].written - 1;
          const uint64_t off = rElem(r0) - S.minE[w];
          keys[j] = (static_cast<uint64_t>(w) << S.fW) | (off << S.fOff) |
                    (static_cast<uint64_t>(blk) << S.fBlk) |
                    (static_cast<uint64_t>(rBp(r1)) << S.fBp) |
                    (static_cast<uint64_t>(warp) << S.fWarp) |
                    (static_cast<uint64_t>(rWp(r1)) << S.fWp) | lane;
        } else {
          keys[j] = ~0ull;
        }
      }
      typename Smem::Sort(S.u.sortTmp).Sort(keys, vals, 0, S.total > 0 ? S.total : 1);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        S.u.rx.skey[tid * IPT + j] = keys[j];
        S.u.rx.sidx[tid * IPT + j] = vals[j];
      }
      __syncthreads();
      // one thread per element group
      const int shLane = S.fWp, shBpF = S.fBp, shElem = S.fOff;
      for (int j = 0; j < IPT; ++j) {
        const int p = tid * IPT + j;
        if (p >= static_cast<int>(n) || S.u.rx.skey[p] == ~0ull)
          break; // unfilled slots sort last
        const uint64_t g = S.u.rx.skey[p] >> shElem;
        if (p > 0 && (S.u.rx.skey[p - 1] >> shElem) == g)
          continue;
        int e = p + 1;
        while (e < static_cast<int>(n) && (S.u.rx.skey[e] >> shElem) == g)
          ++e;
        if (e - p < 2)
          continue;
        uint32_t mn2[kMaxSites], mx2[kMaxSites], mn3[kMaxSites], mx3[kMaxSites];
        uint64_t p2 = 0, p3 = 0;
        uint64_t g2 = S.u.rx.skey[p] >> shBpF, g3 = S.u.rx.skey[p] >> shLane;
        auto flush = [&](uint64_t pres, const uint32_t *mn, const uint32_t *mx, int kind) {
          uint64_t rem = pres;
          while (rem) {
            const int a = __ffsll(static_cast<long long>(rem)) - 1;
            rem &= rem - 1;
            uint64_t mm = sConf[a] & pres & ~((1ull << a) - 1);
            while (mm) {
              const int b = __ffsll(static_cast<long long>(mm)) - 1;
              mm &= mm - 1;
              if (min(mn[a], mn[b]) < max(mx[a], mx[b]))
                noteKey(S, sKeyMin, sReal, keyIndex(sSites, F.nLocs, a, b, kind),
                        static_cast<uint32_t>(p));
            }
          }
        };
        for (int q = p; q < e; ++q) {
          const uint64_t k = S.u.rx.skey[q];
          if ((k >> shBpF) != g2) {
            flush(p2, mn2, mx2, 1);
            p2 = 0;
            g2 = k >> shBpF;
          }
          if ((k >> shLane) != g3) {
            flush(p3, mn3, mx3, 2);
            p3 = 0;
            g3 = k >> shLane;
          }
          const uint32_t ri = S.u.rx.sidx[q];
          const int s = rSite(S.rec[ri].x);
          const uint64_t r1 = S.rec[ri].y;
          const uint32_t wq = rWarp(r1);
          const uint32_t tl = rTli(r1) - rBlk(r1) * tpb;
          note(p2, mn2, mx2, s, wq);
          note(p3, mn3, mx3, s, tl - wq * static_cast<uint32_t>(ws));
        }
        flush(p2, mn2, mx2, 1);
        flush(p3, mn3, mx3, 2);
      }
      __syncthreads();
    }
    // 2. witnesses of the keys realised in this iteration
    const unsigned nReal = S.nReal;
    for (unsigned r = tid; r < nReal; r += kFusedThreads) {
      const int K = static_cast<int>(sReal[r]);
      const int kind = K % 3;
      const int la = (K / 3) / F.nLocs, lb = (K / 3) % F.nLocs;
      const uint32_t v = sKeyMin[K];
      sKeyMin[K] = ~0u; // reset for the next iteration
      // the key's minimum element in this iteration: its records are the
      // slot chain (hash mode) or a sorted range (radix mode)
      uint32_t ge;
      uint32_t g0 = 0, g1 = 0;
      if (hashed) {
        ge = v;
      } else {
        g0 = v;
        ge = rElem(S.rec[S.u.rx.sidx[g0]].x);
        const uint64_t g = S.u.rx.skey[g0] >> S.fOff;
        g1 = g0 + 1;
        while (g1 < n && (S.u.rx.skey[g1] >> S.fOff) == g)
          ++g1;
      }
      if (ge > sKeyBound[K])
        continue; // a smaller element for K is known
      {
        const unsigned long long g = __ldcg(&F.keyElem[K]);
        if (ge > g) { // another block already holds a smaller element for K
          sKeyBound[K] = static_cast<uint32_t>(g);
          continue;
        }
      }
      uint32_t mem[kSmallGroup + 1];
      int nm = 0;
      if (hashed) {
        for (uint32_t q = S.u.ch.head[hashSlot<Smem>(ge)]; q != Smem::kEnd && nm <= kSmallGroup;
             q = S.u.ch.next[q])
          if (rElem(S.rec[q].x) == ge)
            mem[nm++] = q;
      }
      const int cnt = hashed ? nm : static_cast<int>(g1 - g0);
      auto rec = [&](int i) -> uint32_t { return hashed ? mem[i] : S.u.rx.sidx[g0 + i]; };
      uint64_t bestX = ~0ull, bestY = ~0ull;
      int sX = 0, sY = 0;
      auto order = [&](uint64_t r0, uint64_t r1) {
        const uint64_t thread = static_cast<uint64_t>(firstBlock * L.tpb) + rTli(r1);
        return (thread << kSeqBits) | rSeq(r0);
      };
      // lexicographically first (x, y) over the element's racing pairs of K
      for (int a = 0; a < cnt; ++a) {
        const uint64_t a0 = S.rec[rec(a)].x, a1 = S.rec[rec(a)].y;
        const int sa = rSite(a0);
        const int loa = sSites[sa].loc;
        if (loa != la && loa != lb)
          continue;
        const uint64_t oa = order(a0, a1);
        if (oa > bestX)
          continue;
        for (int b = 0; b < cnt; ++b) {
          if (b == a)
            continue;
          const uint64_t b0 = S.rec[rec(b)].x, b1 = S.rec[rec(b)].y;
          const uint64_t ob = order(b0, b1);
          if (ob <= oa)
            continue; // y must follow x in event order
          const int sb = rSite(b0);
          const int lob = sSites[sb].loc;
          if (!((loa == la && lob == lb) || (loa == lb && lob == la)))
            continue;
          if (kind == 0) { // interOnChip: other block, conflicting across blocks
            if (rBlk(a1) == rBlk(b1) || !((sConfX[sa] >> sb) & 1ull))
              continue;
          } else if (!((sConf[sa] >> sb) & 1ull) || intraRule(a1, b1) != kind) {
            continue;
          }
          if (oa < bestX || (oa == bestX && ob < bestY)) {
            bestX = oa;
            bestY = ob;
            sX = sa;
            sY = sb;
          }
        }
      }
      const unsigned long long old = atomicMin(&F.keyElem[K], static_cast<unsigned long long>(ge));
      sKeyBound[K] = old < ge ? static_cast<uint32_t>(old) : ge;
      if (ge <= old) {
        const unsigned c = atomicAdd(F.candCount, 1u);
        if (c < F.candCap) {
          F.cand[c] = Candidate{K, sX, sY, 0, ge, bestX, bestY};
          wroteCand = true;
        } else {
          myFlags |= kFlagFusedOverflow;
        }
      }
    }
  }
  pend.settle(myFlags, sKnown, F.epoch << 20);
  pend2.settle(myFlags, sKnown, F.epoch << 20);
  // counters
  __syncthreads();
  const int lane = tid & 31;
  tally.flags |= myFlags;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tally.steps += __shfl_down_sync(0xffffffffu, tally.steps, o);
    tally.inst += __shfl_down_sync(0xffffffffu, tally.inst, o);
    tally.traps += __shfl_down_sync(0xffffffffu, tally.traps, o);
    tally.recs += __shfl_down_sync(0xffffffffu, tally.recs, o);
    tally.flags |= __shfl_down_sync(0xffffffffu, tally.flags, o);
  }
  if (lane == 0) {
    if (tally.steps)
      atomicAdd(&L.ctr->steps, tally.steps);
    if (tally.inst)
      atomicAdd(&L.ctr->instances, tally.inst);
    if (tally.traps)
      atomicAdd(&L.ctr->traps, tally.traps);
    if (tally.recs)
      atomicAdd(&L.ctr->records, tally.recs);
    if (tally.flags)
      atomicOr(&L.ctr->flags, tally.flags);
  }
  if (tid == 0 && S.flags)
    atomicOr(&L.ctr->flags, S.flags);

  // The last CTA to finish turns the candidates into race records: per key,
  // the lexicographically first pair of the key's minimum element.
  __shared__ bool amLast;
  if (wroteCand) // candidate stores visible device-wide before this CTA counts as done
    __threadfence();
  __syncthreads();
  if (tid == 0)
    amLast = atomicAdd(&L.ctr->doneCtas, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!amLast)
    return;
  __threadfence();
  const unsigned nc = min(atomicAdd(F.candCount, 0u), F.candCap);
  const int wid = tid >> 5;
  // realised keys first, all threads at once (one load latency instead of
  // one per key and warp: this is the kernel's serial tail), listed in sReal
  __shared__ unsigned sFinN;
  if (tid == 0)
    sFinN = 0;
  __syncthreads();
  for (int K = tid; K < F.nKeys; K += kFusedThreads)
    if (__ldcg(&F.keyElem[K]) != ~0ull)
      sReal[atomicAdd(&sFinN, 1u)] = static_cast<uint32_t>(K);
  __syncthreads();
  for (unsigned r = wid; r < sFinN; r += kFusedThreads / 32) {
    const int K = static_cast<int>(sReal[r]);
    const unsigned long long e = __ldcg(&F.keyElem[K]);
    uint64_t x = ~0ull, y = ~0ull;
    int sx = 0, sy = 0;
    for (unsigned c = lane; c < nc; c += 32) {
      const Candidate *cd = &F.cand[c];
      if (__ldcg(&cd->key) != K || __ldcg(&cd->elem) != e)
        continue;
      const uint64_t cx = __ldcg(&cd->xOrd), cy = __ldcg(&cd->yOrd);
      if (cx < x || (cx == x && cy < y)) {
        x = cx;
        y = cy;
        sx = __ldcg(&cd->siteX);
        sy = __ldcg(&cd->siteY);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ox = __shfl_down_sync(0xffffffffu, x, o);
      const uint64_t oy = __shfl_down_sync(0xffffffffu, y, o);
      const int osx = __shfl_down_sync(0xffffffffu, sx, o);
      const int osy = __shfl_down_sync(0xffffffffu, sy, o);
      if (ox < x || (ox == x && oy < y)) {
        x = ox;
        y = oy;
        sx = osx;
        sy = osy;
      }
    }
    if (lane == 0) {
      const unsigned pos = atomicAdd(&L.ctr->nRaces, 1u);
      hgrd_gpu_race &o = F.races[pos];
      o.kind = K % 3;
      o.loc_a = (K / 3) / F.nLocs;
      o.loc_b = (K / 3) % F.nLocs;
      o.site_x = sx;
      o.site_y = sy;
      int w = 0;
      for (int q = 1; q < F.nW; ++q)
        if (F.wBase[q] <= e)
          w = q;
      o.handle = F.wHandle[w];
      o.index = static_cast<int64_t>(e - F.wBase[w]);
      o.thread_x = static_cast<int64_t>(x >> kSeqBits);
      o.seq_x = static_cast<int32_t>(x & kSeqMask);
      o.thread_y = static_cast<int64_t>(y >> kSeqBits);
      o.seq_y = static_cast<int32_t>(y & kSeqMask);
    }
  }
}

} // namespace dev
} // namespace hgrdgpu

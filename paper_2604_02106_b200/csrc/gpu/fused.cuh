// K-fused: block-local race check (PARALLEL launches without lock idioms).
//
// One CTA iteration takes one or more whole MiniCU blocks.  Every
// INTRA-BLOCK / INTRA-WARP pair lies inside one MiniCU block
// (reference src/oracle.cpp:754-769), so they are found entirely on chip:
//   1. expansion into shared memory (records: global element id + meta),
//   2. CUB block radix sort by  w | element offset | block | bp | warp | wp | lane
//      (element offsets relative to the iteration's minimum per buffer, so
//      the key is short: 10 bits for the stencil tile),
//   3. per element group: realised INTRA keys (pairwise for small groups,
//      per-site min/max summaries for large ones), minimum element per key,
//   4. per realised key: the first (x, y) pair of the reference's order
//      inside that element, published as a candidate (global element via
//      atomicMin, candidates filtered by it; k_fused_finalize keeps the
//      lexicographically first pair of the minimum element).
// INTER-BLOCK pairs need a second block: every (element, block) also does
// one ownership update on a per-element table (epoch-tagged, no memset);
// an element reached from two blocks becomes MULTI and only MULTI elements
// go through the global record sort (pass 2 in ctx.cu).
#pragma once

#include "detect.cuh"
#include "device.cuh"
#include "expand.cuh"

#include <cub/block/block_radix_sort.cuh>

namespace hgrdgpu {
namespace dev {

constexpr int kFusedThreads = 256;
constexpr int kMaxWritten = 8;
constexpr uint32_t kOwnerMulti = 0xFFFFFu;
constexpr int kSmallGroup = 24; // pairwise below, summaries above

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
  int64_t nIters;
  uint32_t *owner;
  uint32_t epoch;
  unsigned long long *keyElem;
  Candidate *cand;
  uint32_t candCap;
  unsigned int *candCount;
  int nW;
};

// One exchange per (element, block): whoever replaces another block's tag
// (or MULTI) marks the element MULTI.  The last exchange on an element that
// two blocks touched is always followed by a MULTI store, so the final value
// is MULTI exactly for the elements of >= 2 blocks.
__device__ __forceinline__ void ownerUpdate(const FusedArgs &F, uint64_t e, uint64_t blk,
                                            unsigned &flags) {
  const uint32_t tag = F.epoch << 20;
  const uint32_t mine = static_cast<uint32_t>(blk + 1);
  const uint32_t old = atomicExch(&F.owner[e], tag | mine);
  if ((old >> 20) == F.epoch && (old & kOwnerMulti) != mine) {
    atomicExch(&F.owner[e], tag | kOwnerMulti);
    flags |= kFlagShared;
  }
}

template <int IPT> struct FusedSmem {
  static constexpr int kCap = kFusedThreads * IPT;
  static constexpr int kTable = 2 * kCap; // counting-sort slots (element span)
  using Sort = cub::BlockRadixSort<uint64_t, kFusedThreads, IPT, uint32_t, 6>;
  union {
    typename Sort::TempStorage sortTmp;
    struct {
      uint32_t cnt[kTable]; // per element slot: count, then start
      uint16_t rank[kCap];  // record's rank inside its slot
      uint32_t part[kFusedThreads];
    } cs;
  } u;
  uint64_t elem[kCap];  // global element id, by record index
  uint64_t meta[kCap];  // tli:16 | bp:8 | wp:8 | site:12 | seq:20
  uint64_t key[kCap];   // sorted keys (counting mode: element slot)
  uint32_t idx[kCap];   // sorted -> record index
  unsigned long long minE[kMaxWritten], maxE[kMaxWritten];
  uint32_t prefix[kMaxWritten];
  unsigned int count, maxBp, maxWp, nReal, flags, maxGroup;
  int counting; // this iteration groups by a counting sort over element slots
  // field start bits of the block-local key  w|off|blk|bp|warp|wp|lane
  int fWp, fWarp, fBp, fBlk, fOff, fW, total;
};

__device__ __forceinline__ uint64_t packMeta(uint32_t tli, uint32_t bp, uint32_t wp, int site,
                                             uint32_t seq) {
  return (static_cast<uint64_t>(tli) << 48) | (static_cast<uint64_t>(bp & 255) << 40) |
         (static_cast<uint64_t>(wp & 255) << 32) | (static_cast<uint64_t>(site & 4095) << 20) |
         (seq & kSeqMask);
}
__device__ __forceinline__ uint32_t metaTli(uint64_t m) { return static_cast<uint32_t>(m >> 48); }
__device__ __forceinline__ uint32_t metaBp(uint64_t m) { return (m >> 40) & 255; }
__device__ __forceinline__ uint32_t metaWp(uint64_t m) { return (m >> 32) & 255; }
__device__ __forceinline__ int metaSite(uint64_t m) { return static_cast<int>((m >> 20) & 4095); }
__device__ __forceinline__ uint32_t metaSeq(uint64_t m) { return static_cast<uint32_t>(m & kSeqMask); }

// PARALLEL sink of the fused kernel: records into shared memory.
template <int IPT> struct FusedSink : ParState {
  FusedSmem<IPT> *S;
  uint32_t tli; // thread index within the iteration

  __device__ __forceinline__ void record(int site, const ParamDev *P, int64_t idx) {
    if (!sites[site].record)
      return;
    if (bp > 255 || wp > 255 || seq > kSeqMask || site > kMaxSiteId)
      flags |= kFlagFusedOverflow;
    // warp-aggregated slot allocation (one shared atomic per converged group)
    const unsigned act = __activemask();
    const int ln = threadIdx.x & 31;
    const int leader = __ffs(act) - 1;
    unsigned base = 0;
    if (ln == leader)
      base = atomicAdd(&S->count, static_cast<unsigned>(__popc(act)));
    base = __shfl_sync(act, base, leader);
    const unsigned pos = base + __popc(act & ((1u << ln) - 1));
    if (pos < static_cast<unsigned>(FusedSmem<IPT>::kCap)) {
      S->elem[pos] = P->elemBase + static_cast<uint64_t>(idx);
      S->meta[pos] = packMeta(tli, bp, wp, site, seq);
    } else {
      flags |= kFlagFusedOverflow;
    }
    ++recs;
  }
  __device__ __forceinline__ int64_t load(int site, int64_t idx, bool need) {
    const ParamDev *P = check(site, idx);
    if (!P)
      return 0;
    record(site, P, idx);
    ++seq;
    return need ? __ldg(P->ptr + idx) : 0;
  }
  __device__ __forceinline__ void store(int site, int64_t idx, int64_t) {
    const ParamDev *P = check(site, idx);
    if (!P)
      return;
    record(site, P, idx);
    ++seq;
  }
  __device__ __forceinline__ void atomic(int site, int64_t idx, int64_t, int64_t) {
    store(site, idx, 0);
  }
};

// Conditions of the reference pair rule for two records of one element
// inside one MiniCU block (:750-769), INTRA kinds only.  Returns kind or -1.
__device__ __forceinline__ int intraKind(const LaunchDev &L, const SiteDev *sites, uint64_t ma,
                                         uint64_t mb, uint32_t tpb, int64_t ws) {
  const uint32_t ta = metaTli(ma), tb = metaTli(mb);
  if (ta == tb)
    return -1;
  const uint32_t ba = L.dTpb.div(ta), bb = L.dTpb.div(tb);
  if (ba != bb)
    return -1; // different MiniCU blocks: INTER, handled by ownership
  const SiteDev &sa = sites[metaSite(ma)], &sb = sites[metaSite(mb)];
  if (sa.kind == HGRD_SITE_LOAD && sb.kind == HGRD_SITE_LOAD)
    return -1;
  if (sa.kind == HGRD_SITE_ATOMIC && sb.kind == HGRD_SITE_ATOMIC && sa.scope != HGRD_SCOPE_NONE &&
      sb.scope != HGRD_SCOPE_NONE)
    return -1;
  if (metaBp(ma) != metaBp(mb))
    return -1;
  const uint32_t wa = L.dWs.div(ta - ba * tpb), wb = L.dWs.div(tb - bb * tpb);
  if (wa == wb && metaWp(ma) != metaWp(mb))
    return -1;
  return wa != wb ? 1 : 2;
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

template <int IPT>
__device__ __forceinline__ void noteKey(FusedSmem<IPT> &S, uint32_t *sKeyMin, uint32_t *sReal,
                                        int K, uint32_t pos) {
  if (sKeyMin[K] <= pos)
    return;
  const uint32_t old = atomicMin(&sKeyMin[K], pos);
  if (old == 0xffffffffu) {
    const unsigned slot = atomicAdd(&S.nReal, 1u);
    sReal[slot] = static_cast<uint32_t>(K);
  }
}

template <int IPT, class Body>
__global__ void __launch_bounds__(kFusedThreads, 3) k_fused(FusedArgs F) {
  using Smem = FusedSmem<IPT>;
  extern __shared__ __align__(16) unsigned char dyn[];
  Smem &S = *reinterpret_cast<Smem *>(dyn);
  unsigned char *after = dyn + ((sizeof(Smem) + 15) & ~size_t(15));
  const int nKeysPad = (F.nKeys + 3) & ~3;
  uint32_t *sKeyMin = reinterpret_cast<uint32_t *>(after);
  uint32_t *sReal = sKeyMin + nKeysPad;
  hgrd_gpu_insn *sCode = reinterpret_cast<hgrd_gpu_insn *>(sReal + nKeysPad);
  SiteDev *sSites = reinterpret_cast<SiteDev *>(sCode + F.L.nCode);
  ParamDev *sParams = reinterpret_cast<ParamDev *>(sSites + F.L.nSites);
  uint64_t *sConf = reinterpret_cast<uint64_t *>(sParams + F.L.nParams);
  // dynamic shared memory layout mirrored by fusedSmemBytes() in ctx.cu
  const LaunchDev &L = F.L;
  const int tid = threadIdx.x;
  for (int i = tid; i < L.nCode; i += kFusedThreads)
    sCode[i] = L.code[i];
  for (int i = tid; i < L.nSites; i += kFusedThreads) {
    sSites[i] = L.sites[i];
    sConf[i] = L.confIntra[i];
  }
  for (int i = tid; i < L.nParams; i += kFusedThreads)
    sParams[i] = L.params[i];
  for (int i = tid; i < F.nKeys; i += kFusedThreads)
    sKeyMin[i] = 0xffffffffu;
  if (tid == 0) {
    S.nReal = 0;
    S.flags = 0;
  }
  const uint32_t tpb = static_cast<uint32_t>(L.tpb);
  const int64_t ws = L.ws;
  LaneTally tally;
  unsigned myFlags = 0;
  int64_t regs[kMaxRegs];

  for (int64_t it = blockIdx.x; it < F.nIters; it += gridDim.x) {
    const int64_t firstBlock = it * F.bpi;
    const int64_t nb = min(static_cast<int64_t>(F.bpi), L.nBlocks - firstBlock);
    __syncthreads();
    if (tid == 0) {
      S.count = 0;
      S.maxBp = 0;
      S.maxWp = 0;
    }
    if (tid < kMaxWritten) {
      S.minE[tid] = ~0ull;
      S.maxE[tid] = 0;
    }
    __syncthreads();
    // 1. expansion of the iteration's whole MiniCU blocks
    for (int64_t tl = tid; tl < nb * L.tpb; tl += kFusedThreads) {
      FusedSink<IPT> s;
      s.L = &L;
      s.sites = sSites;
      s.params = sParams;
      s.S = &S;
      s.tli = static_cast<uint32_t>(tl);
      Builtins bi;
      threadIdentity(L, firstBlock * L.tpb + tl, bi, s.block, s.warp, s.lane);
      Body::run(L, sCode, bi, s, regs);
      tally.add(s);
      atomicMax(&S.maxBp, s.bp);
      atomicMax(&S.maxWp, s.wp);
    }
    __syncthreads();
    // per written buffer: the iteration's element range (warp reduction)
    {
      const unsigned nr = min(S.count, static_cast<unsigned>(Smem::kCap));
      unsigned long long lo[kMaxWritten], hi[kMaxWritten];
#pragma unroll
      for (int q = 0; q < kMaxWritten; ++q) {
        lo[q] = ~0ull;
        hi[q] = 0;
      }
      for (unsigned i = tid; i < nr; i += kFusedThreads) {
        const int w = sParams[sSites[metaSite(S.meta[i])].param].written - 1;
        const unsigned long long e = S.elem[i];
#pragma unroll
        for (int q = 0; q < kMaxWritten; ++q)
          if (q == w) {
            lo[q] = min(lo[q], e);
            hi[q] = max(hi[q], e);
          }
      }
#pragma unroll
      for (int q = 0; q < kMaxWritten; ++q) {
        if (q >= F.nW)
          break;
        for (int o = 16; o > 0; o >>= 1) {
          lo[q] = min(lo[q], __shfl_down_sync(0xffffffffu, lo[q], o));
          hi[q] = max(hi[q], __shfl_down_sync(0xffffffffu, hi[q], o));
        }
        if ((tid & 31) == 0 && lo[q] <= hi[q]) {
          atomicMin(&S.minE[q], lo[q]);
          atomicMax(&S.maxE[q], hi[q]);
        }
      }
    }
    __syncthreads();
    const unsigned n = min(S.count, static_cast<unsigned>(Smem::kCap));
    if (S.count > static_cast<unsigned>(Smem::kCap))
      myFlags |= kFlagFusedOverflow;
    if (n == 0)
      continue;
    // 2. grouping by element: counting sort over element slots when the
    //    iteration's element span is small and groups are small, else a
    //    CUB block radix sort of the full key
    if (tid == 0) {
      uint32_t span = 0;
      bool ok = true;
      for (int w = 0; w < F.nW && w < kMaxWritten; ++w) {
        S.prefix[w] = span;
        if (S.minE[w] <= S.maxE[w]) {
          const unsigned long long sw = S.maxE[w] - S.minE[w] + 1;
          if (sw > static_cast<unsigned long long>(Smem::kTable))
            ok = false;
          else
            span += static_cast<uint32_t>(sw);
        }
      }
      S.counting = ok && span <= static_cast<uint32_t>(Smem::kTable);
      S.total = static_cast<int>(span); // slots in counting mode
      S.maxGroup = 0;
    }
    __syncthreads();
    if (S.counting) {
      const int slots = S.total;
      for (int i = tid; i < slots; i += kFusedThreads)
        S.u.cs.cnt[i] = 0;
      __syncthreads();
      unsigned myMax = 0;
      for (unsigned i = tid; i < n; i += kFusedThreads) {
        const int w = sParams[sSites[metaSite(S.meta[i])].param].written - 1;
        const uint32_t slot = S.prefix[w] + static_cast<uint32_t>(S.elem[i] - S.minE[w]);
        const unsigned r = atomicAdd(&S.u.cs.cnt[slot], 1u);
        S.u.cs.rank[i] = static_cast<uint16_t>(r);
        myMax = max(myMax, r + 1);
      }
      if (myMax > kSmallGroup)
        atomicMax(&S.maxGroup, myMax);
      __syncthreads();
      if (S.maxGroup <= kSmallGroup) {
        // exclusive scan of the slot counts: per-thread chunks + warp scans
        const int per = (slots + kFusedThreads - 1) / kFusedThreads;
        const int b0 = min(slots, tid * per), b1 = min(slots, b0 + per);
        uint32_t sum = 0;
        for (int i = b0; i < b1; ++i)
          sum += S.u.cs.cnt[i];
        S.u.cs.part[tid] = sum;
        __syncthreads();
        if (tid < 32) {
          uint32_t acc = 0;
          for (int k = 0; k < kFusedThreads / 32; ++k) {
            const uint32_t v = S.u.cs.part[k * 32 + tid];
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
              if (tid >= o)
                incl += y;
            }
            S.u.cs.part[k * 32 + tid] = acc + incl - v;
            acc += __shfl_sync(0xffffffffu, incl, 31);
          }
        }
        __syncthreads();
        uint32_t run = S.u.cs.part[tid];
        for (int i = b0; i < b1; ++i) {
          const uint32_t c0 = S.u.cs.cnt[i];
          S.u.cs.cnt[i] = run;
          run += c0;
        }
        __syncthreads();
        for (unsigned i = tid; i < n; i += kFusedThreads) {
          const int w = sParams[sSites[metaSite(S.meta[i])].param].written - 1;
          const uint32_t slot = S.prefix[w] + static_cast<uint32_t>(S.elem[i] - S.minE[w]);
          const uint32_t pos = S.u.cs.cnt[slot] + S.u.cs.rank[i];
          S.idx[pos] = i;
          S.key[pos] = slot;
        }
        __syncthreads();
      } else if (tid == 0) {
        S.counting = 0; // a hot element: fall back to the radix sort
      }
      __syncthreads();
    }
    if (!S.counting) {
      if (tid == 0) {
        uint64_t span = 1;
        for (int w = 0; w < F.nW && w < kMaxWritten; ++w)
          if (S.minE[w] <= S.maxE[w])
            span = max(span, static_cast<uint64_t>(S.maxE[w] - S.minE[w] + 1));
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
      const int wpShift = S.fWp, warpShift = S.fWarp, bpShift = S.fBp, blkShift = S.fBlk,
                offShift = S.fOff, wShift = S.fW;
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const unsigned i = static_cast<unsigned>(tid * IPT + j);
        vals[j] = i;
        if (i < n) {
          const uint64_t m = S.meta[i];
          const uint32_t tli = metaTli(m);
          const uint32_t blk = L.dTpb.div(tli), tl = tli - blk * tpb;
          const uint32_t warp = L.dWs.div(tl), lane = tl - warp * static_cast<uint32_t>(ws);
          const SiteDev &sd = sSites[metaSite(m)];
          const int w = sParams[sd.param].written - 1;
          const uint64_t off = S.elem[i] - S.minE[w];
          keys[j] = (static_cast<uint64_t>(w) << wShift) | (off << offShift) |
                    (static_cast<uint64_t>(blk) << blkShift) |
                    (static_cast<uint64_t>(metaBp(m)) << bpShift) |
                    (static_cast<uint64_t>(warp) << warpShift) |
                    (static_cast<uint64_t>(metaWp(m)) << wpShift) | lane;
        } else {
          keys[j] = ~0ull;
        }
      }
      typename Smem::Sort(S.u.sortTmp).Sort(keys, vals, 0, S.total > 0 ? S.total : 1);
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        S.key[tid * IPT + j] = keys[j];
        S.idx[tid * IPT + j] = vals[j];
      }
      __syncthreads();
    }
    // group keys of the sorted key (counting mode: the key is the element slot)
    const bool counting = S.counting != 0;
    const int shLane = S.fWp;                 // element|blk|bp|warp|wp  (INTRA-WARP group)
    const int shBpF = S.fBp;                  // element|blk|bp          (INTRA-BLOCK group)
    const int shElem = counting ? 0 : S.fOff; // element
    // 4. per element group: ownership + INTRA keys
    for (int j = 0; j < IPT; ++j) {
      const int p = tid * IPT + j;
      if (p >= static_cast<int>(n))
        break;
      const uint64_t g = S.key[p] >> shElem;
      if (p > 0 && (S.key[p - 1] >> shElem) == g)
        continue;
      int e = p + 1;
      while (e < static_cast<int>(n) && (S.key[e] >> shElem) == g)
        ++e;
      const uint64_t ge = S.elem[S.idx[p]];
      // ownership per (element, block)
      for (int q = p; q < e; ++q) {
        const uint32_t bq = L.dTpb.div(metaTli(S.meta[S.idx[q]]));
        bool seen = false;
        for (int r2 = p; r2 < q && !seen; ++r2)
          seen = L.dTpb.div(metaTli(S.meta[S.idx[r2]])) == bq;
        if (!seen)
          ownerUpdate(F, ge, static_cast<uint64_t>(firstBlock + bq), myFlags);
      }
      if (e - p < 2)
        continue;
      if (e - p <= kSmallGroup) {
        for (int a = p; a < e; ++a) {
          const uint64_t ma = S.meta[S.idx[a]];
          for (int b = a + 1; b < e; ++b) {
            const uint64_t mb = S.meta[S.idx[b]];
            const int kind = intraKind(L, sSites, ma, mb, tpb, ws);
            if (kind < 0)
              continue;
            const int sa = metaSite(ma), sb = metaSite(mb);
            if (!((sConf[sa] >> sb) & 1ull))
              continue;
            noteKey(S, sKeyMin, sReal, keyIndex(sSites, F.nLocs, sa, sb, kind),
                    static_cast<uint32_t>(p));
          }
        }
      } else {
        // summaries: per site (min,max) warp at (element,blk,bp), lane at (..,warp,wp)
        uint32_t mn2[kMaxSites], mx2[kMaxSites], mn3[kMaxSites], mx3[kMaxSites];
        uint64_t p2 = 0, p3 = 0;
        uint64_t g2 = S.key[p] >> shBpF, g3 = S.key[p] >> shLane;
        auto flush = [&](uint64_t pres, const uint32_t *mn, const uint32_t *mx, int kind) {
          uint64_t rem = pres;
          while (rem) {
            const int a = __ffsll(static_cast<long long>(rem)) - 1;
            rem &= rem - 1;
            uint64_t m = sConf[a] & pres & ~((1ull << a) - 1);
            while (m) {
              const int b = __ffsll(static_cast<long long>(m)) - 1;
              m &= m - 1;
              if (min(mn[a], mn[b]) < max(mx[a], mx[b]))
                noteKey(S, sKeyMin, sReal, keyIndex(sSites, F.nLocs, a, b, kind),
                        static_cast<uint32_t>(p));
            }
          }
        };
        for (int q = p; q < e; ++q) {
          const uint64_t k = S.key[q];
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
          const uint64_t m = S.meta[S.idx[q]];
          const int s = metaSite(m);
          const uint32_t tli = metaTli(m);
          const uint32_t tl = tli - L.dTpb.div(tli) * tpb;
          const uint32_t wq = L.dWs.div(tl);
          note(p2, mn2, mx2, s, wq);
          note(p3, mn3, mx3, s, tl - wq * static_cast<uint32_t>(ws));
        }
        flush(p2, mn2, mx2, 1);
        flush(p3, mn3, mx3, 2);
      }
    }
    __syncthreads();
    // 5. witnesses of the keys realised in this iteration
    const unsigned nReal = S.nReal;
    for (unsigned r = tid; r < nReal; r += kFusedThreads) {
      const int K = static_cast<int>(sReal[r]);
      const int kind = K % 3;
      const int la = (K / 3) / F.nLocs, lb = (K / 3) % F.nLocs;
      const int p = static_cast<int>(sKeyMin[K]);
      sKeyMin[K] = 0xffffffffu; // reset for the next iteration
      const uint64_t gElem = S.elem[S.idx[p]];
      if (gElem > F.keyElem[K])
        continue; // another block already holds a smaller element for K
      const uint64_t g = S.key[p] >> shElem;
      int e = p + 1;
      while (e < static_cast<int>(n) && (S.key[e] >> shElem) == g)
        ++e;
      uint64_t bestX = ~0ull, bestY = ~0ull;
      int sX = 0, sY = 0;
      auto order = [&](uint64_t m) {
        const uint64_t thread = static_cast<uint64_t>(firstBlock * L.tpb) + metaTli(m);
        return (thread << kSeqBits) | metaSeq(m);
      };
      // lexicographically first (x, y) over the group's racing pairs of K
      for (int a = p; a < e; ++a) {
        const uint64_t ma = S.meta[S.idx[a]];
        const int sa = metaSite(ma);
        const int loa = sSites[sa].loc;
        if (loa != la && loa != lb)
          continue;
        const uint64_t oa = order(ma);
        if (oa > bestX)
          continue;
        for (int b = p; b < e; ++b) {
          if (b == a)
            continue;
          const uint64_t mb = S.meta[S.idx[b]];
          const uint64_t ob = order(mb);
          if (ob <= oa)
            continue; // y must follow x in event order
          const int sb = metaSite(mb);
          const int lob = sSites[sb].loc;
          if (!((loa == la && lob == lb) || (loa == lb && lob == la)))
            continue;
          if (!((sConf[sa] >> sb) & 1ull))
            continue;
          if (intraKind(L, sSites, ma, mb, tpb, ws) != kind)
            continue;
          if (oa < bestX || (oa == bestX && ob < bestY)) {
            bestX = oa;
            bestY = ob;
            sX = sa;
            sY = sb;
          }
        }
      }
      const uint64_t ge = S.elem[S.idx[p]];
      const unsigned long long old = atomicMin(&F.keyElem[K], static_cast<unsigned long long>(ge));
      if (ge <= old) {
        const unsigned c = atomicAdd(F.candCount, 1u);
        if (c < F.candCap)
          F.cand[c] = Candidate{K, sX, sY, 0, ge, bestX, bestY};
        else
          myFlags |= kFlagFusedOverflow;
      }
    }
    if (tid == 0)
      S.nReal = 0;
  }
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
}

// One block per key: the lexicographically first candidate pair of the
// key's minimum element becomes the race record.
__global__ void k_fused_finalize(FusedArgs F, DetectArgs A, hgrd_gpu_race *races) {
  const int K = blockIdx.x;
  const unsigned long long e = F.keyElem[K];
  if (e == ~0ull)
    return;
  const unsigned nc = min(*F.candCount, F.candCap);
  __shared__ uint64_t bx[32], by[32];
  __shared__ int bs[32], bt[32];
  uint64_t x = ~0ull, y = ~0ull;
  int sx = 0, sy = 0;
  for (unsigned c = threadIdx.x; c < nc; c += blockDim.x) {
    const Candidate &cd = F.cand[c];
    if (cd.key != K || cd.elem != e)
      continue;
    if (cd.xOrd < x || (cd.xOrd == x && cd.yOrd < y)) {
      x = cd.xOrd;
      y = cd.yOrd;
      sx = cd.siteX;
      sy = cd.siteY;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
    bx[wid] = x;
    by[wid] = y;
    bs[wid] = sx;
    bt[wid] = sy;
  }
  __syncthreads();
  if (threadIdx.x != 0)
    return;
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
    if (bx[w] < x || (bx[w] == x && by[w] < y)) {
      x = bx[w];
      y = by[w];
      sx = bs[w];
      sy = bt[w];
    }
  const unsigned pos = atomicAdd(&F.L.ctr->nRaces, 1u);
  hgrd_gpu_race &o = races[pos];
  o.kind = K % 3;
  o.loc_a = (K / 3) / F.nLocs;
  o.loc_b = (K / 3) % F.nLocs;
  o.site_x = sx;
  o.site_y = sy;
  elementOf(A, e, o.handle, o.index);
  o.thread_x = static_cast<int64_t>(x >> kSeqBits);
  o.seq_x = static_cast<int32_t>(x & kSeqMask);
  o.thread_y = static_cast<int64_t>(y >> kSeqBits);
  o.seq_y = static_cast<int32_t>(y & kSeqMask);
}

} // namespace dev
} // namespace hgrdgpu

// K-batch: many tiny PARALLEL launches checked by one kernel launch
// (sweeps: BASELINE configs 1 and 5, reference enumerateVerdict
// src/oracle.cpp:863-903, where every configuration's launches have a few
// dozen MiniCU threads).
//
// Each launch fits one CTA iteration of the fused kernel (fused.cuh), so a
// CTA checks a whole launch on chip: the expansion pushes every record onto
// its element's hash chain and pairs it with the earlier records of the
// element under the reference's pair rule (:745-769) — INTRA kinds through
// the XOR rule, INTER-BLOCK through the cross-block conflict mask (all the
// launch's blocks are in the CTA) — and keeps per key the minimum element
// (the reference's first-found element: its ordered map by (handle, index),
// :733-735).  The CTA then finds, per realised key, the first (x, y) pair of
// the reference's event order inside that element and writes the race
// record itself: no global candidates, no ownership table, no second pass.
// CTAs take launches from a global work counter (launch sizes vary).
#pragma once

#include "fused.cuh"

namespace hgrdgpu {
namespace dev {

constexpr int kBatchThreads = 256;
constexpr int kBatchIPT = 8; // 2048 records per launch
using BatchSmem = FusedSmem<kBatchThreads, kBatchIPT>;
constexpr int kBatchMaxThreads = 2 * kBatchThreads; // MiniCU threads per launch
constexpr int kBatchMaxBlocks = kMaxIterBlocks;     // the records' 8-bit block field
constexpr int kBatchTraps = 1024;                   // traps per launch kept on chip

struct BatchLaunch {
  LaunchDev L;           // code / sites / params / regInit / conflict masks in the batch blob
  const uint64_t *wBase; // element base of each written buffer
  int32_t nW;
  int32_t nLocs;
  uint32_t R;       // static records per MiniCU thread (0: allocate)
  uint32_t raceOff; // this launch's first race slot
};

struct BatchOut {
  unsigned long long steps, instances, records, traps;
  unsigned int flags, nRaces;
  unsigned int trapOff, nTraps; // this launch's trap entries in the trap area
};

struct BatchArgs {
  const BatchLaunch *launches;
  unsigned n;
  BatchOut *out;
  hgrd_gpu_race *races;
  unsigned *next; // work counter
  uint64_t *trapKey; // trap area (all launches): key, site << 1 | unallocated
  uint32_t *trapSite;
  unsigned *trapCursor;
  unsigned trapCap;
  int maxKeys, maxCode, maxSites, maxParams, maxW;
};

__global__ void __launch_bounds__(kBatchThreads, 2) k_batch(BatchArgs A) {
  constexpr int NT = kBatchThreads;
  extern __shared__ __align__(16) unsigned char dyn[];
  BatchSmem &S = *reinterpret_cast<BatchSmem *>(dyn);
  unsigned char *after = dyn + ((sizeof(BatchSmem) + 15) & ~size_t(15));
  const int keysPad = (A.maxKeys + 3) & ~3;
  uint32_t *sKeyMin = reinterpret_cast<uint32_t *>(after);
  uint32_t *sReal = sKeyMin + keysPad;
  hgrd_gpu_insn *sCode = reinterpret_cast<hgrd_gpu_insn *>(sReal + keysPad);
  SiteDev *sSites = reinterpret_cast<SiteDev *>(sCode + A.maxCode);
  ParamDev *sParams = reinterpret_cast<ParamDev *>(sSites + A.maxSites);
  uint64_t *sConf = reinterpret_cast<uint64_t *>(sParams + A.maxParams);
  uint64_t *sConfX = sConf + A.maxSites;
  uint64_t *sWBase = sConfX + A.maxSites;
  // dynamic shared memory layout mirrored by batchSmemBytes() in ctx.cu
  __shared__ LaunchDev sL;
  __shared__ unsigned sLaunch, sFlags, sNRaces;
  __shared__ unsigned long long sSteps, sInst, sTraps, sRecs;
  __shared__ uint64_t sTrapKey[kBatchTraps];
  __shared__ uint32_t sTrapSite[kBatchTraps];
  __shared__ unsigned sTrapN, sTrapOff;
  const int tid = threadIdx.x;
  int64_t regs[kMaxRegs];

  for (;;) {
    if (tid == 0)
      sLaunch = atomicAdd(A.next, 1u);
    __syncthreads();
    const unsigned li = sLaunch;
    if (li >= A.n)
      return;
    const BatchLaunch &B = A.launches[li];
    {
      const uint32_t *src = reinterpret_cast<const uint32_t *>(&B.L);
      uint32_t *dst = reinterpret_cast<uint32_t *>(&sL);
      for (unsigned i = tid; i < sizeof(LaunchDev) / 4; i += NT)
        dst[i] = src[i];
    }
    const int nLocs = B.nLocs;
    const int nKeys = 3 * nLocs * nLocs;
    const int nW = B.nW;
    const uint32_t R = B.R;
    __syncthreads();
    const int nCode = sL.nCode, nSites = sL.nSites, nParams = sL.nParams;
    for (int i = tid; i < nCode; i += NT)
      sCode[i] = sL.code[i];
    for (int i = tid; i < nSites; i += NT) {
      sSites[i] = sL.sites[i];
      sConf[i] = sL.confIntra[i];
      sConfX[i] = sL.confInter[i];
    }
    for (int i = tid; i < nParams; i += NT)
      sParams[i] = sL.params[i];
    for (int i = tid; i < nW; i += NT)
      sWBase[i] = B.wBase[i];
    for (int i = tid; i < nKeys; i += NT)
      sKeyMin[i] = ~0u;
    for (int i = tid; i < BatchSmem::kTable; i += NT)
      S.u.ch.head[i] = BatchSmem::kEnd;
    const uint32_t nThreads = static_cast<uint32_t>(sL.nThreads);
    if (tid == 0) {
      S.count = R ? nThreads * R : 0;
      S.hot = 0;
      S.nReal = 0;
      S.flags = 0;
      sFlags = 0;
      sNRaces = 0;
      sTrapN = 0;
      sSteps = sInst = sTraps = sRecs = 0;
    }
    __syncthreads();

    // 1. expansion + detection at push time (FusedSink, INTER on chip)
    unsigned long long steps = 0, inst = 0, traps = 0, recs = 0;
    unsigned flags = 0;
    for (uint32_t tl = tid; tl < nThreads; tl += NT) {
      FusedSink<BatchSmem> s;
      s.L = &sL;
      s.sites = sSites;
      s.params = sParams;
      s.S = &S;
      s.tli = tl;
      s.R = R;
      s.stride = nThreads;
      s.myBlk = sL.dTpb.div(tl);
      s.nLocs = nLocs;
      s.keyMin = sKeyMin;
      s.real = sReal;
      s.conf = sConf;
      s.confX = sConfX;
      s.interOnChip = true;
      s.owner = nullptr;
      s.epochTag = 0;
      s.mine = 0;
      s.trapKey = sTrapKey;
      s.trapSite = sTrapSite;
      s.trapCount = &sTrapN;
      s.trapCap = kBatchTraps;
      Builtins bi;
      InterpBody::identity(sL, tl, bi, s.block, s.warp, s.lane);
      InterpBody::run(sL, sCode, bi, s, regs);
      for (uint32_t j = s.nrec; j < R; ++j)
        if (j * nThreads + tl < static_cast<uint32_t>(BatchSmem::kCap))
          S.rec[j * nThreads + tl].x = kNoRec;
      steps += static_cast<unsigned long long>(s.steps);
      inst += s.inst;
      traps += s.traps;
      recs += s.recs;
      flags |= s.flags;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      steps += __shfl_down_sync(0xffffffffu, steps, o);
      inst += __shfl_down_sync(0xffffffffu, inst, o);
      traps += __shfl_down_sync(0xffffffffu, traps, o);
      recs += __shfl_down_sync(0xffffffffu, recs, o);
      flags |= __shfl_down_sync(0xffffffffu, flags, o);
    }
    if ((tid & 31) == 0) {
      if (steps)
        atomicAdd(&sSteps, steps);
      if (inst)
        atomicAdd(&sInst, inst);
      if (traps)
        atomicAdd(&sTraps, traps);
      if (recs)
        atomicAdd(&sRecs, recs);
      if (flags)
        atomicOr(&sFlags, flags);
    }
    __syncthreads();
    if (tid == 0) {
      if (S.count > static_cast<unsigned>(BatchSmem::kCap) || S.hot)
        sFlags |= kFlagFusedOverflow; // (a hot element needs radix grouping: the host re-checks)
      sFlags |= S.flags;
      sTrapOff = 0;
      if (sTrapN > static_cast<unsigned>(kBatchTraps)) {
        sFlags |= kFlagFusedOverflow;
      } else if (sTrapN) {
        sTrapOff = atomicAdd(A.trapCursor, sTrapN);
        if (sTrapOff + sTrapN > A.trapCap)
          sFlags |= kFlagFusedOverflow;
      }
    }
    __syncthreads();
    const bool ok = (sFlags & (kFlagFusedOverflow | kFlagAbort)) == 0;
    if (ok) // the launch's traps, unordered (the host sorts them by key)
      for (unsigned i = tid; i < sTrapN; i += NT) {
        A.trapKey[sTrapOff + i] = sTrapKey[i];
        A.trapSite[sTrapOff + i] = sTrapSite[i];
      }

    // 2. per realised key: the first (x, y) pair of its minimum element
    if (ok) {
      const unsigned nReal = S.nReal;
      for (unsigned r = tid; r < nReal; r += NT) {
        const int K = static_cast<int>(sReal[r]);
        const int kind = K % 3;
        const int la = (K / 3) / nLocs, lb = (K / 3) % nLocs;
        const uint32_t ge = sKeyMin[K];
        uint32_t mem[kSmallGroup + 1];
        int cnt = 0;
        for (uint32_t q = S.u.ch.head[hashSlot<BatchSmem>(ge)];
             q != BatchSmem::kEnd && cnt <= kSmallGroup; q = S.u.ch.next[q])
          if (rElem(S.rec[q].x) == ge)
            mem[cnt++] = q;
        uint64_t bestX = ~0ull, bestY = ~0ull;
        int sX = 0, sY = 0;
        auto order = [&](uint64_t r0, uint64_t r1) {
          return (static_cast<uint64_t>(rTli(r1)) << kSeqBits) | rSeq(r0);
        };
        for (int a = 0; a < cnt; ++a) {
          const uint64_t a0 = S.rec[mem[a]].x, a1 = S.rec[mem[a]].y;
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
            const uint64_t b0 = S.rec[mem[b]].x, b1 = S.rec[mem[b]].y;
            const uint64_t ob = order(b0, b1);
            if (ob <= oa)
              continue; // y follows x in event order
            const int sb = rSite(b0);
            const int lob = sSites[sb].loc;
            if (!((loa == la && lob == lb) || (loa == lb && lob == la)))
              continue;
            if (kind == 0) {
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
        const unsigned pos = atomicAdd(&sNRaces, 1u);
        hgrd_gpu_race &o = A.races[B.raceOff + pos];
        o.kind = kind;
        o.loc_a = la;
        o.loc_b = lb;
        o.site_x = sX;
        o.site_y = sY;
        int w = 0;
        for (int q = 1; q < nW; ++q)
          if (sWBase[q] <= ge)
            w = q;
        o.handle = w;
        o.index = static_cast<int64_t>(ge - sWBase[w]);
        o.thread_x = static_cast<int64_t>(bestX >> kSeqBits);
        o.seq_x = static_cast<int32_t>(bestX & kSeqMask);
        o.thread_y = static_cast<int64_t>(bestY >> kSeqBits);
        o.seq_y = static_cast<int32_t>(bestY & kSeqMask);
      }
    }
    __syncthreads();
    if (tid == 0) {
      BatchOut &o = A.out[li];
      o.steps = sSteps;
      o.instances = sInst;
      o.records = sRecs;
      o.traps = sTraps;
      o.flags = sFlags;
      o.nRaces = ok ? sNRaces : 0;
      o.trapOff = sTrapOff;
      o.nTraps = ok ? sTrapN : 0;
    }
    __syncthreads(); // the next launch reuses the shared state
  }
}

} // namespace dev
} // namespace hgrdgpu

// K1: access-instance expansion.
//
// k_expand_par<Body> — one lane per MiniCU thread, a warp per 32 consecutive
// threads (block-major, so warps of the same MiniCU block stay together),
// grid-stride over the thread space.  Each lane runs the thread body and
// buffers its packed records; at the batch boundary the warp scans the
// per-lane counts and writes them into a per-warp chunk of the record
// arrays reserved with ONE global atomic per >= L.chunk records.  Loads read
// memory only when their value is needed (value-relevant sites of a PARALLEL
// launch read never-written buffers, i.e. the exact launch-entry snapshot);
// stores are not materialised.
//
// k_expand_seq — the reference's canonical order (src/oracle.cpp:440-465)
// with full memory effects, traps in order and the exact step budget; used
// for launches whose loaded values steer addresses or control.
#pragma once

#include "body.cuh"
#include "device.cuh"

namespace hgrdgpu {
namespace dev {

struct LaneRecords {
  uint64_t k[kLaneBuf];
  uint32_t v[kLaneBuf];
  int n;
};

struct LaneTally {
  unsigned long long steps = 0, inst = 0, traps = 0, recs = 0;
  unsigned int maxBp = 0, maxWp = 0, flags = 0;
  __device__ __forceinline__ void add(const ParState &s) {
    steps += static_cast<unsigned long long>(s.steps);
    inst += s.inst;
    traps += s.traps;
    recs += s.recs;
    flags |= s.flags;
    maxBp = max(maxBp, s.bp);
    maxWp = max(maxWp, s.wp);
  }
};

// Per (element, site) block set of the INTER summary: EMPTY, a single block,
// or MULTI.  Atomics only on state changes; repeated blocks are plain reads.
constexpr uint32_t kInterEmpty = 0xffffffffu, kInterMulti = 0xfffffffeu;
__device__ __forceinline__ void interUpdate(uint32_t *w, uint32_t block) {
  uint32_t v = *reinterpret_cast<volatile uint32_t *>(w);
  if (v == block || v == kInterMulti)
    return;
  if (v == kInterEmpty) {
    v = atomicCAS(w, kInterEmpty, block);
    if (v == kInterEmpty || v == block || v == kInterMulti)
      return;
  }
  atomicExch(w, kInterMulti);
}

// Realised INTER keys from the summary table, one thread per element the
// ownership table marks MULTI: sites s1, s2 (static conflict) race across
// blocks iff their block sets' union has two members.  Per key the minimum
// element (the reference's first-found element, :745).
__global__ void k_inter_scan(const uint32_t *owner, uint32_t multiTag, uint64_t nElems,
                             const uint32_t *tab, int nSites, const SiteDev *sites,
                             const uint64_t *confInter, int nLocs,
                             unsigned long long *keyElem) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nElems || !ownerIsMulti(owner, e, multiTag))
    return;
  const uint32_t *w = tab + e * static_cast<uint64_t>(nSites);
  for (int a = 0; a < nSites; ++a) {
    const uint32_t wa = w[a];
    if (wa == kInterEmpty)
      continue;
    for (int b = a; b < nSites; ++b) {
      if (!((confInter[a] >> b) & 1ull))
        continue;
      const uint32_t wb = w[b];
      if (wb == kInterEmpty)
        continue;
      const bool realised = a == b ? wa == kInterMulti
                                   : (wa == kInterMulti || wb == kInterMulti || wa != wb);
      if (!realised)
        continue;
      int la = sites[a].loc, lb = sites[b].loc;
      if (lb < la) {
        const int t = la;
        la = lb;
        lb = t;
      }
      const int K = (la * nLocs + lb) * 3; // kind 0: INTER-BLOCK
      if (__ldcg(&keyElem[K]) > e)
        atomicMin(&keyElem[K], static_cast<unsigned long long>(e));
    }
  }
}

// Written buffers (<= 8) with their single recording site, by value.
struct SingleSites {
  uint64_t wBase[8];
  int32_t site[8]; // -1: no recording site on the buffer
  int nW;
};

// INTER keys without a summary pass, for launches where every buffer two
// blocks can reach has exactly one recording site s: an element is then
// realised for (s, s) iff the ownership table marks it MULTI (two blocks
// reached it, both through s) and s conflicts with itself across blocks.
__global__ void k_inter_scan_single(const uint32_t *owner, uint32_t multiTag, uint64_t nElems,
                                    SingleSites ss, const SiteDev *sites,
                                    const uint64_t *confInter, int nLocs,
                                    unsigned long long *keyElem) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int K = -1;
  if (e < nElems && ownerIsMulti(owner, e, multiTag)) {
    int s = ss.site[0]; // static indices only: the by-value table stays in the parameter bank
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < ss.nW && ss.wBase[q] <= e)
        s = ss.site[q];
    if (s >= 0 && ((confInter[s] >> s) & 1ull))
      K = (sites[s].loc * nLocs + sites[s].loc) * 3; // kind 0: INTER-BLOCK
  }
  // one atomic per key and warp: the lowest lane holds the warp's minimum
  const unsigned act = __ballot_sync(0xffffffffu, K >= 0);
  if (K < 0)
    return;
  const unsigned peers = __match_any_sync(act, K);
  if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1) && __ldcg(&keyElem[K]) > e)
    atomicMin(&keyElem[K], static_cast<unsigned long long>(e));
}

// Empty lo entry of the sharded INTER summary: positive as int32 too, so a
// signed or unsigned MIN all-reduce treats it alike (byte pattern 0x7F).
constexpr uint32_t kShardEmpty = 0x7F7F7F7Fu;

// Sharded INTER summary after the cross-shard MIN/MAX reduction: per
// element, site pairs (a, b) with a static INTER conflict race across
// blocks iff some block of a's set differs from some block of b's set
// (a == b: two distinct blocks).  lo = kShardEmpty marks an empty set.  Per
// key the minimum element (the reference's first-found element, :745).
// (lo / hi: the tables of elements [e0, e0 + nElems))
__global__ void k_inter_scan_minmax(const uint32_t *lo, const uint32_t *hi, uint64_t nElems,
                                    uint64_t e0, int nSites, const SiteDev *sites, const uint64_t *confInter,
                                    int nLocs, unsigned long long *keyElem) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nElems)
    return;
  const uint32_t *l = lo + e * static_cast<uint64_t>(nSites);
  const uint32_t *h = hi + e * static_cast<uint64_t>(nSites);
  for (int a = 0; a < nSites; ++a) {
    const uint32_t la = l[a];
    if (la == kShardEmpty)
      continue;
    const uint32_t ha = h[a];
    for (int b = a; b < nSites; ++b) {
      if (!((confInter[a] >> b) & 1ull))
        continue;
      const uint32_t lb = l[b];
      if (lb == kShardEmpty)
        continue;
      const uint32_t hb = h[b];
      const bool realised = a == b ? la != ha : !(la == ha && lb == hb && la == lb);
      if (!realised)
        continue;
      int ka = sites[a].loc, kb = sites[b].loc;
      if (kb < ka) {
        const int t = ka;
        ka = kb;
        kb = t;
      }
      const int K = (ka * nLocs + kb) * 3; // kind 0: INTER-BLOCK
      if (__ldcg(&keyElem[K]) > e0 + e)
        atomicMin(&keyElem[K], static_cast<unsigned long long>(e0 + e));
    }
  }
}

// PARALLEL sink of k_expand_par: packed records into the lane buffer.
struct ParSink : ParState {
  LaneRecords *out;
  int64_t t = 0;     // global thread (lock launches: op slots)
  uint32_t nOps = 0; // sync ops pushed by this thread

  // PARALLEL lock launches (L->opStride > 0): CAS / Exch / fence ops in the
  // thread's fixed slots, as SeqSink::op does in canonical order (:601-618)
  __device__ __forceinline__ void opPush(int kind, int scope, int handle, int64_t idx,
                                         uint32_t s) {
    if (nOps < L->opStride) {
      const uint64_t slot = static_cast<uint64_t>(t) * L->opStride + nOps;
      L->opMeta[slot] = kind | (scope << 4) | ((handle + 1) << 8);
      L->opIndex[slot] = idx;
      L->opSeq[slot] = static_cast<int32_t>(s);
    } else {
      flags |= kFlagOps;
    }
    ++nOps;
  }
  __device__ __forceinline__ void atomicOp(int site, int param, int64_t idx) {
    const SiteDev &S = sites[site];
    if (S.aop != HGRD_ATOMIC_ADD)
      opPush(S.aop == HGRD_ATOMIC_CAS ? 0 : 1, S.scope, params[param].handle, idx, seq - 1);
  }
  __device__ __forceinline__ void fence(int scope) {
    if (L->opStride)
      opPush(2, scope, -1, 0, seq);
    ++seq;
  }

  __device__ __forceinline__ void record(int site, const ParamDev *P, int64_t idx) {
    recordE(site, P->elemBase + static_cast<uint64_t>(idx), sites[site].own != 0);
  }
  __device__ __forceinline__ void recordE(int site, uint64_t e, bool own) {
    if (L->interLo) { // sharded INTER summary: min / max block per (element, site)
      if (!own)
        return; // block-private buffer: no INTER pair possible
      const uint64_t i = e * static_cast<uint64_t>(L->nSitesTab) + site;
      const uint32_t b = static_cast<uint32_t>(block) + 1;
      if (L->interLo[i] > b)
        atomicMin(&L->interLo[i], b);
      if (L->interHi[i] < b)
        atomicMax(&L->interHi[i], b);
      return;
    }
    if (L->ownerFilter && !ownerIsMulti(L->ownerFilter, e, L->ownerMultiTag))
      return; // fused pass 2: only elements shared by blocks
    if (L->interTab) { // INTER summary: EMPTY -> one block -> MULTI, no record
      interUpdate(&L->interTab[e * static_cast<uint64_t>(L->nSitesTab) + site],
                  static_cast<uint32_t>(block));
      return;
    }
    if (L->nTargets) { // witness pass: only the keys' first-found elements
      bool hit = false;
      for (int i = 0; i < L->nTargets; ++i)
        hit |= L->targets[i] == e;
      if (!hit)
        return;
    }
    const KeyLayout &kl = L->kl;
    const uint64_t maskP = fieldMask(kl.bP), maskQ = fieldMask(kl.bQ);
    if (bp > maskP || wp > maskQ)
      flags |= kFlagPhase;
    if (seq > seqMask(kl))
      flags |= kFlagSeqSite;
    const uint64_t key = packKey(kl, e, static_cast<uint64_t>(block), bp & maskP,
                                 static_cast<uint64_t>(warp), wp & maskQ,
                                 static_cast<uint64_t>(lane));
    const uint32_t val = (static_cast<uint32_t>(site) << kl.bS) | (seq & seqMask(kl));
    if (out->n < kLaneBuf) {
      out->k[out->n] = key;
      out->v[out->n] = val;
      ++out->n;
    } else { // long per-thread access streams spill one by one
      const unsigned long long pos = atomicAdd(&L->ctr->cursor, 1ull);
      if (pos < L->capacity) {
        L->keys[pos] = key;
        L->vals[pos] = val;
      } else {
        flags |= kFlagCapacity;
      }
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
  // S variant: a streamed load (affine.hpp streamSites; staged in shared
  // memory by k_fused only — here a plain value-needed load)
  template <class I>
  __device__ __forceinline__ int64_t loadS(int site, int param, bool rec, bool own, I idx,
                                           int64_t size, uint64_t base) {
    return loadC(site, param, rec, own, idx, true, size, base);
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
    if (L->opStride && !outOfRange(idx, size))
      atomicOp(site, param, static_cast<int64_t>(idx));
  }
  // K variants: the site's parameter and record flag as (JIT) constants
  __device__ __forceinline__ int64_t loadK(int site, int param, bool rec, bool, int64_t idx,
                                           bool need) {
    const ParamDev *P = checkK(param, idx);
    if (!P)
      return 0;
    if (rec)
      record(site, P, idx);
    ++seq;
    return need ? __ldg(P->ptr + idx) : 0;
  }
  __device__ __forceinline__ void storeK(int site, int param, bool rec, bool, int64_t idx,
                                         int64_t) {
    const ParamDev *P = checkK(param, idx);
    if (!P)
      return;
    if (rec)
      record(site, P, idx);
    ++seq;
  }
  __device__ __forceinline__ void atomicK(int site, int param, bool rec, bool own, int64_t idx,
                                          int64_t, int64_t) {
    const unsigned long long before = inst;
    storeK(site, param, rec, own, idx, 0);
    if (L->opStride && inst != before) // in bounds
      atomicOp(site, param, idx);
  }
  __device__ __forceinline__ int64_t load(int site, int64_t idx, bool need) {
    return loadK(site, sites[site].param, sites[site].record, false, idx, need);
  }
  __device__ __forceinline__ void store(int site, int64_t idx, int64_t v) {
    storeK(site, sites[site].param, sites[site].record, false, idx, v);
  }
  __device__ __forceinline__ void atomic(int site, int64_t idx, int64_t v, int64_t c) {
    atomicK(site, sites[site].param, sites[site].record, false, idx, v, c);
  }
};

template <class Body> __global__ void __launch_bounds__(256) k_expand_par(LaunchDev L) {
  extern __shared__ __align__(16) unsigned char smem[];
  hgrd_gpu_insn *sCode = reinterpret_cast<hgrd_gpu_insn *>(smem);
  SiteDev *sSites = reinterpret_cast<SiteDev *>(sCode + L.nCode);
  ParamDev *sParams = reinterpret_cast<ParamDev *>(sSites + L.nSites);
  for (int i = threadIdx.x; i < L.nCode; i += blockDim.x)
    sCode[i] = L.code[i];
  for (int i = threadIdx.x; i < L.nSites; i += blockDim.x)
    sSites[i] = L.sites[i];
  for (int i = threadIdx.x; i < L.nParams; i += blockDim.x)
    sParams[i] = L.params[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int64_t warpId = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nWarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned long long chunkBase = 0, chunkLeft = 0; // warp-uniform
  LaneTally tally;
  LaneRecords out;
  int64_t regs[kMaxRegs];
  for (int64_t batch = warpId; L.threadBase + batch * 32 < L.threadEnd; batch += nWarps) {
    const int64_t t = L.threadBase + batch * 32 + lane;
    out.n = 0;
    if (t < L.threadEnd) {
      ParSink s;
      s.L = &L;
      s.sites = sSites;
      s.params = sParams;
      s.out = &out;
      s.t = t;
      Builtins bi;
      Body::identity(L, t, bi, s.block, s.warp, s.lane);
      Body::run(L, sCode, bi, s, regs);
      for (uint32_t j = s.nOps; j < L.opStride; ++j) // unused op slots
        L.opMeta[static_cast<uint64_t>(t) * L.opStride + j] = 15;
      tally.add(s);
    }
    __syncwarp();
    // warp-level placement of the batch's records
    int incl = out.n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o)
        incl += y;
    }
    const unsigned total = static_cast<unsigned>(__shfl_sync(0xffffffffu, incl, 31));
    if (total == 0)
      continue;
    const unsigned long long base0 = chunkBase, left0 = chunkLeft;
    unsigned long long fresh = 0;
    if (total > left0) {
      const unsigned long long need = total - left0;
      const unsigned long long size = need > L.chunk ? need : L.chunk;
      if (lane == 0)
        fresh = atomicAdd(&L.ctr->cursor, size);
      fresh = __shfl_sync(0xffffffffu, fresh, 0);
      chunkBase = fresh + need;
      chunkLeft = size - need;
    } else {
      chunkBase += total;
      chunkLeft -= total;
    }
    const unsigned excl = static_cast<unsigned>(incl - out.n);
    for (int j = 0; j < out.n; ++j) {
      const unsigned long long w = excl + j;
      const unsigned long long dst = w < left0 ? base0 + w : fresh + (w - left0);
      if (dst < L.capacity) {
        L.keys[dst] = out.k[j];
        L.vals[dst] = out.v[j];
      } else {
        tally.flags |= kFlagCapacity;
      }
    }
  }
  // pad the warp's open chunk with sentinels (they sort last)
  for (unsigned long long j = lane; j < chunkLeft; j += 32) {
    const unsigned long long dst = chunkBase + j;
    if (dst < L.capacity)
      L.keys[dst] = L.kl.sentinel;
  }
  // one atomic per warp per counter
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tally.steps += __shfl_down_sync(0xffffffffu, tally.steps, o);
    tally.inst += __shfl_down_sync(0xffffffffu, tally.inst, o);
    tally.traps += __shfl_down_sync(0xffffffffu, tally.traps, o);
    tally.recs += __shfl_down_sync(0xffffffffu, tally.recs, o);
    tally.maxBp = max(tally.maxBp, __shfl_down_sync(0xffffffffu, tally.maxBp, o));
    tally.maxWp = max(tally.maxWp, __shfl_down_sync(0xffffffffu, tally.maxWp, o));
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
    atomicMax(&L.ctr->maxBp, tally.maxBp);
    atomicMax(&L.ctr->maxWp, tally.maxWp);
    if (tally.flags)
      atomicOr(&L.ctr->flags, tally.flags);
  }
}

// ---------------------------------------------------------------------------
// SEQUENTIAL: canonical order, memory effects, ordered traps, exact budget.
struct SeqSink {
  const LaunchDev *L;
  int64_t t = 0, block = 0, warp = 0, lane = 0;
  uint32_t bp = 0, wp = 0, seq = 0;
  unsigned long long cursor = 0, steps = 0, inst = 0, traps = 0, nOps = 0;
  unsigned maxBp = 0, maxWp = 0, flags = 0;
  int abortStmt = -1;
  bool aborted = false;

  __device__ bool step(int stmt) {
    if (static_cast<int64_t>(++steps) > L->stepBudget) {
      abortStmt = stmt;
      flags |= kFlagAbort;
      aborted = true;
      return false;
    }
    return true;
  }
  __device__ const ParamDev *check(int site, int64_t idx) {
    const SiteDev &S = L->sites[site];
    const ParamDev *P = S.param >= 0 ? &L->params[S.param] : nullptr;
    const bool unalloc = !P || P->handle < 0;
    if (unalloc || idx < 0 || idx >= P->size) {
      if (traps < L->trapCap)
        L->traps[traps] = hgrd_gpu_trap{site, unalloc ? HGRD_TRAP_UNALLOCATED : HGRD_TRAP_OOB, t};
      ++traps;
      return nullptr;
    }
    ++inst;
    if (S.record) {
      const KeyLayout &kl = L->kl;
      const uint64_t maskP = fieldMask(kl.bP), maskQ = fieldMask(kl.bQ);
      if (bp > maskP || wp > maskQ)
        flags |= kFlagPhase;
      if (seq > seqMask(kl))
        flags |= kFlagSeqSite;
      if (cursor < L->capacity) {
        L->keys[cursor] = packKey(kl, P->elemBase + static_cast<uint64_t>(idx),
                                  static_cast<uint64_t>(block), bp & maskP,
                                  static_cast<uint64_t>(warp), wp & maskQ,
                                  static_cast<uint64_t>(lane));
        L->vals[cursor] = (static_cast<uint32_t>(site) << kl.bS) | (seq & seqMask(kl));
      } else {
        flags |= kFlagCapacity;
      }
      ++cursor;
    }
    ++seq;
    return P;
  }
  __device__ void op(int kind, int scope, int handle, int64_t idx, uint32_t s) {
    if (nOps < L->opCap) {
      L->opMeta[nOps] = kind | (scope << 4) | ((handle + 1) << 8);
      L->opIndex[nOps] = idx;
      L->opSeq[nOps] = static_cast<int32_t>(s);
    } else if (L->opStart) {
      flags |= kFlagOps;
    }
    ++nOps;
  }
  __device__ int64_t load(int site, int64_t idx, bool) {
    const ParamDev *P = check(site, idx);
    return P ? P->ptr[idx] : 0;
  }
  __device__ void store(int site, int64_t idx, int64_t v) {
    const ParamDev *P = check(site, idx);
    if (P)
      P->ptr[idx] = v;
  }
  __device__ void atomic(int site, int64_t idx, int64_t v, int64_t cmp) {
    const ParamDev *P = check(site, idx);
    if (!P)
      return;
    const SiteDev &S = L->sites[site];
    int64_t *cell = P->ptr + idx;
    const int64_t old = *cell;
    if (S.aop == HGRD_ATOMIC_ADD) {
      *cell = wrapAdd(old, v);
    } else {
      if (S.aop == HGRD_ATOMIC_EXCH || old == cmp)
        *cell = v;
      op(S.aop == HGRD_ATOMIC_CAS ? 0 : 1, S.scope, P->handle, idx, seq - 1);
    }
  }
  __device__ void syncthreads() {
    ++bp;
    ++wp;
  }
  __device__ void syncwarp() { ++wp; }
  __device__ void fence(int scope) {
    op(2, scope, -1, 0, seq);
    ++seq;
  }
  // NVRTC bodies (jit.cpp): the site's parameter, record flag, buffer size
  // and element base are constants, so in-range accesses skip the site and
  // parameter lookups; out-of-range ones take the generic path, which
  // classifies and orders the trap (a folded size of 0 covers unallocated)
  __device__ __forceinline__ void stepNC() { ++steps; }
  __device__ __forceinline__ int64_t *fastAccess(int site, int param, bool rec, int64_t idx,
                                                 uint64_t base) {
    ++inst;
    if (rec) {
      const KeyLayout &kl = L->kl;
      const uint64_t maskP = fieldMask(kl.bP), maskQ = fieldMask(kl.bQ);
      if (bp > maskP || wp > maskQ)
        flags |= kFlagPhase;
      if (seq > seqMask(kl))
        flags |= kFlagSeqSite;
      if (cursor < L->capacity) {
        L->keys[cursor] = packKey(kl, base + static_cast<uint64_t>(idx),
                                  static_cast<uint64_t>(block), bp & maskP,
                                  static_cast<uint64_t>(warp), wp & maskQ,
                                  static_cast<uint64_t>(lane));
        L->vals[cursor] = (static_cast<uint32_t>(site) << kl.bS) | (seq & seqMask(kl));
      } else {
        flags |= kFlagCapacity;
      }
      ++cursor;
    }
    ++seq;
    return L->params[param].ptr + idx;
  }
  template <class I>
  __device__ __forceinline__ int64_t loadC(int site, int param, bool rec, bool, I idx, bool need,
                                           int64_t size, uint64_t base) {
    if (outOfRange(idx, size))
      return load(site, static_cast<int64_t>(idx), need);
    return *fastAccess(site, param, rec, static_cast<int64_t>(idx), base);
  }
  template <class I>
  __device__ __forceinline__ int64_t loadS(int site, int param, bool rec, bool own, I idx,
                                           int64_t size, uint64_t base) {
    return loadC(site, param, rec, own, idx, true, size, base);
  }
  template <class I>
  __device__ __forceinline__ void storeC(int site, int param, bool rec, bool, I idx, int64_t v,
                                         int64_t size, uint64_t base) {
    if (outOfRange(idx, size))
      store(site, static_cast<int64_t>(idx), v);
    else
      *fastAccess(site, param, rec, static_cast<int64_t>(idx), base) = v;
  }
  template <class I>
  __device__ __forceinline__ void atomicC(int site, int, bool, bool, I idx, int64_t v,
                                          int64_t cmp, int64_t, uint64_t) {
    atomic(site, static_cast<int64_t>(idx), v, cmp);
  }
};

// The canonical order is one serial chain, so its cost is latency: with
// `staged` the register file lives in shared memory (nRegs * 8 bytes of
// dynamic smem) instead of global scratch, where every register
// read-after-write was an L2 round trip.  (The bytecode and initial values
// stay global: the compiler addresses pointers reached from the launch
// parameters as global, and they are read-only L1 hits anyway.)
template <class Body> __global__ void k_expand_seq(LaunchDev L, int staged) {
  extern __shared__ int64_t seqSh[];
  int64_t *regs = staged ? seqSh : L.seqRegs;
  if (blockIdx.x != 0 || threadIdx.x != 0)
    return;
  SeqSink s;
  s.L = &L;
  for (int64_t t = 0; t < L.nThreads && !s.aborted; ++t) {
    Builtins bi;
    Body::identity(L, t, bi, s.block, s.warp, s.lane);
    s.t = t;
    s.bp = s.wp = s.seq = 0;
    if (L.opStart)
      L.opStart[t] = s.nOps;
    Body::run(L, L.code, bi, s, regs);
    s.maxBp = max(s.maxBp, s.bp);
    s.maxWp = max(s.maxWp, s.wp);
  }
  if (L.opStart && !s.aborted)
    L.opStart[L.nThreads] = s.nOps;
  L.ctr->steps = s.steps;
  L.ctr->instances = s.inst;
  L.ctr->records = s.cursor;
  L.ctr->cursor = s.cursor;
  L.ctr->traps = s.traps;
  L.ctr->nOps = s.nOps;
  L.ctr->maxBp = s.maxBp;
  L.ctr->maxWp = s.maxWp;
  L.ctr->flags = s.flags;
  L.ctr->abortStmt = s.abortStmt;
}

} // namespace dev
} // namespace hgrdgpu

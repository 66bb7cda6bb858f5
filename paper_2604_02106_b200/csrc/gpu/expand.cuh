// K1: access-instance expansion.
//
// k_expand_par — one lane per MiniCU thread, a warp per 32 consecutive
// threads (block-major, so warps of the same MiniCU block stay together),
// grid-stride over the thread space.  Each lane interprets the lowered
// kernel (registers in local memory, code/sites/params staged in shared
// memory) and buffers its packed records; at the batch boundary the warp
// scans the per-lane counts and writes them into a per-warp chunk of the
// record arrays reserved with ONE global atomic per kChunk records.
// Loads read memory only when their value is needed (value-relevant sites
// of a PARALLEL launch read never-written buffers, i.e. the exact
// launch-entry snapshot); stores are not materialised.
//
// k_expand_seq — the reference's canonical order (src/oracle.cpp:440-465)
// with full memory effects, traps in order and the exact step budget; used
// for launches whose loaded values steer addresses or control.
#pragma once

#include "device.cuh"

namespace hgrdgpu {
namespace dev {

struct Builtins {
  int64_t v[12];
};

__device__ __forceinline__ void threadIdentity(const LaunchDev &L, int64_t t,
                                               Builtins &b, int64_t &block,
                                               int64_t &warp, int64_t &lane) {
  block = t / L.tpb;
  const int64_t tl = t - block * L.tpb;
  b.v[0] = tl % L.block[0];
  b.v[1] = (tl / L.block[0]) % L.block[1];
  b.v[2] = tl / (L.block[0] * L.block[1]);
  b.v[3] = block % L.grid[0];
  b.v[4] = (block / L.grid[0]) % L.grid[1];
  b.v[5] = block / (L.grid[0] * L.grid[1]);
  b.v[6] = L.block[0];
  b.v[7] = L.block[1];
  b.v[8] = L.block[2];
  b.v[9] = L.grid[0];
  b.v[10] = L.grid[1];
  b.v[11] = L.grid[2];
  warp = tl / L.ws;
  lane = tl - warp * L.ws;
}

struct LaneRecords {
  uint64_t k[kLaneBuf];
  uint32_t v[kLaneBuf];
  int n;
};

struct LaneTally {
  unsigned long long steps = 0, inst = 0, traps = 0, recs = 0;
  unsigned int maxBp = 0, maxWp = 0, flags = 0;
};

// Interpret one MiniCU thread in PARALLEL mode.
__device__ __forceinline__ void runParallel(const LaunchDev &L,
                                            const hgrd_gpu_insn *__restrict__ code,
                                            const SiteDev *__restrict__ sites,
                                            const ParamDev *__restrict__ params,
                                            int64_t t, LaneRecords &out,
                                            LaneTally &tally) {
  int64_t r[kMaxRegs];
  for (int i = 0; i < L.nRegs; ++i)
    r[i] = L.regInit[i];
  Builtins bi;
  int64_t block, warp, lane;
  threadIdentity(L, t, bi, block, warp, lane);
  uint32_t bp = 0, wp = 0, seq = 0;
  int64_t steps = 0;
  const KeyLayout &kl = L.kl;
  const uint64_t maskP = fieldMask(kl.bP), maskQ = fieldMask(kl.bQ);
  int pc = 0;
  for (;;) {
    const hgrd_gpu_insn I = code[pc];
    switch (I.op) {
    case HGRD_OP_END:
      goto done;
    case HGRD_OP_STEP:
      if (++steps > L.stepBudget) {
        tally.flags |= kFlagAbort;
        goto done;
      }
      break;
    case HGRD_OP_CONST:
      r[I.a] = I.imm;
      break;
    case HGRD_OP_MOV:
      r[I.a] = r[I.b];
      break;
    case HGRD_OP_BUILTIN:
      r[I.a] = bi.v[I.sub];
      break;
    case HGRD_OP_BIN:
      r[I.a] = applyBin(I.sub, r[I.b], r[I.c]);
      break;
    case HGRD_OP_LOAD:
    case HGRD_OP_STORE:
    case HGRD_OP_ATOMIC: {
      const int site = static_cast<int>(I.imm);
      const SiteDev S = sites[site];
      const int64_t idx = I.op == HGRD_OP_LOAD ? r[I.b] : r[I.a];
      const ParamDev *P = S.param >= 0 ? &params[S.param] : nullptr;
      if (!P || P->handle < 0 || idx < 0 || idx >= P->size) {
        ++tally.traps; // any trap sends the launch to the ordered path
        if (I.op == HGRD_OP_LOAD)
          r[I.a] = 0;
        break;
      }
      ++tally.inst;
      if (S.record && (!L.ownerFilter ||
                       L.ownerFilter[P->elemBase + static_cast<uint64_t>(idx)] == L.ownerMultiTag)) {
        if (bp > maskP || wp > maskQ)
          tally.flags |= kFlagPhase;
        if (seq > kSeqMask)
          tally.flags |= kFlagSeqSite;
        const uint64_t key =
            packKey(kl, P->elemBase + static_cast<uint64_t>(idx),
                    static_cast<uint64_t>(block), bp & maskP,
                    static_cast<uint64_t>(warp), wp & maskQ,
                    static_cast<uint64_t>(lane));
        const uint32_t val = (static_cast<uint32_t>(site) << kSeqBits) | (seq & kSeqMask);
        if (out.n < kLaneBuf) {
          out.k[out.n] = key;
          out.v[out.n] = val;
          ++out.n;
        } else { // long per-thread access streams spill one by one
          unsigned long long pos = atomicAdd(&L.ctr->cursor, 1ull);
          if (pos < L.capacity) {
            L.keys[pos] = key;
            L.vals[pos] = val;
          } else {
            tally.flags |= kFlagCapacity;
          }
        }
        ++tally.recs;
      }
      ++seq;
      if (I.op == HGRD_OP_LOAD)
        r[I.a] = (I.sub & 1) ? __ldg(P->ptr + idx) : 0;
      break;
    }
    case HGRD_OP_SYNCTHREADS:
      ++bp;
      ++wp;
      break;
    case HGRD_OP_SYNCWARP:
      ++wp;
      break;
    case HGRD_OP_FENCE:
      ++seq; // a fence takes a sequence number (reference :616-618)
      break;
    case HGRD_OP_JZ:
      if (r[I.a] == 0) {
        pc = static_cast<int>(I.imm);
        continue;
      }
      break;
    case HGRD_OP_JMP:
      pc = static_cast<int>(I.imm);
      continue;
    default:
      goto done;
    }
    ++pc;
  }
done:
  tally.steps += static_cast<unsigned long long>(steps);
  tally.maxBp = max(tally.maxBp, bp);
  tally.maxWp = max(tally.maxWp, wp);
}

__global__ void __launch_bounds__(256) k_expand_par(LaunchDev L) {
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
  for (int64_t batch = warpId; batch * 32 < L.nThreads; batch += nWarps) {
    const int64_t t = batch * 32 + lane;
    out.n = 0;
    if (t < L.nThreads)
      runParallel(L, sCode, sSites, sParams, t, out, tally);
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
__global__ void k_expand_seq(LaunchDev L) {
  if (blockIdx.x != 0 || threadIdx.x != 0)
    return;
  int64_t *r = L.seqRegs;
  const KeyLayout &kl = L.kl;
  const uint64_t maskP = fieldMask(kl.bP), maskQ = fieldMask(kl.bQ);
  unsigned long long cursor = 0, steps = 0, inst = 0, traps = 0, nOps = 0;
  unsigned int maxBp = 0, maxWp = 0, flags = 0;
  int abortStmt = -1;
  for (int64_t t = 0; t < L.nThreads; ++t) {
    for (int i = 0; i < L.nRegs; ++i)
      r[i] = L.regInit[i];
    Builtins bi;
    int64_t block, warp, lane;
    threadIdentity(L, t, bi, block, warp, lane);
    uint32_t bp = 0, wp = 0, seq = 0;
    if (L.opStart)
      L.opStart[t] = nOps;
    int pc = 0;
    for (;;) {
      const hgrd_gpu_insn I = L.code[pc];
      if (I.op == HGRD_OP_END)
        break;
      switch (I.op) {
      case HGRD_OP_STEP:
        if (static_cast<int64_t>(++steps) > L.stepBudget) {
          abortStmt = static_cast<int>(I.imm);
          flags |= kFlagAbort;
          goto finish;
        }
        break;
      case HGRD_OP_CONST:
        r[I.a] = I.imm;
        break;
      case HGRD_OP_MOV:
        r[I.a] = r[I.b];
        break;
      case HGRD_OP_BUILTIN:
        r[I.a] = bi.v[I.sub];
        break;
      case HGRD_OP_BIN:
        r[I.a] = applyBin(I.sub, r[I.b], r[I.c]);
        break;
      case HGRD_OP_LOAD:
      case HGRD_OP_STORE:
      case HGRD_OP_ATOMIC: {
        const int site = static_cast<int>(I.imm);
        const SiteDev S = L.sites[site];
        const int64_t idx = I.op == HGRD_OP_LOAD ? r[I.b] : r[I.a];
        const ParamDev *P = S.param >= 0 ? &L.params[S.param] : nullptr;
        const bool unalloc = !P || P->handle < 0;
        if (unalloc || idx < 0 || idx >= P->size) {
          if (traps < L.trapCap)
            L.traps[traps] = hgrd_gpu_trap{site, unalloc ? HGRD_TRAP_UNALLOCATED : HGRD_TRAP_OOB, t};
          ++traps;
          if (I.op == HGRD_OP_LOAD)
            r[I.a] = 0;
          break;
        }
        ++inst;
        if (S.record) {
          if (bp > maskP || wp > maskQ)
            flags |= kFlagPhase;
          if (seq > kSeqMask)
            flags |= kFlagSeqSite;
          if (cursor < L.capacity) {
            L.keys[cursor] = packKey(kl, P->elemBase + static_cast<uint64_t>(idx),
                                     static_cast<uint64_t>(block), bp & maskP,
                                     static_cast<uint64_t>(warp), wp & maskQ,
                                     static_cast<uint64_t>(lane));
            L.vals[cursor] = (static_cast<uint32_t>(site) << kSeqBits) | (seq & kSeqMask);
          } else {
            flags |= kFlagCapacity;
          }
          ++cursor;
        }
        ++seq;
        int64_t *cell = P->ptr + idx;
        if (I.op == HGRD_OP_LOAD) {
          r[I.a] = *cell;
        } else if (I.op == HGRD_OP_STORE) {
          *cell = r[I.b];
        } else {
          const int64_t old = *cell;
          if (S.aop == HGRD_ATOMIC_ADD) {
            *cell = wrapAdd(old, r[I.b]);
          } else {
            if (S.aop == HGRD_ATOMIC_EXCH || old == r[I.c])
              *cell = r[I.b];
            if (nOps < L.opCap) {
              L.opMeta[nOps] = (S.aop == HGRD_ATOMIC_CAS ? 0 : 1) | (S.scope << 4) |
                               ((P->handle + 1) << 8);
              L.opIndex[nOps] = idx;
              L.opSeq[nOps] = static_cast<int32_t>(seq - 1);
            } else if (L.opStart) {
              flags |= kFlagOps;
            }
            ++nOps;
          }
        }
        break;
      }
      case HGRD_OP_SYNCTHREADS:
        ++bp;
        ++wp;
        break;
      case HGRD_OP_SYNCWARP:
        ++wp;
        break;
      case HGRD_OP_FENCE:
        if (nOps < L.opCap) {
          L.opMeta[nOps] = 2 | (I.sub << 4);
          L.opIndex[nOps] = 0;
          L.opSeq[nOps] = static_cast<int32_t>(seq);
        } else if (L.opStart) {
          flags |= kFlagOps;
        }
        ++nOps;
        ++seq;
        break;
      case HGRD_OP_JZ:
        if (r[I.a] == 0) {
          pc = static_cast<int>(I.imm);
          continue;
        }
        break;
      case HGRD_OP_JMP:
        pc = static_cast<int>(I.imm);
        continue;
      default:
        break;
      }
      ++pc;
    }
    maxBp = max(maxBp, bp);
    maxWp = max(maxWp, wp);
  }
  if (L.opStart)
    L.opStart[L.nThreads] = nOps;
finish:
  L.ctr->steps = steps;
  L.ctr->instances = inst;
  L.ctr->records = cursor;
  L.ctr->cursor = cursor;
  L.ctr->traps = traps;
  L.ctr->nOps = nOps;
  L.ctr->maxBp = maxBp;
  L.ctr->maxWp = maxWp;
  L.ctr->flags = flags;
  L.ctr->abortStmt = abortStmt;
}

} // namespace dev
} // namespace hgrdgpu

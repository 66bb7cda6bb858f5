// Thread bodies: how one MiniCU thread's statements execute.
//
// A body runs the lowered kernel for one thread and reports every effect to
// a Sink (the kernel-specific access semantics):
//   bool    step(int stmt)                    one step charged (false: stop)
//   int64_t load(int site, int64_t idx, bool valueNeeded)
//   void    store(int site, int64_t idx, int64_t value)
//   void    atomic(int site, int64_t idx, int64_t value, int64_t compare)
//   void    syncthreads(); syncwarp(); fence(int scope);
//
// InterpBody interprets hgrd_gpu bytecode (any kernel, no compilation).
// JIT bodies are the same bytecode translated to straight-line CUDA C++ by
// csrc/gpu/jit.cpp and compiled with NVRTC for sm_100a: registers become
// locals, jumps become gotos, launch constants fold.
#pragma once

#include "device.cuh"

namespace hgrdgpu {
namespace dev {

struct Builtins {
  int64_t v[12];
};

__device__ __forceinline__ void threadIdentity(const LaunchDev &L, int64_t t, Builtins &b,
                                               int64_t &block, int64_t &warp, int64_t &lane) {
  b.v[6] = L.block[0];
  b.v[7] = L.block[1];
  b.v[8] = L.block[2];
  b.v[9] = L.grid[0];
  b.v[10] = L.grid[1];
  b.v[11] = L.grid[2];
  if (L.small) { // reference :443-460 with magic-number division
    const uint32_t u = static_cast<uint32_t>(t);
    const uint32_t bl = L.dTpb.div(u);
    const uint32_t tl = u - bl * L.dTpb.d;
    const uint32_t q1 = L.dBx.d == 1 ? tl : L.dBx.div(tl);
    const uint32_t tz = L.dBxBy.div(tl);
    b.v[0] = tl - q1 * L.dBx.d;
    b.v[1] = q1 - tz * static_cast<uint32_t>(L.block[1]);
    b.v[2] = tz;
    const uint32_t g1 = L.dGx.div(bl);
    const uint32_t bz = L.dGxGy.div(bl);
    b.v[3] = bl - g1 * L.dGx.d;
    b.v[4] = g1 - bz * static_cast<uint32_t>(L.grid[1]);
    b.v[5] = bz;
    const uint32_t w = L.dWs.div(tl);
    block = bl;
    warp = w;
    lane = tl - w * L.dWs.d;
    return;
  }
  block = t / L.tpb;
  const int64_t tl = t - block * L.tpb;
  b.v[0] = tl % L.block[0];
  b.v[1] = (tl / L.block[0]) % L.block[1];
  b.v[2] = tl / (L.block[0] * L.block[1]);
  b.v[3] = block % L.grid[0];
  b.v[4] = (block / L.grid[0]) % L.grid[1];
  b.v[5] = block / (L.grid[0] * L.grid[1]);
  warp = tl / L.ws;
  lane = tl - warp * L.ws;
}

// Bounds check and element of a JIT access (C variants of the sinks); the
// 32-bit forms are emitted only when the buffer size is below 2^31.
__device__ __forceinline__ bool outOfRange(int64_t idx, int64_t size) {
  return static_cast<uint64_t>(idx) >= static_cast<uint64_t>(size);
}
__device__ __forceinline__ bool outOfRange(int32_t idx, int64_t size) {
  return static_cast<uint32_t>(idx) >= static_cast<uint32_t>(size);
}
__device__ __forceinline__ uint64_t elementAt(uint64_t base, int64_t idx) {
  return base + static_cast<uint64_t>(idx);
}
__device__ __forceinline__ uint64_t elementAt(uint64_t base, int32_t idx) {
  return base + static_cast<uint32_t>(idx);
}

struct InterpBody {
  static constexpr int kFixedR = -1; // records per thread not known at compile time
  static constexpr bool kPair = false; // (no run2: one MiniCU thread per call)
  __device__ static __forceinline__ void identity(const LaunchDev &L, int64_t t, Builtins &b,
                                                  int64_t &block, int64_t &warp, int64_t &lane) {
    threadIdentity(L, t, b, block, warp, lane);
  }
  // `r` holds nRegs registers (local array or global scratch).
  template <class Sink>
  __device__ static void run(const LaunchDev &L, const hgrd_gpu_insn *__restrict__ code,
                             const Builtins &bi, Sink &s, int64_t *r) {
    for (int i = 0; i < L.nRegs; ++i)
      r[i] = L.regInit[i];
    int pc = 0;
    for (;;) {
      const hgrd_gpu_insn I = code[pc];
      switch (I.op) {
      case HGRD_OP_END:
        return;
      case HGRD_OP_STEP:
        if (!s.step(static_cast<int>(I.imm)))
          return;
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
        r[I.a] = s.load(static_cast<int>(I.imm), r[I.b], (I.sub & 1) != 0);
        break;
      case HGRD_OP_STORE:
        s.store(static_cast<int>(I.imm), r[I.a], r[I.b]);
        break;
      case HGRD_OP_ATOMIC:
        s.atomic(static_cast<int>(I.imm), r[I.a], r[I.b], r[I.c]);
        break;
      case HGRD_OP_SYNCTHREADS:
        s.syncthreads();
        break;
      case HGRD_OP_SYNCWARP:
        s.syncwarp();
        break;
      case HGRD_OP_FENCE:
        s.fence(I.sub);
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
        return;
      }
      ++pc;
    }
  }
};

// Shared bookkeeping of the PARALLEL sinks: identity, phases, sequence
// numbers, step budget, bounds checks (reference checkBounds :508-519).
struct ParState {
  const LaunchDev *L;
  const SiteDev *sites;
  const ParamDev *params;
  int64_t block, warp, lane;
  uint32_t bp = 0, wp = 0, seq = 0;
  int64_t steps = 0;
  unsigned long long inst = 0, traps = 0, recs = 0;
  unsigned flags = 0;

  __device__ __forceinline__ bool step(int) {
    if (++steps > L->stepBudget) {
      flags |= kFlagAbort;
      return false;
    }
    return true;
  }
  // JIT bodies of loop-free kernels whose statement count fits the budget
  __device__ __forceinline__ void stepNC() { ++steps; }
  // Returns the parameter when the access is in bounds (an instance).
  __device__ __forceinline__ const ParamDev *check(int site, int64_t idx) {
    return checkK(sites[site].param, idx);
  }
  // Same with the site's parameter known (JIT bodies pass it as a constant).
  __device__ __forceinline__ const ParamDev *checkK(int param, int64_t idx) {
    const ParamDev *P = param >= 0 ? &params[param] : nullptr;
    if (!P || P->handle < 0 || idx < 0 || idx >= P->size) {
      ++traps; // any trap sends the launch to the ordered path
      return nullptr;
    }
    ++inst;
    return P;
  }
  __device__ __forceinline__ void syncthreads() {
    ++bp;
    ++wp;
  }
  __device__ __forceinline__ void syncwarp() { ++wp; }
  __device__ __forceinline__ void fence(int) { ++seq; } // fences take a seq (:616-618)
};

} // namespace dev
} // namespace hgrdgpu

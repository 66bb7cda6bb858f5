// hgrd_gpu_ctx: device-resident buffers + the per-launch race-check
// pipeline (include/hgrd_gpu.h).
//
//   blob H2D -> K1 expand (PARALLEL | SEQUENTIAL) -> counters D2H
//     -> radix sort of packed records (CUB onesweep, bits = key width)
//     -> K3 segment detector (summary | pairwise) -> K4 witness/decode
//     -> races D2H
#include "detect.cuh"
#include "device.cuh"
#include "expand.cuh"
#include "fused.cuh"
#include "batch.cuh"
#include "affine.hpp"
#include "jit.hpp"
#include "parallel_for.hpp"

#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <set>
#include <numeric>
#include <string>
#include <vector>
#include <thread>
#include <atomic>
#include <unordered_map>

using namespace hgrdgpu::dev;

// element ids + identity permutation for the stable element sort
__global__ void k_elem_keys(const uint64_t *keys, uint64_t n, int shE, uint64_t *elem,
                            uint32_t *order) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    elem[i] = shE >= 64 ? 0 : keys[i] >> shE;
    order[i] = static_cast<uint32_t>(i);
  }
}

// the same with the canonical event order below the element: element |
// thread | seq (sentinel padding records keep an all-ones element)
__global__ void k_elem_keys_canon(const uint64_t *keys, const uint32_t *vals, uint64_t n,
                                  KeyLayout kl, int64_t tpb, int64_t ws, int bT, int bS,
                                  uint64_t *elem, uint32_t *order) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  order[i] = static_cast<uint32_t>(i);
  const uint64_t k = keys[i];
  if (k == kl.sentinel) { // chunk padding: the all-ones element, sorts last
    elem[i] = (fieldMask(kl.bE) << (bT + bS)) | fieldMask(bT + bS);
    return;
  }
  const uint64_t e = kl.shE >= 64 ? 0 : k >> kl.shE;
  const uint64_t block = (k >> kl.shB) & fieldMask(kl.bB);
  const uint64_t warp = (k >> kl.shW) & fieldMask(kl.bW);
  const uint64_t lane = k & fieldMask(kl.bL);
  const uint64_t thread =
      block * static_cast<uint64_t>(tpb) + warp * static_cast<uint64_t>(ws) + lane;
  elem[i] = (e << (bT + bS)) | (thread << bS) | (vals[i] & seqMask(kl));
}

__global__ void k_shift_keys(uint64_t *x, uint64_t n, int sh) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n)
    x[i] >>= sh;
}

namespace {

template <class T> struct DevVec {
  T *p = nullptr;
  size_t cap = 0;
};

struct BigBlock {
  void *p;
  size_t bytes;
};

int bitsFor(uint64_t n) { // bits to hold values 0 .. n-1
  if (n <= 1)
    return 0;
  return 64 - __builtin_clzll(n - 1);
}

} // namespace

// k_expand_seq's shared-memory register file limit (larger register files
// stay in global scratch)
constexpr size_t kSeqSharedMax = 200 * 1024;

struct hgrd_gpu_ctx {
  bool seqSharedSet = false;           // k_expand_seq opted into > 48 KB
  std::vector<hgrd_gpu_ctx *> workers; // sweep workers: own streams and buffers (same device)
  int device = 0;
  int nSM = 148;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // asynchronous uploads: copy stream, one event per upload in flight
  cudaStream_t up = nullptr;
  std::vector<cudaEvent_t> upEvents;
  std::vector<int> upFree;
  std::string err;

  struct Buf {
    int64_t *p;
    int64_t elems;
    bool zeroPending; // allocated, zero-initialisation not yet materialised
    int upload = -1;  // hgrd_gpu_buffer_write_async in flight: its upEvents slot
  };
  std::vector<Buf> bufs;
  // small allocations: bump arena over 256 MiB chunks; large: size-keyed cache
  std::vector<char *> chunks;
  size_t chunkBytes = size_t(256) << 20;
  size_t chunkIdx = 0, chunkUsed = 0;
  std::multimap<size_t, void *> bigFree;
  std::vector<BigBlock> bigUsed;

  DevVec<uint64_t> keys, keysAlt, elemK, elemKAlt;
  DevVec<uint32_t> vals, valsAlt, order, orderAlt;
  DevVec<unsigned char> cubTemp, blob, snapshot;
  DevVec<uint32_t> keySeg;
  DevVec<unsigned long long> keyPair;
  DevVec<hgrd_gpu_race> races;
  DevVec<Counters> ctr;
  DevVec<int64_t> seqRegs, opIndex;
  DevVec<uint64_t> lockC;              // pairwise path: per-event compact lock facts
  DevVec<int32_t> opMeta, opSeq;
  DevVec<uint64_t> opStart;
  DevVec<hgrd_gpu_trap> traps;
  DevVec<uint32_t> owner;              // fused path: per-element ownership
  bool ownerBits = false;              // owner last held the bit-map layout
  DevVec<uint32_t> shardLo, shardHi;   // sharded launches: INTER summary (min / max block)
  DevVec<uint32_t> hot;                // INTER detection: [0] count, then hot element starts
  DevVec<int> doneKeys;                // pass 2b early stop: per INTER key done flag, key id
  DevVec<uint64_t> doneTargets;        // ... and its first-found element
  uint32_t epoch = 0;
  DevVec<unsigned long long> keyElem;  // fused path: per key minimum element
  DevVec<Candidate> cand;
  DevVec<Counters> ctr2;               // fused pass 2 counters
  DevVec<uint32_t> interTab;           // fused pass 2: (element, site) block sets
  DevVec<unsigned long long> interKeyElem;
  DevVec<uint64_t> targets;
  DevVec<unsigned char> batchBlob;     // hgrd_gpu_check_batch: descriptors | outputs
  unsigned char *hBatch = nullptr;     // pinned staging of the batch blob / outputs
  size_t hBatchCap = 0;
  bool fusedEnabled = true;
  // NVRTC specialisation: 0 off, 1 auto (large launches), 2 always
  int jitMode = 1;
  bool timing = std::getenv("HGRD_NO_DEVICE_TIMING") == nullptr; // device_ms via events
  // development: HGRD_HOST_TRACE=1 prints host-side phase times per check
  bool hostTrace = std::getenv("HGRD_HOST_TRACE") != nullptr;
  bool e1AtSync = false; // e1 recorded at readCountersAndRaces' synchronisation
  bool e1Done = false;   // ... and no GPU work since: the check's end
  bool fusedOrdered = false; // the fused attempt saw traps / the step budget
  bool fusedShardTables = false; // the fused check filled the shard's INTER tables
  std::vector<std::pair<const char *, std::chrono::steady_clock::time_point>> trace;
  hgrdgpu::jit::Cache *jit = nullptr;
  std::string jitErr;
  int jitFailures = 0;
  std::string jitInfo;

  unsigned char *hStage = nullptr;
  size_t hStageCap = 0;
  // per check: counters / per-key minima / race array live in the blob, so
  // a check is one H2D (descriptor + zeroed counters), kernels, one D2H
  Counters *cur = nullptr;
  hgrd_gpu_race *curRaces = nullptr;
  unsigned long long *curKeyElem = nullptr;
  unsigned char *hResult = nullptr; // pinned: counters + races
  size_t hResultCap = 0;
  hgrd_gpu_race *hRaces = nullptr; // pinned copy of the device race array
  hgrd_gpu_trap *hTraps = nullptr; // pinned: traps read with the counters
  size_t hTrapsCap = 0;
  size_t hRacesCap = 0;
  bool racesOnHost = false;
  hgrd_gpu_race *hRacesView = nullptr;
  Counters *hCtr = nullptr;
  uint64_t capHint = 1 << 16;
  uint64_t opHint = 1 << 12;

  // optional per-stage timing (CUDA events on the launching stream)
  bool profiling = false;
  struct Stage {
    const char *name;
    cudaEvent_t a, b;
  };
  std::vector<Stage> stages;      // recorded in the current check
  std::vector<cudaEvent_t> evPool;
  size_t evUsed = 0;
  std::string profileJson;
  unsigned long long kernelLaunches = 0; // own kernels launched (lifetime)
  unsigned long long h2dBytes = 0, d2hBytes = 0; // host<->device copies (lifetime)
  std::map<std::pair<const void *, size_t>, int> occupancy; // (kernel, smem) -> CTAs/SM
  std::set<const void *> smemOptIn;
};

namespace {

int cudaFail(hgrd_gpu_ctx *c, cudaError_t e, const char *what) {
  c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return HGRD_GPU_ECUDA;
}

#define CK(expr)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return cudaFail(c, _e, #expr);                                                   \
  } while (0)

template <class T> int need(hgrd_gpu_ctx *c, DevVec<T> &v, size_t n) {
  if (n == 0)
    n = 1;
  if (v.cap >= n)
    return 0;
  size_t want = std::max(n, v.cap + v.cap / 2);
  if (v.p) {
    CK(cudaStreamSynchronize(c->st));
    CK(cudaFree(v.p));
    v.p = nullptr;
    v.cap = 0;
  }
  cudaError_t e = cudaMalloc(&v.p, want * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    e = cudaMalloc(&v.p, n * sizeof(T));
    want = n;
  }
  if (e != cudaSuccess) {
    v.p = nullptr;
    c->err = "device allocation failed";
    return HGRD_GPU_ENOMEM;
  }
  v.cap = want;
  return 0;
}

#define NEED(v, n)                                                                     \
  do {                                                                                 \
    int _rc = need(c, v, n);                                                           \
    if (_rc < 0)                                                                       \
      return _rc;                                                                      \
  } while (0)

cudaEvent_t poolEvent(hgrd_gpu_ctx *c) {
  if (c->evUsed == c->evPool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evPool.push_back(e);
  }
  return c->evPool[c->evUsed++];
}

// RAII marker around one pipeline stage when profiling is on.
inline void htrace(hgrd_gpu_ctx *c, const char *what) {
  if (c->hostTrace)
    c->trace.emplace_back(what, std::chrono::steady_clock::now());
}

struct StageTimer {
  hgrd_gpu_ctx *c;
  size_t idx = SIZE_MAX;
  StageTimer(hgrd_gpu_ctx *ctx, const char *name) : c(ctx) {
    if (!c->profiling)
      return;
    hgrd_gpu_ctx::Stage s{name, poolEvent(c), poolEvent(c)};
    cudaEventRecord(s.a, c->st);
    c->stages.push_back(s);
    idx = c->stages.size() - 1;
  }
  ~StageTimer() {
    if (idx != SIZE_MAX)
      cudaEventRecord(c->stages[idx].b, c->st);
  }
};

int stage(hgrd_gpu_ctx *c, size_t bytes) {
  if (c->hStageCap >= bytes)
    return 0;
  if (c->hStage) {
    CK(cudaStreamSynchronize(c->st));
    CK(cudaFreeHost(c->hStage));
  }
  size_t want = std::max(bytes, size_t(1) << 20);
  CK(cudaMallocHost(&c->hStage, want));
  c->hStageCap = want;
  return 0;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Static bound on the barrier phases of one thread: straight-line code
// executes each barrier at most once; a barrier inside a loop is unbounded.
void phaseBounds(const hgrd_gpu_launch &L, int &bP, int &bQ, bool &bounded,
                 uint32_t &recInsns, bool &loops) {
  uint32_t nS = 0, nW = 0;
  loops = false;
  bounded = true;
  recInsns = 0;
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (I.op == HGRD_OP_SYNCTHREADS)
      ++nS;
    if (I.op == HGRD_OP_SYNCWARP)
      ++nW;
    if (I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC)
      ++recInsns;
    if (I.op == HGRD_OP_JMP && I.imm <= static_cast<int64_t>(pc)) {
      loops = true;
      for (int64_t q = I.imm; q <= static_cast<int64_t>(pc); ++q) {
        uint8_t op = L.code[q].op;
        if (op == HGRD_OP_SYNCTHREADS || op == HGRD_OP_SYNCWARP)
          bounded = false;
      }
    }
  }
  if (bounded) {
    bP = bitsFor(uint64_t(nS) + 1);
    bQ = bitsFor(uint64_t(nS) + nW + 1);
  } else {
    bP = 8;
    bQ = 8;
  }
}

bool makeLayout(KeyLayout &k, int bE, int bB, int bP, int bW, int bQ, int bL, int nSites) {
  k.bS = 32 - std::max(1, bitsFor(static_cast<uint64_t>(nSites)));
  k.bE = bE;
  k.bB = bB;
  k.bP = bP;
  k.bW = bW;
  k.bQ = bQ;
  k.bL = bL;
  k.shQ = bL;
  k.shW = k.shQ + bQ;
  k.shP = k.shW + bW;
  k.shB = k.shP + bP;
  k.shE = k.shB + bB;
  k.total = k.shE + bE;
  if (k.total > 64)
    return false;
  k.sentinel = k.total == 64 ? ~0ull : ((1ull << k.total) - 1);
  return true;
}

struct Plan {
  std::vector<ParamDev> params;
  std::vector<SiteDev> sites;
  std::vector<uint64_t> confInter, confIntra, locMask, wBase;
  std::vector<int32_t> wHandle;
  uint64_t totalW = 0;
  bool summaryOk = true;
};

// A buffer's upload in flight (hgrd_gpu_buffer_write_async): the context
// stream waits for it on the device before the next work that touches the
// buffer; the host does not block.
void awaitUpload(hgrd_gpu_ctx *c, int32_t h) {
  auto &b = c->bufs[static_cast<size_t>(h)];
  if (b.upload >= 0) {
    cudaStreamWaitEvent(c->st, c->upEvents[static_cast<size_t>(b.upload)], 0);
    c->upFree.push_back(b.upload);
    b.upload = -1;
  }
}

// Every upload a launch's buffers wait for (all of them when L is null).
void awaitUploads(hgrd_gpu_ctx *c, const hgrd_gpu_launch *L) {
  if (c->upFree.size() == c->upEvents.size())
    return; // none in flight
  if (!L) {
    for (size_t h = 0; h < c->bufs.size(); ++h)
      awaitUpload(c, static_cast<int32_t>(h));
    return;
  }
  for (uint32_t p = 0; p < L->n_params; ++p) {
    const int32_t h = L->param_handle[p];
    if (h >= 0 && static_cast<size_t>(h) < c->bufs.size())
      awaitUpload(c, h);
  }
}

// A buffer's pending zero-initialisation, done before anything reads its
// values (host reads and writes, value-needed loads, sequential launches).
int materialize(hgrd_gpu_ctx *c, int32_t h) {
  awaitUpload(c, h);
  auto &b = c->bufs[static_cast<size_t>(h)];
  if (b.zeroPending) {
    CK(cudaMemsetAsync(b.p, 0, static_cast<size_t>(b.elems) * 8, c->st));
    b.zeroPending = false;
  }
  return 0;
}

void planLaunch(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, Plan &P) {
  std::vector<char> written(c->bufs.size(), 0);
  auto handleOfParam = [&](int p) -> int32_t {
    if (p < 0 || static_cast<uint32_t>(p) >= L.n_params)
      return -1;
    int32_t h = L.param_handle[p];
    return (h >= 0 && static_cast<size_t>(h) < c->bufs.size()) ? h : -1;
  };
  for (uint32_t s = 0; s < L.n_sites; ++s)
    if (L.sites[s].kind != HGRD_SITE_LOAD && handleOfParam(L.sites[s].param) >= 0)
      written[static_cast<size_t>(handleOfParam(L.sites[s].param))] = 1;
  std::vector<uint64_t> base(c->bufs.size(), 0);
  std::vector<int> windex(c->bufs.size(), 0);
  for (size_t h = 0; h < c->bufs.size(); ++h)
    if (written[h]) {
      windex[h] = static_cast<int>(P.wBase.size()) + 1;
      base[h] = P.totalW;
      P.wBase.push_back(P.totalW);
      P.wHandle.push_back(static_cast<int32_t>(h));
      P.totalW += static_cast<uint64_t>(c->bufs[h].elems);
    }
  if (P.wBase.empty()) {
    P.wBase.push_back(0);
    P.wHandle.push_back(-1);
  }
  P.params.resize(std::max<uint32_t>(L.n_params, 1));
  for (uint32_t p = 0; p < L.n_params; ++p) {
    ParamDev d{};
    int32_t h = handleOfParam(static_cast<int>(p));
    d.handle = h;
    if (h >= 0) {
      d.ptr = c->bufs[static_cast<size_t>(h)].p;
      d.size = c->bufs[static_cast<size_t>(h)].elems;
      d.written = windex[static_cast<size_t>(h)];
      d.elemBase = base[static_cast<size_t>(h)];
    }
    P.params[p] = d;
  }
  // value-needed loads read buffer contents even in PARALLEL mode
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (I.op == HGRD_OP_LOAD && (I.sub & 1) && static_cast<uint64_t>(I.imm) < L.n_sites) {
      const int32_t h = handleOfParam(L.sites[static_cast<size_t>(I.imm)].param);
      if (h >= 0)
        materialize(c, h);
    }
  }
  P.sites.resize(std::max<uint32_t>(L.n_sites, 1));
  // block privacy only matters for launches spread over several k_fused
  // iterations (one-iteration launches pair INTER on chip): tiny launches
  // skip the analysis and keep every exchange (always correct)
  const int64_t nThreads = L.grid[0] * L.grid[1] * L.grid[2] * L.block[0] * L.block[1] *
                           L.block[2];
  const std::vector<uint8_t> priv = nThreads <= 512 ? std::vector<uint8_t>(L.n_sites, 0)
                                                    : hgrdgpu::blockPrivateSites(L);
  for (uint32_t s = 0; s < L.n_sites; ++s) {
    SiteDev d{};
    d.param = L.sites[s].param;
    d.loc = L.sites[s].loc;
    d.kind = L.sites[s].kind;
    d.aop = L.sites[s].atomic_op;
    d.scope = L.sites[s].scope;
    int32_t h = handleOfParam(d.param);
    d.record = (h >= 0 && written[static_cast<size_t>(h)]) ? 1 : 0;
    d.own = d.record && !priv[s];
    P.sites[s] = d;
  }
  P.summaryOk = L.n_sites <= static_cast<uint32_t>(kMaxSites);
  const uint32_t ns = std::min<uint32_t>(L.n_sites, kMaxSites);
  P.confInter.assign(std::max<uint32_t>(ns, 1), 0);
  P.confIntra.assign(std::max<uint32_t>(ns, 1), 0);
  P.locMask.assign(std::max<uint32_t>(L.n_locs, 1), 0);
  // static pair rules (reference :752-758): a write, and not two atomics
  // whose scopes both cover the pair
  for (uint32_t a = 0; a < ns; ++a) {
    const auto &A = L.sites[a];
    P.locMask[static_cast<size_t>(A.loc)] |= 1ull << a;
    for (uint32_t b = 0; b < ns; ++b) {
      const auto &B = L.sites[b];
      const bool write = A.kind != HGRD_SITE_LOAD || B.kind != HGRD_SITE_LOAD;
      const bool bothAtomic = A.kind == HGRD_SITE_ATOMIC && B.kind == HGRD_SITE_ATOMIC;
      const bool devBoth = A.scope == HGRD_SCOPE_DEVICE && B.scope == HGRD_SCOPE_DEVICE;
      const bool blkBoth = A.scope != HGRD_SCOPE_NONE && B.scope != HGRD_SCOPE_NONE;
      if (write && !(bothAtomic && devBoth))
        P.confInter[a] |= 1ull << b;
      if (write && !(bothAtomic && blkBoth))
        P.confIntra[a] |= 1ull << b;
    }
  }
}

struct BlobOffsets {
  size_t code, sites, params, regs, cInter, cIntra, locMask, wBase, wHandle;
  size_t keyElem, ctr, races, h2d, total;
  int nW, nKeys;
};

int uploadBlob(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const Plan &P, BlobOffsets &o) {
  size_t off = 0;
  auto put = [&](size_t bytes) {
    size_t at = off;
    off = align16(off + bytes);
    return at;
  };
  o.code = put(sizeof(hgrd_gpu_insn) * L.n_code);
  o.sites = put(sizeof(SiteDev) * P.sites.size());
  o.params = put(sizeof(ParamDev) * P.params.size());
  o.regs = put(sizeof(int64_t) * std::max<uint32_t>(L.n_regs, 1));
  o.cInter = put(8 * P.confInter.size());
  o.cIntra = put(8 * P.confIntra.size());
  o.locMask = put(8 * P.locMask.size());
  o.wBase = put(8 * P.wBase.size());
  o.wHandle = put(4 * P.wHandle.size());
  const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  o.nKeys = 3 * nLocs * nLocs;
  o.keyElem = put(8 * static_cast<size_t>(o.nKeys));
  o.ctr = put(sizeof(Counters));
  o.h2d = off;
  o.races = put(sizeof(hgrd_gpu_race) * static_cast<size_t>(o.nKeys));
  o.total = off;
  o.nW = static_cast<int>(P.wBase.size());
  int rc = stage(c, o.total);
  if (rc < 0)
    return rc;
  // every check ends synchronised, so the pinned staging buffer is free here
  NEED(c->blob, o.total);
  unsigned char *h = c->hStage;
  std::memcpy(h + o.code, L.code, sizeof(hgrd_gpu_insn) * L.n_code);
  std::memcpy(h + o.sites, P.sites.data(), sizeof(SiteDev) * P.sites.size());
  std::memcpy(h + o.params, P.params.data(), sizeof(ParamDev) * P.params.size());
  if (L.n_regs)
    std::memcpy(h + o.regs, L.reg_init, sizeof(int64_t) * L.n_regs);
  std::memcpy(h + o.cInter, P.confInter.data(), 8 * P.confInter.size());
  std::memcpy(h + o.cIntra, P.confIntra.data(), 8 * P.confIntra.size());
  std::memcpy(h + o.locMask, P.locMask.data(), 8 * P.locMask.size());
  std::memcpy(h + o.wBase, P.wBase.data(), 8 * P.wBase.size());
  std::memcpy(h + o.wHandle, P.wHandle.data(), 4 * P.wHandle.size());
  std::memset(h + o.keyElem, 0xff, 8 * static_cast<size_t>(o.nKeys));
  std::memset(h + o.ctr, 0, sizeof(Counters));
  CK(cudaMemcpyAsync(c->blob.p, h, o.h2d, cudaMemcpyHostToDevice, c->st));
  c->h2dBytes += o.h2d;
  c->cur = reinterpret_cast<Counters *>(c->blob.p + o.ctr);
  c->curRaces = reinterpret_cast<hgrd_gpu_race *>(c->blob.p + o.races);
  c->curKeyElem = reinterpret_cast<unsigned long long *>(c->blob.p + o.keyElem);
  return 0;
}

// Counters and (speculatively) the whole race array in one round trip
// (they are adjacent in the blob).
int readCountersAndRaces(hgrd_gpu_ctx *c, size_t nKeys) {
  const size_t racesOff = reinterpret_cast<unsigned char *>(c->curRaces) -
                          reinterpret_cast<unsigned char *>(c->cur);
  const size_t bytes = racesOff + sizeof(hgrd_gpu_race) * nKeys;
  if (c->hResultCap < bytes) {
    if (c->hResult)
      CK(cudaFreeHost(c->hResult));
    CK(cudaMallocHost(&c->hResult, std::max<size_t>(bytes, 4096)));
    c->hResultCap = std::max<size_t>(bytes, 4096);
  }
  CK(cudaMemcpyAsync(c->hResult, c->cur, bytes, cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += bytes;
  // the check's end event rides on this synchronisation: when the check
  // finishes here (no INTER pass), no second round trip is needed
  if (c->timing)
    CK(cudaEventRecord(c->e1, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->e1AtSync = c->timing;
  std::memcpy(c->hCtr, c->hResult, sizeof(Counters));
  c->hRacesView = reinterpret_cast<hgrd_gpu_race *>(c->hResult + racesOff);
  c->racesOnHost = true;
  return 0;
}

// Counters and (speculatively) the first `trapCap` trap slots in one round
// trip: a SEQUENTIAL launch needs both, and tiny sweep launches are bound by
// round trips.
int readCountersAndTraps(hgrd_gpu_ctx *c, size_t trapCap) {
  if (c->hTrapsCap < trapCap) {
    if (c->hTraps)
      CK(cudaFreeHost(c->hTraps));
    c->hTraps = nullptr;
    CK(cudaMallocHost(&c->hTraps, sizeof(hgrd_gpu_trap) * trapCap));
    c->hTrapsCap = trapCap;
  }
  CK(cudaMemcpyAsync(c->hCtr, c->cur, sizeof(Counters), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(c->hTraps, c->traps.p, sizeof(hgrd_gpu_trap) * trapCap,
                     cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += sizeof(Counters) + sizeof(hgrd_gpu_trap) * trapCap;
  if (c->timing) // the check's end event, when nothing follows (see e1AtSync)
    CK(cudaEventRecord(c->e1, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->e1AtSync = c->timing;
  return 0;
}

int readCounters(hgrd_gpu_ctx *c) {
  CK(cudaMemcpyAsync(c->hCtr, c->cur, sizeof(Counters), cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += sizeof(Counters);
  CK(cudaStreamSynchronize(c->st));
  return 0;
}

// Sort + detect + witness over `n` records in c->keys/c->vals (layout kl).
int fetchRaces(hgrd_gpu_ctx *c, hgrd_gpu_result *R);

DetectArgs detectArgs(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const LaunchDev &D,
                      const BlobOffsets &o, uint64_t n, int kindMask) {
  DetectArgs A{};
  A.n = n;
  A.kl = D.kl;
  A.sites = D.sites;
  A.confInter = D.confInter;
  A.confIntra = D.confIntra;
  A.locMask = D.locMask;
  A.nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  A.nSites = static_cast<int>(L.n_sites);
  A.tpb = D.tpb;
  A.ws = D.ws;
  A.wBase = reinterpret_cast<const uint64_t *>(c->blob.p + o.wBase);
  A.wHandle = reinterpret_cast<const int32_t *>(c->blob.p + o.wHandle);
  A.nW = o.nW;
  A.kindMask = kindMask;
  return A;
}

int detect(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, LaunchDev &D, const BlobOffsets &o,
           uint64_t n, bool pairwise, bool locks, hgrd_gpu_result *R, int kindMask = 7,
           bool append = false) {
  const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  const int nKeys = 3 * nLocs * nLocs;
  if (n <= 1 && !append) {
    // fewer than two records hold no pair (detectRaces needs x < y in one
    // element group): no detect kernels, no read-back round trip -- tiny
    // sweep launches are bound by these round trips
    c->racesOnHost = false;
    R->n_races = 0;
    return 0;
  }
  if (!append)
    CK(cudaMemsetAsync(&c->cur->nRaces, 0, sizeof(unsigned), c->st));
  DetectArgs A = detectArgs(c, L, D, o, n, kindMask);
  if (n > 1) {
    if (!pairwise) {
      NEED(c->keysAlt, n);
      NEED(c->valsAlt, n);
      cub::DoubleBuffer<uint64_t> dk(c->keys.p, c->keysAlt.p);
      cub::DoubleBuffer<uint32_t> dv(c->vals.p, c->valsAlt.p);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, static_cast<int64_t>(n), 0,
                                         D.kl.total, c->st));
      NEED(c->cubTemp, tb);
      {
        StageTimer t(c, "sort_records");
        CK(cub::DeviceRadixSort::SortPairs(c->cubTemp.p, tb, dk, dv, static_cast<int64_t>(n),
                                           0, D.kl.total, c->st));
      }
      A.keys = dk.Current();
      A.vals = dv.Current();
      NEED(c->keySeg, static_cast<size_t>(nKeys));
      CK(cudaMemsetAsync(c->keySeg.p, 0xff, sizeof(uint32_t) * nKeys, c->st));
      const unsigned g = static_cast<unsigned>((n + 255) / 256);
      if (kindMask == 1) { // INTER only: hot elements go to a warp each
        const uint32_t hotCap = 1u << 16;
        NEED(c->hot, hotCap + 1);
        CK(cudaMemsetAsync(c->hot.p, 0, sizeof(uint32_t), c->st));
        A.hotCount = c->hot.p;
        A.hotList = c->hot.p + 1;
        A.hotCap = hotCap;
      }
      {
        StageTimer t(c, "k_detect_summary");
        k_detect_summary<<<g, 256, 0, c->st>>>(A, c->keySeg.p);
      }
      CK(cudaGetLastError());
      if (A.hotList) {
        StageTimer t(c, "k_detect_hot");
        k_detect_hot<<<c->nSM * 2, 256, 0, c->st>>>(A, c->keySeg.p);
        CK(cudaGetLastError());
        ++c->kernelLaunches;
      }
      if (kindMask & 6) {
        DetectArgs Ai = A;
        Ai.kindMask = kindMask & 6;
        StageTimer t(c, "k_witness");
        k_witness<<<(nKeys + 127) / 128, 128, 0, c->st>>>(Ai, c->keySeg.p, nKeys, c->curRaces,
                                                           c->cur);
        ++c->kernelLaunches;
      }
      CK(cudaGetLastError());
      if (kindMask & 1) { // INTER-BLOCK: warp per key (hot elements)
        StageTimer t(c, "k_witness_inter");
        const int warps = (nKeys + 2) / 3;
        k_witness_inter<<<(warps + 7) / 8, 256, 0, c->st>>>(A, c->keySeg.p, nKeys, c->curRaces,
                                                             c->cur);
        ++c->kernelLaunches;
      }
      CK(cudaGetLastError());
      ++c->kernelLaunches;
    } else {
      // canonical-order records, stable sort by element
      A.keys = c->keys.p;
      A.vals = c->vals.p;
      NEED(c->elemK, n);
      NEED(c->elemKAlt, n);
      NEED(c->order, n);
      NEED(c->orderAlt, n);
      const unsigned g = static_cast<unsigned>((n + 255) / 256);
      // PARALLEL lock launches (D.opStride): records arrive in chunk order,
      // so the sort key carries the canonical order too (element | thread |
      // seq), shifted back to the element afterwards
      const int canonBits = D.opStride ? bitsFor(static_cast<uint64_t>(D.nThreads)) +
                                             bitsFor(L.n_code + 1)
                                       : 0;
      if (canonBits)
        k_elem_keys_canon<<<g, 256, 0, c->st>>>(
            c->keys.p, c->vals.p, n, D.kl, D.tpb, D.ws,
            bitsFor(static_cast<uint64_t>(D.nThreads)), bitsFor(L.n_code + 1), c->elemK.p,
            c->order.p);
      else
        k_elem_keys<<<g, 256, 0, c->st>>>(c->keys.p, n, D.kl.shE, c->elemK.p, c->order.p);
      CK(cudaGetLastError());
      cub::DoubleBuffer<uint64_t> dk(c->elemK.p, c->elemKAlt.p);
      cub::DoubleBuffer<uint32_t> dv(c->order.p, c->orderAlt.p);
      size_t tb = 0;
      const int sortBits = std::max(D.kl.bE, 1) + canonBits;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, static_cast<int64_t>(n), 0,
                                         sortBits, c->st));
      NEED(c->cubTemp, tb);
      CK(cub::DeviceRadixSort::SortPairs(c->cubTemp.p, tb, dk, dv, static_cast<int64_t>(n), 0,
                                         sortBits, c->st));
      if (canonBits) {
        k_shift_keys<<<g, 256, 0, c->st>>>(dk.Current(), n, canonBits);
        CK(cudaGetLastError());
      }
      NEED(c->keyPair, 2 * static_cast<size_t>(nKeys)); // first rows, then their y
      CK(cudaMemsetAsync(c->keyPair.p, 0xff, 2 * sizeof(unsigned long long) * nKeys, c->st));
      unsigned long long *keyY = c->keyPair.p + nKeys;
      {
        const uint32_t bigCap = 1u << 16; // (group start, end) pairs
        NEED(c->hot, 2 * bigCap + 1);
        CK(cudaMemsetAsync(c->hot.p, 0, sizeof(uint32_t), c->st));
        A.hotCount = c->hot.p;
        A.hotList = c->hot.p + 1;
        A.hotCap = bigCap;
        LockC *lc = nullptr;
        if (locks) {
          NEED(c->lockC, n * (sizeof(LockC) / 8));
          lc = reinterpret_cast<LockC *>(c->lockC.p);
          StageTimer t(c, "k_lock_info");
          k_lock_info<<<g, 256, 0, c->st>>>(A, D, dv.Current(), lc);
          ++c->kernelLaunches;
        }
        StageTimer t(c, "k_detect_pairwise");
        k_detect_pairwise<<<g, 256, 0, c->st>>>(A, D, dk.Current(), dv.Current(), locks, lc,
                                                 c->keyPair.p);
        k_detect_pairwise_big<<<c->nSM * 4, 256, 0, c->st>>>(A, D, dk.Current(), dv.Current(),
                                                             locks, lc, c->keyPair.p);
        k_pair_first_y<<<nKeys, 128, 0, c->st>>>(A, D, dk.Current(), dv.Current(), locks, lc,
                                                 c->keyPair.p, keyY);
        c->kernelLaunches += 2;
      }
      CK(cudaGetLastError());
      k_decode_pairwise<<<(nKeys + 127) / 128, 128, 0, c->st>>>(
          A, dk.Current(), dv.Current(), c->keyPair.p, keyY, nKeys, c->curRaces, c->cur);
      CK(cudaGetLastError());
      c->kernelLaunches += 3;
    }
  }
  int rc = readCountersAndRaces(c, static_cast<size_t>(nKeys));
  if (rc < 0)
    return rc;
  return fetchRaces(c, R);
}

int fetchRaces(hgrd_gpu_ctx *c, hgrd_gpu_result *R) {
  if (c->hCtr->flags & (kFlagLockSet | kFlagSegment)) {
    c->err = (c->hCtr->flags & kFlagLockSet)
                 ? std::string("pairwise detector limit exceeded: a lock set of more than 8 locks")
                 : std::string("pairwise detector limit exceeded: 2^32 or more events");
    return HGRD_GPU_ENOTSUP;
  }
  const unsigned nr = c->hCtr->nRaces;
  R->n_races = nr;
  if (nr > R->race_cap)
    return HGRD_GPU_E2BIG;
  if (nr && c->racesOnHost) {
    std::memcpy(R->races, c->hRacesView, sizeof(hgrd_gpu_race) * nr);
  } else if (nr) {
    CK(cudaMemcpyAsync(R->races, c->curRaces, sizeof(hgrd_gpu_race) * nr,
                       cudaMemcpyDeviceToHost, c->st));
    c->d2hBytes += sizeof(hgrd_gpu_race) * nr;
    CK(cudaStreamSynchronize(c->st));
  }
  c->racesOnHost = false;
  return 0;
}

} // namespace


// Lazily compiled specialised kernels of one launch.
struct JitGetter {
  hgrd_gpu_ctx *c;
  const hgrd_gpu_launch *L;
  bool enabled;
  std::vector<uint8_t> rec; // per site: produces race-check records
  std::vector<hgrdgpu::jit::JitParam> params; // per kernel parameter: size, element base
  int streamSite = -1;      // a streamed load (staged by k_fused), or -1
  int64_t streamOff = 0;
  const void *get(hgrdgpu::jit::Variant v) {
    if (!enabled)
      return nullptr;
    if (!c->jit)
      c->jit = hgrdgpu::jit::create();
    std::string err;
    const void *k = hgrdgpu::jit::get(c->jit, *L, rec, params, v, err);
    if (!k && !err.empty()) {
      c->jitErr = err;
      ++c->jitFailures;
    }
    return k;
  }
};

// The launch's streamed load, if any (JIT bodies only): a value-needed load
// of a buffer the launch does not write whose index is the dense thread id
// plus a constant (affine.hpp streamSites) — k_fused stages its values.
void markStream(const hgrd_gpu_launch &L, const std::vector<ParamDev> &params,
                JitGetter &jk) {
  if (!jk.enabled || std::getenv("HGRD_NO_STREAM"))
    return;
  std::vector<char> needed(L.n_sites, 0);
  for (uint32_t pc = 0; pc < L.n_code; ++pc)
    if (L.code[pc].op == HGRD_OP_LOAD && (L.code[pc].sub & 1))
      needed[static_cast<size_t>(L.code[pc].imm)] = 1;
  bool any = false;
  for (char n : needed)
    any |= n != 0;
  if (!any)
    return;
  const std::vector<int64_t> off = hgrdgpu::streamSites(L);
  for (uint32_t s = 0; s < L.n_sites; ++s) {
    const int32_t p = L.sites[s].param;
    if (!needed[s] || off[s] == hgrdgpu::kNoStream || p < 0 ||
        static_cast<size_t>(p) >= params.size() || params[static_cast<size_t>(p)].handle < 0 ||
        params[static_cast<size_t>(p)].written)
      continue;
    jk.streamSite = static_cast<int>(s);
    jk.streamOff = off[s];
    jk.rec[s] |= 4;
    return;
  }
}

int launchExpandPar(hgrd_gpu_ctx *c, const LaunchDev &D, unsigned blocks, size_t smem,
                    const void *jitKernel, const char *stage) {
  const void *fn = jitKernel ? jitKernel : reinterpret_cast<const void *>(k_expand_par<InterpBody>);
  if (smem > 48 * 1024 && c->smemOptIn.insert(fn).second) {
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            227 * 1024 - static_cast<int>(fa.sharedSizeBytes)));
  }
  void *args[] = {const_cast<LaunchDev *>(&D)};
  {
    StageTimer t(c, stage);
    CK(cudaLaunchKernel(fn, dim3(blocks), dim3(256), args, smem, c->st));
  }
  ++c->kernelLaunches;
  return 0;
}

// ---------------------------------------------------------------------------
// Fused block-local path (fused.cuh) + pass 2 for elements shared by blocks.

template <int NT, int IPT>
size_t fusedSmemBytes(const hgrd_gpu_launch &L, const Plan &P, int nKeys) {
  const size_t nKeysPad = (static_cast<size_t>(nKeys) + 3) & ~size_t(3);
  return align16(sizeof(FusedSmem<NT, IPT>)) + 12 * nKeysPad + sizeof(hgrd_gpu_insn) * L.n_code +
         sizeof(SiteDev) * P.sites.size() + sizeof(ParamDev) * P.params.size() +
         16 * P.sites.size();
}

int readCountersFrom(hgrd_gpu_ctx *c, Counters *dev) {
  CK(cudaMemcpyAsync(c->hCtr, dev, sizeof(Counters), cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += sizeof(Counters);
  CK(cudaStreamSynchronize(c->st));
  return 0;
}

template <int NT, int IPT>
int launchFused(hgrd_gpu_ctx *c, const FusedArgs &F, size_t smem, const void *jitKernel) {
  const void *fn =
      jitKernel ? jitKernel : reinterpret_cast<const void *>(k_fused<NT, IPT, InterpBody>);
  if (c->smemOptIn.insert(fn).second) { // once per kernel: allow up to 227 KB in total
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            227 * 1024 - static_cast<int>(fa.sharedSizeBytes)));
  }
  int &perSM = c->occupancy[std::make_pair(fn, smem)];
  if (perSM == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSM, fn, NT, smem));
    perSM = std::max(perSM, 1);
  }
  const int64_t grid = std::max<int64_t>(
      1, std::min<int64_t>(F.nIters, static_cast<int64_t>(c->nSM) * std::max(perSM, 1)));
  void *args[] = {const_cast<FusedArgs *>(&F)};
  htrace(c, "pre-launch");
  StageTimer t(c, jitKernel ? "k_fused[jit]" : "k_fused");
  CK(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(NT), args, smem,
                      c->st));
  htrace(c, "launched");
  return 0;
}

// Returns 1 when the launch was fully checked, 0 to fall back to the
// general pipeline, < 0 on error.  D.kl must hold the general key layout
// (used by pass 2).
// Shard mode (shard = true): only blocks [b0, b1), no ownership exchanges
// and no pass 2 — the caller combines the shards' INTER summaries
// (hgrd_gpu_shard_*).
int runFused(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, LaunchDev D, const BlobOffsets &o,
             const Plan &P, hgrd_gpu_result *R, uint32_t recInsns, bool loops,
             JitGetter &jk, int64_t b0 = 0, int64_t b1 = -1, bool shard = false,
             uint32_t *shardLo = nullptr, uint32_t *shardHi = nullptr) {
  c->fusedOrdered = false;
  c->fusedShardTables = false;
  if (b1 < 0)
    b1 = D.nBlocks;
  const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  const int nKeys = 3 * nLocs * nLocs;
  static const int64_t kIterThreads = [] { // development knob: MiniCU threads per iteration
    const char *e = std::getenv("HGRD_FUSED_ITER");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(0);
  }();
  const uint64_t per = std::max<uint32_t>(recInsns, 1);
  // MiniCU threads per iteration: 512, or 1024 when one record per thread
  // still fills only the x4 record capacity and the launch is large enough
  // (2^22+ threads) for the fewer iterations to keep every CTA busy — the
  // per-iteration barriers and resets are then paid half as often
  // (A/B: profiles/r02/ab_pair_bits.txt, histogram 1.29 -> 1.12 ms; the
  // 2^20-thread stencil lost with larger iterations)
  const int64_t iterThreads =
      kIterThreads ? kIterThreads
                   : (!loops && per == 1 && D.nThreads >= (int64_t(1) << 22) ? 1024 : 512);
  // (at most 256: a record keeps its MiniCU block within the iteration in
  // 8 bits, packR1 / rBlk in fused.cuh)
  int64_t bpi = std::min<int64_t>(kMaxIterBlocks, std::max<int64_t>(1, iterThreads / D.tpb));
  while (bpi > 1 && static_cast<uint64_t>(bpi * D.tpb) * per > 4096)
    bpi /= 2;
  const uint64_t perIter = static_cast<uint64_t>(bpi * D.tpb) * per;
  if (bpi * D.tpb > 65536 || (!loops && perIter > 4096))
    return 0;
  // record capacity per iteration: 256 threads x 4, x 8, x 12 or x 16 (the
  // smallest that holds a straight-line iteration: shared memory decides how
  // many CTAs share an SM — x 12 keeps two, x 16 one)
  const int ipt = (!loops && perIter <= 1024)   ? 4
                  : (!loops && perIter <= 2048) ? 8
                  : (!loops && perIter <= 3072) ? 12
                                                : 16;
  const hgrdgpu::jit::Variant variant = ipt == 4    ? hgrdgpu::jit::kFusedNarrow
                                        : ipt == 8  ? hgrdgpu::jit::kFusedMid
                                        : ipt == 12 ? hgrdgpu::jit::kFused12
                                                    : hgrdgpu::jit::kFusedWide;
  const void *jitKernel = jk.get(variant);
  // the streamed load's staging: two buffers of one iteration's values (+
  // 16-byte alignment slack), only with the JIT body that reads them
  const bool streamed = jitKernel && jk.streamSite >= 0;
  const int stageCap = streamed ? static_cast<int>(bpi * D.tpb) + 4 : 0;
  // ownership table (device.cuh): the reduction layout (two words per
  // element, epoch-tagged: no memset between launches) when it fits L2
  // comfortably, else the bit map (two bits per element, cleared per launch)
  static const char *redEnv = std::getenv("HGRD_OWNER_RED"); // A/B knob: 0 / 1 forces a layout
  const bool ownerRed = redEnv ? std::atoi(redEnv) != 0 : 8 * P.totalW <= (uint64_t(32) << 20);
  // small reduction tables: each CTA keeps a bit map of the elements it has
  // seen become MULTI and skips their joins (a hot 2^16-bin table is joined
  // by every block; HGRD_NO_KNOWN=1 for A/B)
  static const bool noKnown = std::getenv("HGRD_NO_KNOWN") != nullptr;
  const uint32_t knownWords =
      ownerRed && !noKnown && P.totalW <= kKnownMax ? static_cast<uint32_t>((P.totalW + 31) / 32)
                                                    : 0;
  const size_t smem = (ipt == 4    ? fusedSmemBytes<256, 4>(L, P, nKeys)
                       : ipt == 8  ? fusedSmemBytes<256, 8>(L, P, nKeys)
                       : ipt == 12 ? fusedSmemBytes<256, 12>(L, P, nKeys)
                                   : fusedSmemBytes<256, 16>(L, P, nKeys)) +
                      (streamed ? 16 + 16 * static_cast<size_t>(stageCap) : 0) +
                      (knownWords ? 16 + 4 * static_cast<size_t>(knownWords) : 0);
  // (+16: the device places the stage and the known map after a 16-byte
  // alignment of the layout above, which this sum does not round up)
  if (smem > 227 * 1024)
    return 0;

  const uint64_t nOwn = std::max<uint64_t>(P.totalW, 1);
  const size_t ownerN = ownerRed ? 2 * nOwn : (nOwn + 15) / 16;
  const bool fresh = c->owner.cap < ownerN;
  NEED(c->owner, ownerN);
  if (ownerRed) {
    // (a bit map leaves words that are no valid epoch tags: clear after one)
    if (fresh || c->epoch >= 4094 || c->ownerBits) {
      CK(cudaMemsetAsync(c->owner.p, 0, c->owner.cap * sizeof(uint32_t), c->st));
      c->epoch = 0;
      c->ownerBits = false;
    }
    ++c->epoch;
  } else {
    CK(cudaMemsetAsync(c->owner.p, 0, ownerN * sizeof(uint32_t), c->st));
    c->ownerBits = true;
  }
  const uint32_t candCap = 1u << 16;
  NEED(c->cand, candCap);

  FusedArgs F{};
  F.L = D;
  F.nLocs = nLocs;
  F.nKeys = nKeys;
  F.bpi = static_cast<int>(bpi);
  F.R = (loops || recInsns == 0) ? 0u : recInsns; // straight-line code: static record slots
  F.blockBase = b0;
  F.blockEnd = b1;
  F.nIters = (b1 - b0 + bpi - 1) / bpi;
  // a launch that fits one iteration finds its INTER pairs on chip as well
  // (no ownership exchanges, no pass 2); shards leave INTER to their tables
  F.interOnChip = !shard && F.nIters == 1;
  bool anyOwn = false; // a buffer two blocks may reach (affine.cpp could not prove privacy)
  for (const SiteDev &sd : P.sites)
    anyOwn |= sd.record && sd.own;
  F.owner = (shard || F.interOnChip || !anyOwn) ? nullptr : c->owner.p;
  F.ownerRed = ownerRed;
  if (shard && shardLo) { // the shard's (element, site) block min / max, from the records
    F.shardLo = shardLo;
    F.shardHi = shardHi;
    F.nSitesTab = static_cast<int>(L.n_sites);
  }
  F.epoch = c->epoch;
  F.keyElem = c->curKeyElem;
  F.cand = c->cand.p;
  F.candCap = candCap;
  F.candCount = &c->cur->candCount;
  F.nW = o.nW;
  F.races = c->curRaces;
  F.wBase = reinterpret_cast<const uint64_t *>(c->blob.p + o.wBase);
  F.wHandle = reinterpret_cast<const int32_t *>(c->blob.p + o.wHandle);
  if (const char *ab = std::getenv("HGRD_FUSED_ABLATE"))
    F.ablate = std::atoi(ab);
  if (streamed) {
    const ParamDev &sp = P.params[static_cast<size_t>(P.sites[jk.streamSite].param)];
    F.stream = sp.ptr;
    F.streamOff = jk.streamOff;
    F.streamSize = sp.size;
    F.stageCap = stageCap;
  }
  F.knownWords = F.owner ? knownWords : 0;
  int rc = ipt == 4    ? launchFused<256, 4>(c, F, smem, jitKernel)
           : ipt == 8  ? launchFused<256, 8>(c, F, smem, jitKernel)
           : ipt == 12 ? launchFused<256, 12>(c, F, smem, jitKernel)
                       : launchFused<256, 16>(c, F, smem, jitKernel);
  if (rc < 0)
    return rc;
  CK(cudaGetLastError());
  ++c->kernelLaunches;
  if (F.owner && ownerRed) { // any element reached from two blocks? (read with the counters)
    StageTimer t(c, "k_owner_any");
    k_owner_any<<<static_cast<unsigned>(std::min<uint64_t>((P.totalW + 255) / 256,
                                                           uint64_t(c->nSM) * 8)),
                  256, 0, c->st>>>(c->owner.p, P.totalW, c->epoch << 20, D.ctr);
    CK(cudaGetLastError());
    ++c->kernelLaunches;
  }
  rc = readCountersAndRaces(c, static_cast<size_t>(nKeys));
  if (rc < 0)
    return rc;
  htrace(c, "counters");
  const Counters h = *c->hCtr;
  // traps and the step budget need the canonical order: the PARALLEL
  // expansion would see the same counts, so the caller goes SEQUENTIAL
  c->fusedOrdered = (h.flags & kFlagAbort) || h.traps > 0 ||
                    static_cast<int64_t>(h.steps) > L.step_budget;
  if (c->fusedOrdered || (h.flags & kFlagFusedOverflow))
    return 0;
  R->steps = static_cast<int64_t>(h.steps);
  R->instances = h.instances;
  R->records = h.records;
  R->mode = L.flags & ~HGRD_LAUNCH_SEQUENTIAL;
  c->fusedShardTables = F.shardLo != nullptr;
  if (shard || !(h.flags & kFlagShared)) {
    if (fetchRaces(c, R) < 0) // (races read from the same synchronisation)
      return -1;
    c->e1Done = c->e1AtSync;
    return 1;
  }

  // pass 2: INTER-BLOCK over the elements two or more blocks touched
  NEED(c->ctr2, 1);
  LaunchDev D2 = D;
  D2.ctr = c->ctr2.p;
  D2.ownerFilter = c->owner.p;
  D2.ownerMultiTag = (c->epoch << 20) | (ownerRed ? 0u : kOwnerMulti); // (ownerIsMulti)
  const size_t sm2 = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * P.sites.size() +
                     sizeof(ParamDev) * P.params.size();
  const unsigned grid2 = static_cast<unsigned>(std::min<uint64_t>(
      ((static_cast<uint64_t>(D.nThreads) + 31) / 32 + 7) / 8, uint64_t(c->nSM) * 8));
  std::vector<int> interKeys;        // realised INTER keys ...
  std::vector<uint64_t> interTarget; // ... and their first-found elements
  // buffers two blocks can reach with exactly one recording site each: the
  // ownership table alone gives the INTER keys (no summary pass)
  SingleSites ss{};
  bool single = o.nW <= 8;
  if (single) {
    ss.nW = o.nW;
    for (int w = 0; w < o.nW; ++w) {
      ss.wBase[w] = P.wBase[static_cast<size_t>(w)];
      ss.site[w] = -1;
    }
    for (uint32_t s = 0; s < L.n_sites && single; ++s) {
      const SiteDev &sd = P.sites[s];
      if (!sd.record || !sd.own || sd.param < 0)
        continue;
      const int w = P.params[static_cast<size_t>(sd.param)].written - 1;
      if (w < 0 || w >= o.nW)
        continue;
      if (ss.site[w] >= 0 && ss.site[w] != static_cast<int32_t>(s))
        single = false;
      ss.site[w] = static_cast<int32_t>(s);
    }
  }
  if (single) {
    NEED(c->interKeyElem, static_cast<size_t>(nKeys));
    CK(cudaMemsetAsync(c->interKeyElem.p, 0xff, 8 * static_cast<size_t>(nKeys), c->st));
    StageTimer t(c, "k_inter_scan_single");
    k_inter_scan_single<<<static_cast<unsigned>((P.totalW + 255) / 256), 256, 0, c->st>>>(
        c->owner.p, D2.ownerMultiTag, P.totalW, ss, D.sites, D.confInter, nLocs,
        c->interKeyElem.p);
  } else {
    // 2a: record-free INTER summary of the shared elements, then the realised
    //     INTER keys and their first-found (minimum) elements
    const size_t nTab = static_cast<size_t>(P.totalW) * L.n_sites;
    NEED(c->interTab, nTab);
    CK(cudaMemsetAsync(c->interTab.p, 0xff, nTab * 4, c->st));
    NEED(c->interKeyElem, static_cast<size_t>(nKeys));
    CK(cudaMemsetAsync(c->interKeyElem.p, 0xff, 8 * static_cast<size_t>(nKeys), c->st));
    CK(cudaMemsetAsync(c->ctr2.p, 0, sizeof(Counters), c->st));
    LaunchDev Ds = D2;
    Ds.interTab = c->interTab.p;
    Ds.nSitesTab = static_cast<int>(L.n_sites);
    Ds.keys = nullptr;
    Ds.vals = nullptr;
    Ds.capacity = 0;
    Ds.chunk = 64;
    const void *jx = jk.get(hgrdgpu::jit::kExpandPar);
    rc = launchExpandPar(c, Ds, grid2, sm2, jx,
                         jx ? "k_expand_par_inter[jit]" : "k_expand_par_inter");
    if (rc < 0)
      return rc;
    {
      StageTimer t(c, "k_inter_scan");
      k_inter_scan<<<static_cast<unsigned>((P.totalW + 255) / 256), 256, 0, c->st>>>(
          c->owner.p, D2.ownerMultiTag, P.totalW, c->interTab.p, static_cast<int>(L.n_sites),
          D.sites, D.confInter, nLocs, c->interKeyElem.p);
    }
  }
  {
    CK(cudaGetLastError());
    c->kernelLaunches += 1;
    std::vector<unsigned long long> ke(static_cast<size_t>(nKeys));
    CK(cudaMemcpyAsync(ke.data(), c->interKeyElem.p, 8 * static_cast<size_t>(nKeys),
                       cudaMemcpyDeviceToHost, c->st));
    c->d2hBytes += 8 * static_cast<size_t>(nKeys);
    CK(cudaStreamSynchronize(c->st));
    std::vector<uint64_t> targets;
    for (int K = 0; K < nKeys; K += 3)
      if (ke[static_cast<size_t>(K)] != ~0ull) {
        targets.push_back(ke[static_cast<size_t>(K)]);
        interKeys.push_back(K);
        interTarget.push_back(ke[static_cast<size_t>(K)]);
      }
    std::sort(targets.begin(), targets.end());
    targets.erase(std::unique(targets.begin(), targets.end()), targets.end());
    if (targets.empty())
      return fetchRaces(c, R) < 0 ? -1 : 1; // no INTER race (pass-1 races stand)
    NEED(c->targets, targets.size());
    CK(cudaMemcpy(c->targets.p, targets.data(), 8 * targets.size(), cudaMemcpyHostToDevice));
    c->h2dBytes += 8 * targets.size();
    // 2b: records of only those elements -> first pairs (witnesses)
    D2.targets = c->targets.p;
    D2.nTargets = static_cast<int>(targets.size());
  }
  int bP = D.kl.bP, bQ = D.kl.bQ;
  for (int attempt = 0; attempt < 8; ++attempt) {
    if (!makeLayout(D2.kl, D.kl.bE, D.kl.bB, bP, D.kl.bW, bQ, D.kl.bL, D.nSites)) {
      c->err = "packed record key wider than 64 bits";
      return HGRD_GPU_ENOTSUP;
    }
    const uint64_t nBatches = (static_cast<uint64_t>(D.nThreads) + 31) / 32;
    const uint64_t blocks = std::min<uint64_t>((nBatches + 7) / 8, uint64_t(c->nSM) * 8);
    const uint64_t warps = blocks * 8;
    const uint64_t chunk = 64;
    uint64_t cap = std::max<uint64_t>(warps * chunk * 2 + (uint64_t(1) << 20), c->capHint);
    D2.chunk = static_cast<uint32_t>(chunk);
    NEED(c->keys, cap);
    NEED(c->vals, cap);
    D2.keys = c->keys.p;
    D2.vals = c->vals.p;
    D2.capacity = cap;
    CK(cudaMemsetAsync(c->ctr2.p, 0, sizeof(Counters), c->st));
    const size_t sm = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * P.sites.size() +
                      sizeof(ParamDev) * P.params.size();
    const void *jx = jk.get(hgrdgpu::jit::kExpandPar);
    // block prefixes of doubling length: every key's witness lies in the
    // earliest blocks reaching its element (later blocks' events come later
    // in the reference order), so k_inter_done usually stops this pass after
    // the first 1/64 of the launch
    const int nK = static_cast<int>(interKeys.size());
    NEED(c->doneKeys, 2 * static_cast<size_t>(std::max(nK, 1)));
    int *dDone = c->doneKeys.p;
    int *dKeys = dDone + std::max(nK, 1);
    NEED(c->doneTargets, static_cast<size_t>(std::max(nK, 1)));
    CK(cudaMemcpyAsync(dKeys, interKeys.data(), 4 * static_cast<size_t>(nK),
                       cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->doneTargets.p, interTarget.data(), 8 * static_cast<size_t>(nK),
                       cudaMemcpyHostToDevice, c->st));
    c->h2dBytes += 12 * static_cast<size_t>(nK);
    bool retry = false;
    Counters h2{};
    for (int64_t b0 = 0, b1 = std::max<int64_t>(1, D.nBlocks / 64); b0 < D.nBlocks;
         b0 = b1, b1 = std::min<int64_t>(D.nBlocks, 2 * b1)) {
      D2.threadBase = b0 * D.tpb;
      D2.threadEnd = b1 * D.tpb;
      rc = launchExpandPar(c, D2, static_cast<unsigned>(blocks), sm, jx,
                           jx ? "k_expand_par_shared[jit]" : "k_expand_par_shared");
      if (rc < 0)
        return rc;
      rc = readCountersFrom(c, c->ctr2.p);
      if (rc < 0)
        return rc;
      h2 = *c->hCtr;
      if (h2.flags & kFlagCapacity) {
        c->capHint = std::max<uint64_t>(c->capHint, h2.cursor + warps * chunk + 4096) * 2;
        retry = true;
        break;
      }
      if (h2.flags & kFlagPhase) {
        bP = std::max(bP, bitsFor(uint64_t(h2.maxBp) + 1));
        bQ = std::max(bQ, bitsFor(uint64_t(h2.maxWp) + 1));
        retry = true;
        break;
      }
      if (b1 < D.nBlocks && nK > 0) {
        {
          StageTimer t(c, "k_inter_done");
          k_inter_done<<<(nK + 7) / 8, 256, 0, c->st>>>(
              c->keys.p, c->vals.p, std::min<uint64_t>(h2.cursor, cap), D2.kl, D.tpb, D.ws,
              D.sites, D.confInter, nLocs, dKeys, c->doneTargets.p, nK, dDone);
        }
        CK(cudaGetLastError());
        ++c->kernelLaunches;
        std::vector<int> dn(static_cast<size_t>(nK));
        CK(cudaMemcpyAsync(dn.data(), dDone, 4 * static_cast<size_t>(nK), cudaMemcpyDeviceToHost,
                           c->st));
        c->d2hBytes += 4 * static_cast<size_t>(nK);
        CK(cudaStreamSynchronize(c->st));
        if (std::all_of(dn.begin(), dn.end(), [](int v) { return v != 0; }))
          break; // every INTER key's witness is in the records so far
      }
    }
    if (retry)
      continue;
    rc = detect(c, L, D2, o, std::min<uint64_t>(h2.cursor, cap), false, false, R, 1, true);
    return rc < 0 ? rc : 1;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// C ABI

namespace {

bool validLaunch(const hgrd_gpu_launch &L, std::string &why) {
  if (!L.code || L.n_code == 0) {
    why = "empty code";
    return false;
  }
  if (L.warp_size <= 0) {
    why = "warp size must be positive";
    return false;
  }
  for (int d = 0; d < 3; ++d)
    if (L.grid[d] <= 0 || L.block[d] <= 0) {
      why = "non-positive launch dimension";
      return false;
    }
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (I.op > HGRD_OP_JMP) {
      why = "bad opcode";
      return false;
    }
    if ((I.op == HGRD_OP_JZ || I.op == HGRD_OP_JMP) &&
        (I.imm < 0 || I.imm >= static_cast<int64_t>(L.n_code))) {
      why = "bad jump target";
      return false;
    }
    if ((I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC) &&
        (I.imm < 0 || I.imm >= static_cast<int64_t>(L.n_sites))) {
      why = "bad site";
      return false;
    }
    if (I.op != HGRD_OP_STEP && I.op != HGRD_OP_JMP && I.op != HGRD_OP_END &&
        (I.a >= L.n_regs || I.b >= std::max<uint32_t>(L.n_regs, 1) ||
         I.c >= std::max<uint32_t>(L.n_regs, 1)))
      if (I.op != HGRD_OP_SYNCTHREADS && I.op != HGRD_OP_SYNCWARP && I.op != HGRD_OP_FENCE) {
        why = "register out of range";
        return false;
      }
    if (I.op == HGRD_OP_BUILTIN && I.sub >= 12) {
      why = "bad builtin";
      return false;
    }
  }
  if (L.code[L.n_code - 1].op != HGRD_OP_END) {
    why = "code must end with END";
    return false;
  }
  for (uint32_t s = 0; s < L.n_sites; ++s)
    if (L.sites[s].loc < 0 || static_cast<uint32_t>(L.sites[s].loc) >= L.n_locs ||
        L.sites[s].param >= static_cast<int32_t>(L.n_params)) {
      why = "bad site table";
      return false;
    }
  return true;
}

int snapshot(hgrd_gpu_ctx *c, const Plan &P, bool restore) {
  size_t off = 0;
  for (int32_t h : P.wHandle) {
    if (h < 0)
      continue;
    const auto &b = c->bufs[static_cast<size_t>(h)];
    const size_t bytes = static_cast<size_t>(b.elems) * 8;
    if (!restore) {
      CK(cudaMemcpyAsync(c->snapshot.p + off, b.p, bytes, cudaMemcpyDeviceToDevice, c->st));
    } else {
      CK(cudaMemcpyAsync(b.p, c->snapshot.p + off, bytes, cudaMemcpyDeviceToDevice, c->st));
    }
    off += bytes;
  }
  return 0;
}

// Per-launch setup shared by the full and the sharded checks: plan (buffer
// bases, site flags, conflict masks), one blob upload, device descriptor.
int prepareLaunch(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, Plan &P, BlobOffsets &o,
                  LaunchDev &D) {
  planLaunch(c, L, P);
  htrace(c, "plan");
  int rc = uploadBlob(c, L, P, o);
  if (rc < 0)
    return rc;
  htrace(c, "upload");
  D = LaunchDev{};
  D.code = reinterpret_cast<const hgrd_gpu_insn *>(c->blob.p + o.code);
  D.sites = reinterpret_cast<const SiteDev *>(c->blob.p + o.sites);
  D.params = reinterpret_cast<const ParamDev *>(c->blob.p + o.params);
  D.regInit = reinterpret_cast<const int64_t *>(c->blob.p + o.regs);
  D.confInter = reinterpret_cast<const uint64_t *>(c->blob.p + o.cInter);
  D.confIntra = reinterpret_cast<const uint64_t *>(c->blob.p + o.cIntra);
  D.locMask = reinterpret_cast<const uint64_t *>(c->blob.p + o.locMask);
  D.nCode = static_cast<int>(L.n_code);
  D.nRegs = static_cast<int>(L.n_regs);
  D.nSites = static_cast<int>(L.n_sites);
  D.nParams = static_cast<int>(L.n_params);
  D.nLocs = static_cast<int>(L.n_locs);
  for (int d = 0; d < 3; ++d) {
    D.grid[d] = L.grid[d];
    D.block[d] = L.block[d];
  }
  D.ws = L.warp_size;
  D.tpb = L.block[0] * L.block[1] * L.block[2];
  D.nBlocks = L.grid[0] * L.grid[1] * L.grid[2];
  D.nThreads = D.nBlocks * D.tpb;
  D.stepBudget = L.step_budget;
  D.ctr = c->cur;
  D.small = D.nThreads < (int64_t(1) << 32) - 1 && L.warp_size < (int64_t(1) << 32);
  if (D.small) {
    D.dTpb = FastDiv::make(static_cast<uint32_t>(D.tpb));
    D.dBx = FastDiv::make(static_cast<uint32_t>(L.block[0]));
    D.dBxBy = FastDiv::make(static_cast<uint32_t>(L.block[0] * L.block[1]));
    D.dGx = FastDiv::make(static_cast<uint32_t>(L.grid[0]));
    D.dGxGy = FastDiv::make(static_cast<uint32_t>(L.grid[0] * L.grid[1]));
    D.dWs = FastDiv::make(static_cast<uint32_t>(std::min<int64_t>(L.warp_size, 0xffffffffLL)));
  }

  D.threadBase = 0;
  D.threadEnd = D.nThreads;
  return 0;
}

// Per-stage device times of the check just finished (profiling on; the
// stream is synchronised), as the JSON hgrd_gpu_last_profile returns.
void finishProfile(hgrd_gpu_ctx *c) {
  if (!c->profiling)
    return;
  std::string j = "[";
  for (size_t i = 0; i < c->stages.size(); ++i) {
    float sm = 0;
    cudaEventElapsedTime(&sm, c->stages[i].a, c->stages[i].b);
    char buf[128];
    std::snprintf(buf, sizeof buf, "%s{\"name\":\"%s\",\"ms\":%.6f}", i ? "," : "",
                  c->stages[i].name, sm);
    j += buf;
  }
  c->profileJson = j + "]";
}

int checkLaunch(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, hgrd_gpu_result *R) {
  if (c->hostTrace) {
    c->trace.clear();
    c->trace.emplace_back("start", std::chrono::steady_clock::now());
  }
  R->n_races = 0;
  R->n_traps = 0;
  R->n_traps_total = 0;
  R->steps = 0;
  R->instances = 0;
  R->records = 0;
  R->aborted = 0;
  R->abort_stmt = -1;
  R->mode = 0;
  R->device_ms = 0;
  c->stages.clear();
  c->evUsed = 0;
  c->racesOnHost = false;
  c->e1Done = false;
  if (c->timing)
    CK(cudaEventRecord(c->e0, c->st));

  Plan P;
  BlobOffsets o{};
  LaunchDev D{};
  int rc = prepareLaunch(c, L, P, o, D);
  if (rc < 0)
    return rc;

  int bP, bQ;
  bool bounded, loops;
  uint32_t accessInsns;
  phaseBounds(L, bP, bQ, bounded, accessInsns, loops);
  uint32_t recInsns = 0;
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if ((I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC) &&
        P.sites[static_cast<size_t>(I.imm)].record)
      ++recInsns;
  }
  const int bE = bitsFor(P.totalW + 1);
  const int bB = bitsFor(static_cast<uint64_t>(D.nBlocks));
  const int bW = bitsFor(static_cast<uint64_t>((D.tpb + D.ws - 1) / D.ws));
  const int bL = bitsFor(static_cast<uint64_t>(std::min<int64_t>(D.ws, D.tpb)));

  const bool locks = (L.flags & HGRD_LAUNCH_PAIRWISE) != 0;
  const bool pairwise = locks || !P.summaryOk;
  // Lock idioms in a PARALLEL launch: loop-free threads have a static op
  // count (fixed op slots per thread) and at most kLaneBuf records (kept in
  // program order), and the canonical sort key (element | thread | seq)
  // must fit 64 bits
  uint32_t opsPerThread = 0;
  for (uint32_t pc = 0; pc < L.n_code; ++pc)
    opsPerThread += L.code[pc].op == HGRD_OP_ATOMIC || L.code[pc].op == HGRD_OP_FENCE;
  const int canonBits = bitsFor(static_cast<uint64_t>(D.nThreads)) + bitsFor(L.n_code + 1);
  const bool parLocks = locks && !loops && recInsns <= static_cast<uint32_t>(kLaneBuf) &&
                        opsPerThread > 0 && bE + canonBits <= 64 &&
                        static_cast<uint64_t>(D.nThreads) * opsPerThread < (uint64_t(1) << 32);
  bool seq = (L.flags & HGRD_LAUNCH_SEQUENTIAL) || (pairwise && !parLocks) ||
             L.n_regs > kMaxRegs;
  // (the interpreter keeps at most kMaxRegs registers per lane)
  const size_t smem = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * P.sites.size() +
                      sizeof(ParamDev) * P.params.size();
  if (smem > 200 * 1024)
    seq = true;
  bool snapped = false;

  // (the fused kernel keeps per-key minimum elements as 32-bit values)
  const bool fusedOk = c->fusedEnabled && !seq && !locks && P.summaryOk && L.n_locs <= 32 &&
                       P.totalW < 0xFFFFFFFFull &&
                       o.nW <= kMaxWritten && D.nBlocks < (1 << 20) - 2 &&
                       !(L.flags & HGRD_LAUNCH_GENERAL);
  // NVRTC specialisation for large PARALLEL launches (compiled on first use)
  const bool useJit = c->jitMode == 2 || (c->jitMode == 1 && D.nThreads >= (int64_t(1) << 14));
  JitGetter jk{c, &L, useJit, {}, {}};
  for (uint32_t p = 0; p < L.n_params; ++p) {
    const ParamDev &d = P.params[p];
    jk.params.push_back(hgrdgpu::jit::JitParam{d.handle >= 0 ? d.size : 0, d.elemBase});
  }
  for (const auto &s : P.sites) // bit 0: record, bit 1: ownership exchange
    jk.rec.push_back(static_cast<uint8_t>((s.record ? 1 : 0) | (s.own ? 2 : 0)));
  markStream(L, P.params, jk); // bit 2: streamed load
  if (fusedOk && makeLayout(D.kl, bE, bB, bP, bW, bQ, bL, D.nSites)) {
    rc = runFused(c, L, D, o, P, R, recInsns, loops, jk);
    if (rc < 0)
      return rc;
    if (rc == 1)
      goto finish;
    if (c->fusedOrdered)
      seq = true; // (one round trip less than finding it again in k_expand_par)
  }

  for (int attempt = 0; attempt < 16; ++attempt) {
    if (!makeLayout(D.kl, bE, bB, bP, bW, bQ, bL, D.nSites)) {
      c->err = "packed record key wider than 64 bits";
      return HGRD_GPU_ENOTSUP;
    }
    CK(cudaMemsetAsync(c->cur, 0, sizeof(Counters), c->st));
    if (!seq) {
      const uint64_t nBatches = (static_cast<uint64_t>(D.nThreads) + 31) / 32;
      const uint64_t blocks = std::min<uint64_t>((nBatches + 7) / 8, uint64_t(c->nSM) * 8);
      const uint64_t warps = blocks * 8;
      const uint64_t expected = static_cast<uint64_t>(D.nThreads) * recInsns;
      uint64_t chunk = std::clamp<uint64_t>(expected / std::max<uint64_t>(warps, 1) / 4, 64, kChunk);
      uint64_t cap = expected + warps * chunk + 4096;
      if (loops)
        cap = std::max(cap, c->capHint);
      D.chunk = static_cast<uint32_t>(chunk);
      NEED(c->keys, cap);
      NEED(c->vals, cap);
      D.keys = c->keys.p;
      D.vals = c->vals.p;
      D.capacity = cap;
      D.opStart = nullptr;
      D.opStride = 0;
      if (parLocks) {
        const size_t nOps = static_cast<size_t>(D.nThreads) * opsPerThread;
        NEED(c->opIndex, nOps);
        NEED(c->opMeta, nOps);
        NEED(c->opSeq, nOps);
        D.opIndex = c->opIndex.p;
        D.opMeta = c->opMeta.p;
        D.opSeq = c->opSeq.p;
        D.opCap = nOps;
        D.opStride = opsPerThread;
      }
      const void *jx = jk.get(hgrdgpu::jit::kExpandPar);
      rc = launchExpandPar(c, D, static_cast<unsigned>(blocks), smem, jx,
                           jx ? "k_expand_par[jit]" : "k_expand_par");
      if (rc < 0)
        return rc;
      rc = readCounters(c);
      if (rc < 0)
        return rc;
      const Counters h = *c->hCtr;
      if ((h.flags & kFlagAbort) || static_cast<int64_t>(h.steps) > L.step_budget ||
          h.traps > 0) {
        seq = true; // traps / budget need the canonical order
        continue;
      }
      if (h.flags & kFlagCapacity) {
        c->capHint = std::max<uint64_t>(c->capHint, h.cursor + warps * chunk + 4096) * 2;
        continue;
      }
      if (h.flags & kFlagPhase) {
        bP = std::max(bP, bitsFor(uint64_t(h.maxBp) + 1));
        bQ = std::max(bQ, bitsFor(uint64_t(h.maxWp) + 1));
        continue;
      }
      if (h.flags & kFlagSeqSite) {
        c->err = "more than 2^" + std::to_string(D.kl.bS) + " accesses in one thread";
        return HGRD_GPU_ENOTSUP;
      }
      if (h.flags & kFlagOps) { // (cannot happen: static op count)
        seq = true;
        continue;
      }
      R->steps = static_cast<int64_t>(h.steps);
      R->instances = h.instances;
      R->records = h.records;
      R->mode = L.flags & ~HGRD_LAUNCH_SEQUENTIAL;
      rc = detect(c, L, D, o, std::min<uint64_t>(h.cursor, cap), parLocks, parLocks, R);
      if (rc < 0)
        return rc;
      break;
    }
    D.opStride = 0;
    // SEQUENTIAL: kernel loads and stores read and write every parameter buffer
    for (uint32_t p = 0; p < L.n_params; ++p)
      if (L.param_handle[p] >= 0 && static_cast<size_t>(L.param_handle[p]) < c->bufs.size() &&
          materialize(c, L.param_handle[p]) < 0)
        return HGRD_GPU_ECUDA;
    if (!snapped) {
      size_t bytes = 0;
      for (int32_t hnd : P.wHandle)
        if (hnd >= 0)
          bytes += static_cast<size_t>(c->bufs[static_cast<size_t>(hnd)].elems) * 8;
      NEED(c->snapshot, bytes);
      rc = snapshot(c, P, false);
      if (rc < 0)
        return rc;
      snapped = true;
    } else {
      rc = snapshot(c, P, true);
      if (rc < 0)
        return rc;
    }
    uint64_t cap = loops ? c->capHint : static_cast<uint64_t>(D.nThreads) * recInsns + 16;
    cap = std::max<uint64_t>(cap, 16);
    NEED(c->keys, cap);
    NEED(c->vals, cap);
    D.keys = c->keys.p;
    D.vals = c->vals.p;
    D.capacity = cap;
    D.chunk = 0;
    NEED(c->seqRegs, std::max<uint32_t>(L.n_regs, 1));
    D.seqRegs = c->seqRegs.p;
    NEED(c->traps, std::max<uint32_t>(R->trap_cap, 1));
    D.traps = c->traps.p;
    D.trapCap = R->trap_cap;
    if (locks) {
      NEED(c->opStart, static_cast<size_t>(D.nThreads) + 1);
      uint64_t ocap = std::max<uint64_t>(c->opHint, 16);
      if (!loops) { // loop-free: each sync-op instruction runs at most once per thread
        uint64_t perThread = 0;
        for (uint32_t pc = 0; pc < L.n_code; ++pc)
          perThread += L.code[pc].op == HGRD_OP_ATOMIC || L.code[pc].op == HGRD_OP_FENCE;
        ocap = std::max<uint64_t>(ocap, static_cast<uint64_t>(D.nThreads) * perThread + 16);
      }
      NEED(c->opIndex, ocap);
      NEED(c->opMeta, ocap);
      NEED(c->opSeq, ocap);
      D.opStart = c->opStart.p;
      D.opIndex = c->opIndex.p;
      D.opMeta = c->opMeta.p;
      D.opSeq = c->opSeq.p;
      D.opCap = ocap;
    } else {
      D.opStart = nullptr;
      D.opCap = 0;
    }
    {
      const size_t sh = static_cast<size_t>(D.nRegs) * sizeof(int64_t);
      const bool staged = sh <= kSeqSharedMax;
      if (staged && sh > 48 * 1024 && !c->seqSharedSet) {
        CK(cudaFuncSetAttribute(k_expand_seq<InterpBody>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSeqSharedMax)));
        c->seqSharedSet = true;
      }
      // an NVRTC body removes the interpreter's dispatch from the chain
      if (const void *jf = jk.get(hgrdgpu::jit::kExpandSeq)) {
        int noStage = 0;
        void *args[] = {&D, &noStage};
        StageTimer t(c, "k_expand_seq[jit]");
        CK(cudaLaunchKernel(jf, dim3(1), dim3(32), args, 0, c->st));
      } else {
        StageTimer t(c, "k_expand_seq");
        k_expand_seq<InterpBody><<<1, 32, staged ? sh : 0, c->st>>>(D, staged ? 1 : 0);
      }
    }
    CK(cudaGetLastError());
    ++c->kernelLaunches;
    rc = readCountersAndTraps(c, std::max<uint32_t>(R->trap_cap, 1));
    if (rc < 0)
      return rc;
    const Counters h = *c->hCtr;
    const uint32_t nt = static_cast<uint32_t>(std::min<uint64_t>(h.traps, R->trap_cap));
    if (!(h.flags & kFlagAbort)) {
      bool retry = false;
      if (h.flags & kFlagCapacity) {
        c->capHint = std::max<uint64_t>(c->capHint, h.cursor) * 2;
        retry = true;
      }
      if (h.flags & kFlagOps) {
        c->opHint = std::max<uint64_t>(c->opHint, h.nOps) * 2;
        retry = true;
      }
      if (h.flags & kFlagPhase) {
        bP = std::max(bP, bitsFor(uint64_t(h.maxBp) + 1));
        bQ = std::max(bQ, bitsFor(uint64_t(h.maxWp) + 1));
        retry = true;
      }
      if (retry)
        continue;
      if (h.flags & kFlagSeqSite) {
        c->err = "more than 2^" + std::to_string(D.kl.bS) + " accesses in one thread";
        return HGRD_GPU_ENOTSUP;
      }
    }
    if (nt) // (read with the counters)
      std::memcpy(R->traps, c->hTraps, sizeof(hgrd_gpu_trap) * nt);
    R->n_traps = nt;
    R->n_traps_total = h.traps;
    R->steps = static_cast<int64_t>(h.steps);
    R->instances = h.instances;
    R->records = h.records;
    R->mode = L.flags | HGRD_LAUNCH_SEQUENTIAL;
    if (h.flags & kFlagAbort) {
      R->aborted = 1;
      R->abort_stmt = h.abortStmt;
      break;
    }
    rc = detect(c, L, D, o, h.cursor, pairwise, locks, R);
    if (rc < 0)
      return rc;
    if (h.cursor <= 1) // no GPU work since the counters' synchronisation
      c->e1Done = c->e1AtSync;
    break;
  }
finish:
  float ms = 0;
  if (c->timing) {
    if (!c->e1Done) {
      CK(cudaEventRecord(c->e1, c->st));
      CK(cudaEventSynchronize(c->e1));
    }
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  } else {
    CK(cudaStreamSynchronize(c->st));
  }
  R->device_ms = ms;
  if (c->hostTrace) {
    htrace(c, "end");
    std::fprintf(stderr, "[hgrd host]");
    for (size_t i = 1; i < c->trace.size(); ++i)
      std::fprintf(stderr, " %s %.1f", c->trace[i].first,
                   std::chrono::duration<double, std::micro>(c->trace[i].second -
                                                             c->trace[i - 1].second)
                       .count());
    std::fprintf(stderr, " (us)\n");
  }
  finishProfile(c);
  return 0;
}


// ---------------------------------------------------------------------------
// Sharded single-launch check: each rank checks a whole-
// block range; INTRA kinds are rank-local, INTER-BLOCK needs the ranks'
// per-(element, site) block summaries combined (MIN/MAX all-reduce by the
// caller), then the witness records of the realised INTER keys' elements.

struct ShardSetup {
  Plan P;
  BlobOffsets o{};
  LaunchDev D{};
  uint32_t recInsns = 0;
  bool loops = false;
};

// Plan + key layout; HGRD_GPU_ENOTSUP (c->err says why) when the launch
// needs a path that does not shard (replicas then).
int shardPrepare(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, int64_t b0, int64_t b1,
                 ShardSetup &S) {
  int rc = prepareLaunch(c, L, S.P, S.o, S.D);
  if (rc < 0)
    return rc;
  LaunchDev &D = S.D;
  if (b0 < 0 || b1 < b0 || b1 > D.nBlocks) {
    c->err = "bad shard block range";
    return HGRD_GPU_EINVAL;
  }
  int bP, bQ;
  bool bounded;
  uint32_t accessInsns;
  phaseBounds(L, bP, bQ, bounded, accessInsns, S.loops);
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if ((I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC) &&
        S.P.sites[static_cast<size_t>(I.imm)].record)
      ++S.recInsns;
  }
  const size_t smem = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * S.P.sites.size() +
                      sizeof(ParamDev) * S.P.params.size();
  const char *why = nullptr;
  if (L.flags & (HGRD_LAUNCH_SEQUENTIAL | HGRD_LAUNCH_PAIRWISE | HGRD_LAUNCH_GENERAL))
    why = "sequential / lock-idiom launches are replicas only";
  else if (!S.P.summaryOk || L.n_locs > 32 || L.n_regs > kMaxRegs || smem > 200 * 1024)
    why = "launch outside the fused envelope";
  else if (S.P.totalW >= 0xFFFFFFFFull || S.o.nW > kMaxWritten || D.nBlocks >= (1 << 20) - 2)
    why = "written buffers / blocks outside the fused envelope";
  else if (!bounded)
    why = "barriers inside loops (phase bits not static)";
  const int bE = bitsFor(S.P.totalW + 1);
  const int bB = bitsFor(static_cast<uint64_t>(D.nBlocks));
  const int bW = bitsFor(static_cast<uint64_t>((D.tpb + D.ws - 1) / D.ws));
  const int bL = bitsFor(static_cast<uint64_t>(std::min<int64_t>(D.ws, D.tpb)));
  if (!why && !makeLayout(D.kl, bE, bB, bP, bW, bQ, bL, D.nSites))
    why = "packed record key wider than 64 bits";
  if (why) {
    c->err = std::string("not shardable: ") + why;
    return HGRD_GPU_ENOTSUP;
  }
  return 0;
}

JitGetter shardJit(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const ShardSetup &S) {
  const bool useJit =
      c->jitMode == 2 || (c->jitMode == 1 && S.D.nThreads >= (int64_t(1) << 14));
  JitGetter jk{c, &L, useJit, {}, {}};
  for (uint32_t p = 0; p < L.n_params; ++p) {
    const ParamDev &d = S.P.params[p];
    jk.params.push_back(hgrdgpu::jit::JitParam{d.handle >= 0 ? d.size : 0, d.elemBase});
  }
  for (const auto &s : S.P.sites)
    jk.rec.push_back(static_cast<uint8_t>((s.record ? 1 : 0) | (s.own ? 2 : 0)));
  markStream(L, S.P.params, jk);
  return jk;
}

void resetResult(hgrd_gpu_result *R) {
  R->n_races = 0;
  R->n_traps = 0;
  R->n_traps_total = 0;
  R->steps = 0;
  R->instances = 0;
  R->records = 0;
  R->aborted = 0;
  R->abort_stmt = -1;
  R->mode = 0;
  R->device_ms = 0;
}

int shardCheck(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, hgrd_gpu_shard *Sh,
               hgrd_gpu_result *R) {
  resetResult(R);
  Sh->inter_lo = Sh->inter_hi = nullptr;
  Sh->inter_n = 0;
  c->stages.clear();
  c->evUsed = 0;
  c->racesOnHost = false;
  if (c->timing)
    CK(cudaEventRecord(c->e0, c->st));
  ShardSetup S;
  int rc = shardPrepare(c, L, Sh->block_begin, Sh->block_end, S);
  if (rc < 0)
    return rc;
  JitGetter jk = shardJit(c, L, S);
  bool anyOwn = false;
  for (const auto &s : S.P.sites)
    anyOwn |= s.record && s.own;
  const uint64_t nTab = S.P.totalW * static_cast<uint64_t>(L.n_sites);
  if (anyOwn) { // the shard's INTER summary tables, filled by k_fused's records
    NEED(c->shardLo, nTab);
    NEED(c->shardHi, nTab);
    CK(cudaMemsetAsync(c->shardLo.p, 0x7f, nTab * sizeof(uint32_t), c->st)); // kShardEmpty
    CK(cudaMemsetAsync(c->shardHi.p, 0, nTab * sizeof(uint32_t), c->st));
  }
  rc = runFused(c, L, S.D, S.o, S.P, R, S.recInsns, S.loops, jk, Sh->block_begin,
                Sh->block_end, true, anyOwn ? c->shardLo.p : nullptr,
                anyOwn ? c->shardHi.p : nullptr);
  if (rc < 0)
    return rc;
  if (rc == 0) { // traps, step budget, overflow: the canonical order is needed
    c->err = "shard needs the ordered path (traps / step budget / capacity)";
    return HGRD_GPU_ENOTSUP;
  }
  if (anyOwn && !c->fusedShardTables) { // INTER summary of this shard's blocks (separate pass)
    const uint64_t n = nTab;
    NEED(c->ctr2, 1);
    CK(cudaMemsetAsync(c->ctr2.p, 0, sizeof(Counters), c->st));
    LaunchDev Ds = S.D;
    Ds.ctr = c->ctr2.p;
    Ds.interLo = c->shardLo.p;
    Ds.interHi = c->shardHi.p;
    Ds.nSitesTab = static_cast<int>(L.n_sites);
    Ds.keys = nullptr;
    Ds.vals = nullptr;
    Ds.capacity = 0;
    Ds.chunk = 64;
    Ds.threadBase = Sh->block_begin * S.D.tpb;
    Ds.threadEnd = Sh->block_end * S.D.tpb;
    const size_t sm = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * S.P.sites.size() +
                      sizeof(ParamDev) * S.P.params.size();
    const uint64_t nt = static_cast<uint64_t>(std::max<int64_t>(Ds.threadEnd - Ds.threadBase, 1));
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(((nt + 31) / 32 + 7) / 8, uint64_t(c->nSM) * 8));
    const void *jx = jk.get(hgrdgpu::jit::kExpandPar);
    rc = launchExpandPar(c, Ds, grid, sm, jx, jx ? "k_expand_par_shard[jit]" : "k_expand_par_shard");
    if (rc < 0)
      return rc;
    CK(cudaStreamSynchronize(c->st));
  }
  if (anyOwn) {
    Sh->inter_lo = c->shardLo.p;
    Sh->inter_hi = c->shardHi.p;
    Sh->inter_n = nTab;
  }
  float ms = 0;
  if (c->timing) {
    CK(cudaEventRecord(c->e1, c->st));
    CK(cudaEventSynchronize(c->e1));
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  } else {
    CK(cudaStreamSynchronize(c->st));
  }
  R->device_ms = ms;
  finishProfile(c);
  return 0;
}

// INTER keys of one element range of the (reduced) summary tables: per key
// its minimum element in [e0, e0 + nE) into keyElem (host, ~0: none).
int shardInterScan(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const uint32_t *lo,
                   const uint32_t *hi, uint64_t e0, uint64_t nE, uint64_t *keyElem,
                   uint32_t nKeysCap) {
  ShardSetup S;
  int rc = shardPrepare(c, L, 0, 0, S);
  if (rc < 0)
    return rc;
  const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  const int nKeys = 3 * nLocs * nLocs;
  if (nKeysCap < static_cast<uint32_t>(nKeys)) {
    c->err = "key table too small";
    return HGRD_GPU_E2BIG;
  }
  if (e0 + nE > S.P.totalW) {
    c->err = "element range outside the launch's written buffers";
    return HGRD_GPU_EINVAL;
  }
  NEED(c->interKeyElem, static_cast<size_t>(nKeys));
  CK(cudaMemsetAsync(c->interKeyElem.p, 0xff, 8 * static_cast<size_t>(nKeys), c->st));
  if (nE) {
    StageTimer t(c, "k_inter_scan_minmax");
    k_inter_scan_minmax<<<static_cast<unsigned>((nE + 255) / 256), 256, 0, c->st>>>(
        lo, hi, nE, e0, static_cast<int>(L.n_sites), S.D.sites, S.D.confInter, nLocs,
        c->interKeyElem.p);
    CK(cudaGetLastError());
    ++c->kernelLaunches;
  }
  CK(cudaMemcpyAsync(keyElem, c->interKeyElem.p, 8 * static_cast<size_t>(nKeys),
                     cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += 8 * static_cast<size_t>(nKeys);
  CK(cudaStreamSynchronize(c->st));
  return 0;
}

// This shard's packed records of the realised INTER keys' first-found
// elements (keyElem: the ranks' per-key minima, MIN-reduced).
int shardInterRecords(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const hgrd_gpu_shard *Sh,
                      const uint64_t *keyElem, uint32_t nKeysIn, uint64_t *keys, uint32_t *vals,
                      uint64_t cap, uint64_t *nOut) {
  *nOut = 0;
  ShardSetup S;
  int rc = shardPrepare(c, L, Sh->block_begin, Sh->block_end, S);
  if (rc < 0)
    return rc;
  const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
  const int nKeys = 3 * nLocs * nLocs;
  if (nKeysIn < static_cast<uint32_t>(nKeys)) {
    c->err = "key table too small";
    return HGRD_GPU_EINVAL;
  }
  std::vector<uint64_t> targets;
  for (int K = 0; K < nKeys; K += 3)
    if (keyElem[K] != ~0ull)
      targets.push_back(keyElem[K]);
  std::sort(targets.begin(), targets.end());
  targets.erase(std::unique(targets.begin(), targets.end()), targets.end());
  if (targets.empty())
    return 0;
  NEED(c->targets, targets.size());
  CK(cudaMemcpy(c->targets.p, targets.data(), 8 * targets.size(), cudaMemcpyHostToDevice));
  c->h2dBytes += 8 * targets.size();
  JitGetter jk = shardJit(c, L, S);
  LaunchDev D2 = S.D;
  NEED(c->ctr2, 1);
  D2.ctr = c->ctr2.p;
  D2.targets = c->targets.p;
  D2.nTargets = static_cast<int>(targets.size());
  D2.threadBase = Sh->block_begin * S.D.tpb;
  D2.threadEnd = Sh->block_end * S.D.tpb;
  const uint64_t nt = static_cast<uint64_t>(std::max<int64_t>(D2.threadEnd - D2.threadBase, 1));
  const uint64_t blocks = std::min<uint64_t>(((nt + 31) / 32 + 7) / 8, uint64_t(c->nSM) * 8);
  const uint64_t warps = blocks * 8, chunk = 64;
  const size_t sm = sizeof(hgrd_gpu_insn) * L.n_code + sizeof(SiteDev) * S.P.sites.size() +
                    sizeof(ParamDev) * S.P.params.size();
  for (int attempt = 0; attempt < 8; ++attempt) {
    const uint64_t dcap = std::max<uint64_t>(warps * chunk * 2 + (uint64_t(1) << 16), c->capHint);
    NEED(c->keys, dcap);
    NEED(c->vals, dcap);
    D2.keys = c->keys.p;
    D2.vals = c->vals.p;
    D2.capacity = dcap;
    D2.chunk = static_cast<uint32_t>(chunk);
    CK(cudaMemsetAsync(c->ctr2.p, 0, sizeof(Counters), c->st));
    const void *jx = jk.get(hgrdgpu::jit::kExpandPar);
    rc = launchExpandPar(c, D2, static_cast<unsigned>(blocks), sm, jx,
                         jx ? "k_expand_par_shard_targets[jit]" : "k_expand_par_shard_targets");
    if (rc < 0)
      return rc;
    rc = readCountersFrom(c, c->ctr2.p);
    if (rc < 0)
      return rc;
    const Counters h = *c->hCtr;
    if (h.flags & kFlagCapacity) {
      c->capHint = std::max<uint64_t>(c->capHint, h.cursor + warps * chunk + 4096) * 2;
      continue;
    }
    if (h.flags & (kFlagPhase | kFlagSeqSite)) {
      c->err = "shard records outside the static key layout";
      return HGRD_GPU_ENOTSUP;
    }
    const uint64_t n = std::min<uint64_t>(h.cursor, dcap);
    std::vector<uint64_t> hk(n);
    std::vector<uint32_t> hv(n);
    if (n) {
      CK(cudaMemcpyAsync(hk.data(), c->keys.p, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hv.data(), c->vals.p, 4 * n, cudaMemcpyDeviceToHost, c->st));
      c->d2hBytes += 12 * n;
      CK(cudaStreamSynchronize(c->st));
    }
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i) {
      if (hk[i] == S.D.kl.sentinel)
        continue; // chunk padding
      if (m >= cap) {
        *nOut = m + 1;
        return HGRD_GPU_E2BIG;
      }
      keys[m] = hk[i];
      vals[m] = hv[i];
      ++m;
    }
    *nOut = m;
    return 0;
  }
  c->err = "shard target records exceed capacity";
  return HGRD_GPU_ENOTSUP;
}


// All-reduce variant: the caller reduced the whole tables in place.
int shardInter(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const hgrd_gpu_shard *Sh,
               uint64_t *keys, uint32_t *vals, uint64_t cap, uint64_t *nOut) {
  *nOut = 0;
  ShardSetup S;
  int rc = shardPrepare(c, L, Sh->block_begin, Sh->block_end, S);
  if (rc < 0)
    return rc;
  const uint64_t nTab = S.P.totalW * static_cast<uint64_t>(L.n_sites);
  if (Sh->inter_n == 0)
    return 0; // no buffer reachable from two blocks
  if (Sh->inter_n != nTab || c->shardLo.cap < nTab) {
    c->err = "shard INTER tables do not match the launch";
    return HGRD_GPU_EINVAL;
  }
  const uint32_t nKeys = 3 * std::max<uint32_t>(L.n_locs, 1) * std::max<uint32_t>(L.n_locs, 1);
  std::vector<uint64_t> ke(nKeys);
  rc = shardInterScan(c, L, c->shardLo.p, c->shardHi.p, 0, S.P.totalW, ke.data(), nKeys);
  if (rc < 0)
    return rc;
  return shardInterRecords(c, L, Sh, ke.data(), nKeys, keys, vals, cap, nOut);
}

int shardDetect(hgrd_gpu_ctx *c, const hgrd_gpu_launch &L, const uint64_t *keys,
                const uint32_t *vals, uint64_t n, hgrd_gpu_result *R) {
  resetResult(R);
  c->racesOnHost = false;
  ShardSetup S;
  int rc = shardPrepare(c, L, 0, 0, S);
  if (rc < 0)
    return rc;
  const uint64_t cap = std::max<uint64_t>(n, 1);
  NEED(c->keys, cap);
  NEED(c->vals, cap);
  if (n) {
    CK(cudaMemcpyAsync(c->keys.p, keys, 8 * n, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->vals.p, vals, 4 * n, cudaMemcpyHostToDevice, c->st));
    c->h2dBytes += 12 * n;
  }
  return detect(c, L, S.D, S.o, n, false, false, R, /*kindMask=*/1);
}

// ---------------------------------------------------------------------------
// Batched check of many small launches (batch.cuh): one H2D of every
// descriptor, one k_batch launch, one D2H of every launch's counters and
// races.

struct BatchPlan {
  bool ok = false;
  uint32_t R = 0;
  std::vector<ParamDev> params;
  std::vector<SiteDev> sites;
  std::vector<uint64_t> confInter, confIntra, wBase;
  std::vector<int32_t> wHandle;
  std::vector<char> needData; // per buffer: a value-needed load reads it
  uint64_t totalW = 0;
};

void planBatchLaunch(const hgrd_gpu_batch_launch &B, BatchPlan &P) {
  // (P may hold an earlier batch's plan: reused storage, no allocations)
  P.ok = false;
  P.R = 0;
  P.totalW = 0;
  P.wBase.clear();
  P.wHandle.clear();
  const hgrd_gpu_launch &L = B.launch;
  std::string why;
  if (!validLaunch(L, why))
    return;
  if (L.flags & (HGRD_LAUNCH_SEQUENTIAL | HGRD_LAUNCH_PAIRWISE | HGRD_LAUNCH_GENERAL))
    return;
  const int64_t tpb = L.block[0] * L.block[1] * L.block[2];
  const int64_t nBlocks = L.grid[0] * L.grid[1] * L.grid[2];
  if (L.n_regs > static_cast<uint32_t>(kMaxRegs) || L.n_sites > static_cast<uint32_t>(kMaxSites) ||
      L.n_locs > 32 || nBlocks > kBatchMaxBlocks || tpb > kBatchMaxThreads ||
      nBlocks * tpb > kBatchMaxThreads || L.warp_size >= (int64_t(1) << 31))
    return;
  const uint32_t nb = B.n_buffers;
  auto bufOf = [&](int32_t param) -> int32_t {
    if (param < 0 || static_cast<uint32_t>(param) >= L.n_params)
      return -1;
    const int32_t h = L.param_handle[param];
    return (h >= 0 && static_cast<uint32_t>(h) < nb) ? h : -1;
  };
  static thread_local std::vector<char> written; // (per-thread scratch, no allocations)
  static thread_local std::vector<uint64_t> base;
  static thread_local std::vector<int> windex;
  written.assign(nb, 0);
  base.assign(nb, 0);
  windex.assign(nb, 0);
  for (uint32_t s = 0; s < L.n_sites; ++s)
    if (L.sites[s].kind != HGRD_SITE_LOAD && bufOf(L.sites[s].param) >= 0)
      written[static_cast<size_t>(bufOf(L.sites[s].param))] = 1;
  for (uint32_t h = 0; h < nb; ++h)
    if (written[h]) {
      windex[h] = static_cast<int>(P.wBase.size()) + 1;
      base[h] = P.totalW;
      P.wBase.push_back(P.totalW);
      P.wHandle.push_back(static_cast<int32_t>(h));
      P.totalW += static_cast<uint64_t>(std::max<int64_t>(B.buffer_elems[h], 0));
    }
  if (P.wBase.empty()) {
    P.wBase.push_back(0);
    P.wHandle.push_back(-1);
  }
  if (P.totalW >= 0xFFFFFFFFull || P.wBase.size() > static_cast<size_t>(kMaxWritten))
    return;
  P.needData.assign(nb, 0);
  uint32_t recInsns = 0;
  bool loops = false;
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (I.op == HGRD_OP_LOAD && (I.sub & 1)) {
      const int32_t h = bufOf(L.sites[static_cast<size_t>(I.imm)].param);
      if (h >= 0)
        P.needData[static_cast<size_t>(h)] = 1;
    }
    if ((I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC) &&
        bufOf(L.sites[static_cast<size_t>(I.imm)].param) >= 0 &&
        written[static_cast<size_t>(bufOf(L.sites[static_cast<size_t>(I.imm)].param))])
      ++recInsns;
    if (I.op == HGRD_OP_JMP && I.imm <= static_cast<int64_t>(pc))
      loops = true;
  }
  P.R = loops ? 0 : recInsns;
  if (!loops && static_cast<uint64_t>(nBlocks * tpb) * recInsns > BatchSmem::kCap)
    return;
  P.params.resize(std::max<uint32_t>(L.n_params, 1));
  for (uint32_t p = 0; p < L.n_params; ++p) {
    ParamDev d{};
    const int32_t h = bufOf(static_cast<int32_t>(p));
    d.handle = h;
    if (h >= 0) {
      d.size = B.buffer_elems[h];
      d.written = windex[static_cast<size_t>(h)];
      d.elemBase = base[static_cast<size_t>(h)];
    }
    P.params[p] = d;
  }
  P.sites.resize(std::max<uint32_t>(L.n_sites, 1));
  for (uint32_t s = 0; s < L.n_sites; ++s) {
    SiteDev d{};
    d.param = L.sites[s].param;
    d.loc = L.sites[s].loc;
    d.kind = L.sites[s].kind;
    d.aop = L.sites[s].atomic_op;
    d.scope = L.sites[s].scope;
    const int32_t h = bufOf(d.param);
    d.record = (h >= 0 && written[static_cast<size_t>(h)]) ? 1 : 0;
    P.sites[s] = d;
  }
  P.confInter.assign(P.sites.size(), 0);
  P.confIntra.assign(P.sites.size(), 0);
  for (uint32_t a = 0; a < L.n_sites; ++a) // reference :752-758, as planLaunch
    for (uint32_t b = 0; b < L.n_sites; ++b) {
      const auto &X = L.sites[a];
      const auto &Y = L.sites[b];
      const bool write = X.kind != HGRD_SITE_LOAD || Y.kind != HGRD_SITE_LOAD;
      const bool bothAtomic = X.kind == HGRD_SITE_ATOMIC && Y.kind == HGRD_SITE_ATOMIC;
      const bool devBoth = X.scope == HGRD_SCOPE_DEVICE && Y.scope == HGRD_SCOPE_DEVICE;
      const bool blkBoth = X.scope != HGRD_SCOPE_NONE && Y.scope != HGRD_SCOPE_NONE;
      if (write && !(bothAtomic && devBoth))
        P.confInter[a] |= 1ull << b;
      if (write && !(bothAtomic && blkBoth))
        P.confIntra[a] |= 1ull << b;
    }
  P.ok = true;
}

template <class T> size_t batchPut(std::vector<unsigned char> &blob, const T *src, size_t n) {
  const size_t at = align16(blob.size());
  blob.resize(at + sizeof(T) * n);
  if (n)
    std::memcpy(blob.data() + at, src, sizeof(T) * n);
  return at;
}

int checkBatch(hgrd_gpu_ctx *c, const hgrd_gpu_batch_launch *BL, uint32_t n,
               hgrd_gpu_result *R) {
  // development: HGRD_SWEEP_TRACE=1 prints the batch's size and phase times
  static const bool trace = std::getenv("HGRD_SWEEP_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t i = 0; i < n; ++i) {
    resetResult(&R[i]);
    R[i].mode = HGRD_RESULT_UNCHECKED;
  }
  // 1. per-launch plans, on host threads (storage kept across batches of
  //    this host thread: a sweep's batches allocate nothing after the first)
  static thread_local std::vector<BatchPlan> tlPlans;
  std::vector<BatchPlan> &plans = tlPlans; // (the caller's: lambdas on other threads use it)
  if (plans.size() < n)
    plans.resize(n);
  hgrdgpu::parallelFor(n, [&](size_t i) { planBatchLaunch(BL[i], plans[i]); });
  std::vector<uint32_t> idx; // batch entry -> launch
  for (uint32_t i = 0; i < n; ++i)
    if (plans[i].ok)
      idx.push_back(i);
  const uint32_t m = static_cast<uint32_t>(idx.size());
  if (m == 0)
    return 0;
  // 2. layout of the blob: [BatchLaunch x m] | per launch: code (shared by
  //    launches of one kernel), sites, params, regs, masks, wBase, the
  //    contents of value-needed buffers | work counter, trap cursor
  struct Fix {
    size_t code, sites, params, regs, cInter, cIntra, wBase, data;
    bool codeOwner;
  };
  std::vector<Fix> fix(m);
  std::unordered_map<const hgrd_gpu_insn *, size_t> codeAt;
  size_t off = align16(sizeof(BatchLaunch) * m);
  auto put = [&](size_t bytes) {
    const size_t at = off;
    off = align16(off + bytes);
    return at;
  };
  int maxKeys = 3, maxCode = 1, maxSites = 1, maxParams = 1, maxW = 1;
  std::vector<uint32_t> raceOffs(m);
  uint32_t raceOff = 0;
  for (uint32_t k = 0; k < m; ++k) {
    const hgrd_gpu_batch_launch &B = BL[idx[k]];
    const hgrd_gpu_launch &L = B.launch;
    const BatchPlan &P = plans[idx[k]];
    Fix &f = fix[k];
    auto ci = codeAt.find(L.code);
    f.codeOwner = ci == codeAt.end();
    if (f.codeOwner)
      ci = codeAt.emplace(L.code, put(sizeof(hgrd_gpu_insn) * L.n_code)).first;
    f.code = ci->second;
    f.sites = put(sizeof(SiteDev) * P.sites.size());
    f.params = put(sizeof(ParamDev) * P.params.size());
    f.regs = put(8 * std::max<size_t>(L.n_regs, 1));
    f.cInter = put(8 * P.confInter.size());
    f.cIntra = put(8 * P.confIntra.size());
    f.wBase = put(8 * P.wBase.size());
    f.data = off;
    for (uint32_t h = 0; h < B.n_buffers; ++h)
      if (P.needData[h] && B.buffer_elems[h] > 0)
        put(8 * static_cast<size_t>(B.buffer_elems[h]));
    const int nLocs = static_cast<int>(std::max<uint32_t>(L.n_locs, 1));
    raceOffs[k] = raceOff;
    raceOff += static_cast<uint32_t>(3 * nLocs * nLocs);
    maxKeys = std::max(maxKeys, 3 * nLocs * nLocs);
    maxCode = std::max(maxCode, static_cast<int>(L.n_code));
    maxSites = std::max(maxSites, std::max(static_cast<int>(L.n_sites), 1));
    maxParams = std::max(maxParams, std::max(static_cast<int>(L.n_params), 1));
    maxW = std::max(maxW, static_cast<int>(P.wBase.size()));
  }
  const size_t nextAt = put(16); // work counter, trap cursor
  const size_t h2d = off;
  const size_t outAt = align16(h2d);
  const size_t racesAt = align16(outAt + sizeof(BatchOut) * m);
  const size_t total = racesAt + sizeof(hgrd_gpu_race) * std::max<uint32_t>(raceOff, 1);
  // trap area: every trap of the batch's launches (12 B each), read back only
  // when the trap cursor is non-zero
  const unsigned trapCap = static_cast<unsigned>(std::min<uint64_t>(uint64_t(m) * 256, 1u << 22));
  const size_t trapKeyAt = align16(total);
  const size_t trapSiteAt = align16(trapKeyAt + 8 * static_cast<size_t>(trapCap));
  const size_t devTotal = trapSiteAt + 4 * static_cast<size_t>(trapCap);
  NEED(c->batchBlob, devTotal);
  unsigned char *dev = c->batchBlob.p;
  if (c->hBatchCap < std::max(h2d, total - outAt)) {
    if (c->hBatch)
      CK(cudaFreeHost(c->hBatch));
    c->hBatch = nullptr;
    c->hBatchCap = std::max(std::max(h2d, total - outAt), size_t(1) << 20);
    CK(cudaMallocHost(&c->hBatch, c->hBatchCap));
  }
  // 3. fill the pinned staging buffer (device addresses fixed up), on host threads
  unsigned char *h = c->hBatch;
  std::memset(h + nextAt, 0, 16);
  hgrdgpu::parallelFor(m, [&](size_t k) {
    const hgrd_gpu_batch_launch &B = BL[idx[k]];
    const hgrd_gpu_launch &L = B.launch;
    BatchPlan &P = plans[idx[k]];
    const Fix &f = fix[k];
    if (f.codeOwner)
      std::memcpy(h + f.code, L.code, sizeof(hgrd_gpu_insn) * L.n_code);
    std::memcpy(h + f.sites, P.sites.data(), sizeof(SiteDev) * P.sites.size());
    int64_t *regs = reinterpret_cast<int64_t *>(h + f.regs);
    regs[0] = 0;
    if (L.n_regs)
      std::memcpy(regs, L.reg_init, 8 * L.n_regs);
    std::memcpy(h + f.cInter, P.confInter.data(), 8 * P.confInter.size());
    std::memcpy(h + f.cIntra, P.confIntra.data(), 8 * P.confIntra.size());
    std::memcpy(h + f.wBase, P.wBase.data(), 8 * P.wBase.size());
    // value-needed buffers: their launch-entry contents (zeros when absent)
    size_t at = f.data;
    for (uint32_t b = 0; b < B.n_buffers; ++b) {
      if (!P.needData[b] || B.buffer_elems[b] <= 0)
        continue;
      const size_t bytes = 8 * static_cast<size_t>(B.buffer_elems[b]);
      if (B.buffer_data && B.buffer_data[b])
        std::memcpy(h + at, B.buffer_data[b], bytes);
      else
        std::memset(h + at, 0, bytes);
      for (uint32_t p = 0; p < L.n_params; ++p)
        if (P.params[p].handle == static_cast<int32_t>(b))
          P.params[p].ptr = reinterpret_cast<int64_t *>(dev + at);
      at = align16(at + bytes);
    }
    std::memcpy(h + f.params, P.params.data(), sizeof(ParamDev) * P.params.size());
    BatchLaunch bl{};
    LaunchDev &D = bl.L;
    D.code = reinterpret_cast<const hgrd_gpu_insn *>(dev + f.code);
    D.sites = reinterpret_cast<const SiteDev *>(dev + f.sites);
    D.params = reinterpret_cast<const ParamDev *>(dev + f.params);
    D.regInit = reinterpret_cast<const int64_t *>(dev + f.regs);
    D.confInter = reinterpret_cast<const uint64_t *>(dev + f.cInter);
    D.confIntra = reinterpret_cast<const uint64_t *>(dev + f.cIntra);
    D.nCode = static_cast<int>(L.n_code);
    D.nRegs = static_cast<int>(L.n_regs);
    D.nSites = static_cast<int>(L.n_sites);
    D.nParams = static_cast<int>(L.n_params);
    D.nLocs = static_cast<int>(L.n_locs);
    for (int d = 0; d < 3; ++d) {
      D.grid[d] = L.grid[d];
      D.block[d] = L.block[d];
    }
    D.ws = L.warp_size;
    D.tpb = L.block[0] * L.block[1] * L.block[2];
    D.nBlocks = L.grid[0] * L.grid[1] * L.grid[2];
    D.nThreads = D.nBlocks * D.tpb;
    D.stepBudget = L.step_budget;
    D.small = true;
    D.dTpb = FastDiv::make(static_cast<uint32_t>(D.tpb));
    D.dBx = FastDiv::make(static_cast<uint32_t>(L.block[0]));
    D.dBxBy = FastDiv::make(static_cast<uint32_t>(L.block[0] * L.block[1]));
    D.dGx = FastDiv::make(static_cast<uint32_t>(L.grid[0]));
    D.dGxGy = FastDiv::make(static_cast<uint32_t>(L.grid[0] * L.grid[1]));
    D.dWs = FastDiv::make(static_cast<uint32_t>(L.warp_size));
    D.threadEnd = D.nThreads;
    bl.wBase = reinterpret_cast<const uint64_t *>(dev + f.wBase);
    bl.nW = static_cast<int32_t>(P.wBase.size());
    bl.nLocs = static_cast<int32_t>(std::max<uint32_t>(L.n_locs, 1));
    bl.R = P.R;
    bl.raceOff = raceOffs[k];
    std::memcpy(h + sizeof(BatchLaunch) * k, &bl, sizeof(BatchLaunch));
  });
  const auto t1 = std::chrono::steady_clock::now();
  CK(cudaMemcpyAsync(dev, h, h2d, cudaMemcpyHostToDevice, c->st));
  c->h2dBytes += h2d;

  const int keysPad = (maxKeys + 3) & ~3;
  const size_t smem = align16(sizeof(BatchSmem)) + 8 * static_cast<size_t>(keysPad) +
                      sizeof(hgrd_gpu_insn) * maxCode + sizeof(SiteDev) * maxSites +
                      sizeof(ParamDev) * maxParams + 16 * static_cast<size_t>(maxSites) +
                      8 * static_cast<size_t>(maxW) + 64;
  if (smem > 200 * 1024) {
    c->err = "batch launches too large for shared memory";
    return HGRD_GPU_ENOTSUP;
  }
  const void *fn = reinterpret_cast<const void *>(k_batch);
  if (c->smemOptIn.insert(fn).second) {
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            227 * 1024 - static_cast<int>(fa.sharedSizeBytes)));
  }
  int &perSM = c->occupancy[std::make_pair(fn, smem)];
  if (perSM == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSM, fn, kBatchThreads, smem));
    perSM = std::max(perSM, 1);
  }
  BatchArgs A{};
  A.launches = reinterpret_cast<const BatchLaunch *>(dev);
  A.n = m;
  A.out = reinterpret_cast<BatchOut *>(dev + outAt);
  A.races = reinterpret_cast<hgrd_gpu_race *>(dev + racesAt);
  A.next = reinterpret_cast<unsigned *>(dev + nextAt);
  A.trapCursor = reinterpret_cast<unsigned *>(dev + nextAt + 4);
  A.trapKey = reinterpret_cast<uint64_t *>(dev + trapKeyAt);
  A.trapSite = reinterpret_cast<uint32_t *>(dev + trapSiteAt);
  A.trapCap = trapCap;
  A.maxKeys = maxKeys;
  A.maxCode = maxCode;
  A.maxSites = maxSites;
  A.maxParams = maxParams;
  A.maxW = maxW;
  const unsigned grid =
      static_cast<unsigned>(std::min<int64_t>(m, static_cast<int64_t>(c->nSM) * perSM));
  {
    StageTimer t(c, "k_batch");
    void *args[] = {&A};
    CK(cudaLaunchKernel(fn, dim3(grid), dim3(kBatchThreads), args, smem, c->st));
  }
  CK(cudaGetLastError());
  ++c->kernelLaunches;
  const size_t d2h = total - outAt;
  CK(cudaMemcpyAsync(c->hBatch, dev + outAt, d2h, cudaMemcpyDeviceToHost, c->st));
  unsigned nTrapsAll = 0;
  CK(cudaMemcpyAsync(&nTrapsAll, dev + nextAt + 4, 4, cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += d2h + 4;
  CK(cudaStreamSynchronize(c->st));
  const auto t2 = std::chrono::steady_clock::now();
  std::vector<uint64_t> trapKey;
  std::vector<uint32_t> trapSite;
  nTrapsAll = std::min(nTrapsAll, trapCap);
  if (nTrapsAll) { // second round trip only when some launch trapped
    trapKey.resize(nTrapsAll);
    trapSite.resize(nTrapsAll);
    CK(cudaMemcpyAsync(trapKey.data(), dev + trapKeyAt, 8 * static_cast<size_t>(nTrapsAll),
                       cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(trapSite.data(), dev + trapSiteAt, 4 * static_cast<size_t>(nTrapsAll),
                       cudaMemcpyDeviceToHost, c->st));
    c->d2hBytes += 12 * static_cast<size_t>(nTrapsAll);
    CK(cudaStreamSynchronize(c->st));
  }
  const BatchOut *out = reinterpret_cast<const BatchOut *>(c->hBatch);
  const hgrd_gpu_race *races = reinterpret_cast<const hgrd_gpu_race *>(c->hBatch + (racesAt - outAt));
  for (uint32_t k = 0; k < m; ++k) {
    const BatchOut &o = out[k];
    hgrd_gpu_result &r = R[idx[k]];
    if (o.flags & (kFlagFusedOverflow | kFlagAbort))
      continue; // capacity, a hot element or the step budget: the ordered path decides
    if (o.nRaces > r.race_cap) {
      r.n_races = o.nRaces;
      continue;
    }
    if (o.nTraps) { // canonical order: thread, then the thread's program order
      std::vector<uint32_t> ord(o.nTraps);
      std::iota(ord.begin(), ord.end(), o.trapOff);
      std::sort(ord.begin(), ord.end(),
                [&](uint32_t a, uint32_t b) { return trapKey[a] < trapKey[b]; });
      for (uint32_t q = 0; q < o.nTraps && q < r.trap_cap; ++q) {
        const uint32_t t = ord[q];
        r.traps[q] = hgrd_gpu_trap{static_cast<int32_t>(trapSite[t] >> 1),
                                   (trapSite[t] & 1) ? HGRD_TRAP_UNALLOCATED : HGRD_TRAP_OOB,
                                   static_cast<int64_t>(trapKey[t] >> 20)};
        r.n_traps = q + 1;
      }
      r.n_traps_total = o.nTraps;
    }
    const BatchPlan &P = plans[idx[k]];
    for (uint32_t q = 0; q < o.nRaces; ++q) {
      hgrd_gpu_race x = races[raceOffs[k] + q];
      x.handle = P.wHandle[static_cast<size_t>(x.handle)];
      r.races[q] = x;
    }
    r.n_races = o.nRaces;
    r.steps = static_cast<int64_t>(o.steps);
    r.instances = o.instances;
    r.records = o.records;
    r.mode = 0;
  }
  if (trace) {
    const auto t3 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    std::fprintf(stderr, "[hgrd batch] %u launches (%u in the envelope), blob %zu B, smem %zu B, "
                 "grid %u, traps %u; plan+stage %.0f, h2d+kernel+d2h %.0f, results %.0f (us)\n",
                 n, m, h2d, smem, grid, nTrapsAll, us(t0, t1), us(t1, t2), us(t2, t3));
  }
  return 0;
}
} // namespace

extern "C" {

int hgrd_gpu_create(int device, hgrd_gpu_ctx **out) {
  if (!out)
    return HGRD_GPU_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
    (void)cudaGetLastError();
    return HGRD_GPU_ENODEV;
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10)
    return HGRD_GPU_ENODEV; // built for sm_100a only
  auto *c = new hgrd_gpu_ctx();
  c->device = device;
  c->nSM = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->e0) != cudaSuccess || cudaEventCreate(&c->e1) != cudaSuccess ||
      cudaMallocHost(&c->hCtr, sizeof(Counters)) != cudaSuccess) {
    delete c;
    return HGRD_GPU_ECUDA;
  }
  *out = c;
  return 0;
}

void hgrd_gpu_destroy(hgrd_gpu_ctx *c) {
  if (!c)
    return;
  for (hgrd_gpu_ctx *w : c->workers)
    hgrd_gpu_destroy(w);
  cudaSetDevice(c->device);
  if (c->up)
    cudaStreamSynchronize(c->up);
  cudaStreamSynchronize(c->st);
  auto f = [](auto &v) {
    if (v.p)
      cudaFree(v.p);
  };
  f(c->keys), f(c->keysAlt), f(c->elemK), f(c->elemKAlt), f(c->vals), f(c->valsAlt);
  f(c->order), f(c->orderAlt), f(c->cubTemp), f(c->blob), f(c->snapshot), f(c->keySeg);
  f(c->keyPair), f(c->races), f(c->ctr), f(c->seqRegs), f(c->opIndex), f(c->opMeta);
  f(c->opSeq), f(c->opStart), f(c->traps), f(c->owner), f(c->keyElem), f(c->cand), f(c->ctr2);
  f(c->interTab), f(c->interKeyElem), f(c->targets), f(c->shardLo), f(c->shardHi), f(c->hot);
  f(c->doneKeys), f(c->doneTargets), f(c->lockC);
  for (char *ch : c->chunks)
    cudaFree(ch);
  for (auto &b : c->bigUsed)
    cudaFree(b.p);
  for (auto &kv : c->bigFree)
    cudaFree(kv.second);
  if (c->hStage)
    cudaFreeHost(c->hStage);
  if (c->hCtr)
    cudaFreeHost(c->hCtr);
  if (c->hRaces)
    cudaFreeHost(c->hRaces);
  if (c->hTraps)
    cudaFreeHost(c->hTraps);
  if (c->hResult)
    cudaFreeHost(c->hResult);
  if (c->hBatch)
    cudaFreeHost(c->hBatch);
  if (c->batchBlob.p)
    cudaFree(c->batchBlob.p);
  hgrdgpu::jit::destroy(c->jit);
  for (cudaEvent_t e : c->evPool)
    cudaEventDestroy(e);
  if (c->up) {
    cudaStreamSynchronize(c->up);
    cudaStreamDestroy(c->up);
  }
  for (cudaEvent_t e : c->upEvents)
    cudaEventDestroy(e);
  cudaEventDestroy(c->e0);
  cudaEventDestroy(c->e1);
  cudaStreamDestroy(c->st);
  delete c;
}

const char *hgrd_gpu_last_error(hgrd_gpu_ctx *c) { return c ? c->err.c_str() : "no context"; }

int hgrd_gpu_set_profiling(hgrd_gpu_ctx *c, int on) {
  if (!c)
    return HGRD_GPU_EINVAL;
  c->profiling = on != 0;
  return 0;
}

const char *hgrd_gpu_last_profile(hgrd_gpu_ctx *c) { return c ? c->profileJson.c_str() : "[]"; }

int hgrd_gpu_set_jit(hgrd_gpu_ctx *c, int mode) {
  if (!c || mode < 0 || mode > 2)
    return HGRD_GPU_EINVAL;
  c->jitMode = mode;
  return 0;
}

const char *hgrd_gpu_jit_info(hgrd_gpu_ctx *c) {
  if (!c)
    return "{}";
  char buf[256];
  std::snprintf(buf, sizeof buf,
                "{\"mode\":%d,\"compiles\":%d,\"compileMs\":%.1f,\"failures\":%d,\"lastError\":",
                c->jitMode, hgrdgpu::jit::compiles(c->jit), hgrdgpu::jit::compileMs(c->jit),
                c->jitFailures);
  std::string e;
  for (char ch : c->jitErr.substr(0, 2000))
    e += (ch == '"' || ch == '\\') ? ' ' : (ch == '\n' ? ' ' : ch);
  c->jitInfo = std::string(buf) + "\"" + e + "\"}";
  return c->jitInfo.c_str();
}

int hgrd_gpu_set_fused(hgrd_gpu_ctx *c, int enabled) {
  if (!c)
    return HGRD_GPU_EINVAL;
  c->fusedEnabled = enabled != 0;
  return 0;
}

unsigned long long hgrd_gpu_kernel_launches(hgrd_gpu_ctx *c) { return c ? c->kernelLaunches : 0; }

int hgrd_gpu_transfer_bytes(hgrd_gpu_ctx *c, unsigned long long *h2d, unsigned long long *d2h) {
  if (!c || !h2d || !d2h)
    return HGRD_GPU_EINVAL;
  *h2d = c->h2dBytes;
  *d2h = c->d2hBytes;
  return 0;
}

int hgrd_gpu_buffers_reset(hgrd_gpu_ctx *c) {
  if (!c)
    return HGRD_GPU_EINVAL;
  awaitUploads(c, nullptr); // (the memory is reused by later work on c->st)
  c->bufs.clear();
  c->chunkIdx = 0;
  c->chunkUsed = 0;
  for (auto &b : c->bigUsed)
    c->bigFree.emplace(b.bytes, b.p);
  c->bigUsed.clear();
  return 0;
}

int hgrd_gpu_buffer_alloc(hgrd_gpu_ctx *c, int64_t elems, int32_t *handle) {
  if (!c || !handle || elems <= 0)
    return HGRD_GPU_EINVAL;
  CK(cudaSetDevice(c->device));
  const size_t bytes = (static_cast<size_t>(elems) * 8 + 255) & ~size_t(255);
  char *p = nullptr;
  if (bytes <= c->chunkBytes / 4) {
    while (c->chunkIdx < c->chunks.size() && c->chunkUsed + bytes > c->chunkBytes) {
      ++c->chunkIdx;
      c->chunkUsed = 0;
    }
    if (c->chunkIdx == c->chunks.size()) {
      char *ch = nullptr;
      CK(cudaMalloc(&ch, c->chunkBytes));
      c->chunks.push_back(ch);
      c->chunkUsed = 0;
    }
    p = c->chunks[c->chunkIdx] + c->chunkUsed;
    c->chunkUsed += bytes;
  } else {
    auto it = c->bigFree.find(bytes);
    if (it != c->bigFree.end()) {
      p = static_cast<char *>(it->second);
      c->bigFree.erase(it);
    } else {
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        for (auto &kv : c->bigFree)
          cudaFree(kv.second);
        c->bigFree.clear();
        CK(cudaMalloc(&p, bytes));
      }
    }
    c->bigUsed.push_back(BigBlock{p, bytes});
  }
  // zero-initialised lazily: only values a check or the host reads need it
  c->bufs.push_back(hgrd_gpu_ctx::Buf{reinterpret_cast<int64_t *>(p), elems, true});
  *handle = static_cast<int32_t>(c->bufs.size() - 1);
  return 0;
}

int hgrd_gpu_buffer_write(hgrd_gpu_ctx *c, int32_t h, int64_t off, int64_t n,
                          const int64_t *src) {
  if (!c || h < 0 || static_cast<size_t>(h) >= c->bufs.size() || off < 0 || n < 0 ||
      off + n > c->bufs[static_cast<size_t>(h)].elems || (n && !src))
    return HGRD_GPU_EINVAL;
  if (n == 0)
    return 0;
  CK(cudaSetDevice(c->device));
  if (off == 0 && n == c->bufs[static_cast<size_t>(h)].elems)
    c->bufs[static_cast<size_t>(h)].zeroPending = false; // fully overwritten
  if (materialize(c, h) < 0)
    return HGRD_GPU_ECUDA;
  CK(cudaMemcpyAsync(c->bufs[static_cast<size_t>(h)].p + off, src, static_cast<size_t>(n) * 8,
                     cudaMemcpyHostToDevice, c->st));
  c->h2dBytes += static_cast<size_t>(n) * 8;
  return 0;
}

// The copy runs on the context's copy stream, after the work already queued
// on the context stream (which may still read the buffer) and any zeroing;
// later work touching the buffer waits for it on the device.
int hgrd_gpu_buffer_write_async(hgrd_gpu_ctx *c, int32_t h, int64_t off, int64_t n,
                                const int64_t *src) {
  if (!c || h < 0 || static_cast<size_t>(h) >= c->bufs.size() || off < 0 || n < 0 ||
      off + n > c->bufs[static_cast<size_t>(h)].elems || (n && !src))
    return HGRD_GPU_EINVAL;
  if (n == 0)
    return 0;
  CK(cudaSetDevice(c->device));
  if (!c->up)
    CK(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking));
  if (off == 0 && n == c->bufs[static_cast<size_t>(h)].elems)
    c->bufs[static_cast<size_t>(h)].zeroPending = false; // fully overwritten
  if (materialize(c, h) < 0) // (also orders a previous upload of h on c->st)
    return HGRD_GPU_ECUDA;
  if (c->upFree.empty()) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->upEvents.push_back(e);
    c->upFree.push_back(static_cast<int>(c->upEvents.size()) - 1);
  }
  const int slot = c->upFree.back();
  c->upFree.pop_back();
  cudaEvent_t ev = c->upEvents[static_cast<size_t>(slot)];
  CK(cudaEventRecord(ev, c->st)); // the copy follows the context stream's queued work
  CK(cudaStreamWaitEvent(c->up, ev, 0));
  CK(cudaMemcpyAsync(c->bufs[static_cast<size_t>(h)].p + off, src, static_cast<size_t>(n) * 8,
                     cudaMemcpyHostToDevice, c->up));
  CK(cudaEventRecord(ev, c->up));
  c->bufs[static_cast<size_t>(h)].upload = slot;
  c->h2dBytes += static_cast<size_t>(n) * 8;
  return 0;
}

int hgrd_gpu_buffer_read(hgrd_gpu_ctx *c, int32_t h, int64_t off, int64_t n, int64_t *dst) {
  if (!c || h < 0 || static_cast<size_t>(h) >= c->bufs.size() || off < 0 || n < 0 ||
      off + n > c->bufs[static_cast<size_t>(h)].elems || (n && !dst))
    return HGRD_GPU_EINVAL;
  if (n == 0)
    return 0;
  CK(cudaSetDevice(c->device));
  if (materialize(c, h) < 0)
    return HGRD_GPU_ECUDA;
  CK(cudaMemcpyAsync(dst, c->bufs[static_cast<size_t>(h)].p + off, static_cast<size_t>(n) * 8,
                     cudaMemcpyDeviceToHost, c->st));
  c->d2hBytes += static_cast<size_t>(n) * 8;
  CK(cudaStreamSynchronize(c->st));
  return 0;
}

int hgrd_gpu_check_launch(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch,
                          hgrd_gpu_result *result) {
  if (!c || !launch || !result || (!result->races && result->race_cap) ||
      (!result->traps && result->trap_cap))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return checkLaunch(c, *launch, result);
}

int hgrd_gpu_shard_check(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch, hgrd_gpu_shard *shard,
                         hgrd_gpu_result *result) {
  if (!c || !launch || !shard || !result || (!result->races && result->race_cap))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return shardCheck(c, *launch, shard, result);
}

int hgrd_gpu_check_batch(hgrd_gpu_ctx *c, const hgrd_gpu_batch_launch *launches, uint32_t n,
                         hgrd_gpu_result *results) {
  if (!c || (n && (!launches || !results)))
    return HGRD_GPU_EINVAL;
  for (uint32_t i = 0; i < n; ++i)
    if (!launches[i].buffer_elems && launches[i].n_buffers)
      return HGRD_GPU_EINVAL;
  CK(cudaSetDevice(c->device));
  awaitUploads(c, nullptr);
  try {
    return checkBatch(c, launches, n, results);
  } catch (const std::exception &e) {
    c->err = e.what();
    return HGRD_GPU_ENOMEM;
  }
}

void *hgrd_gpu_stream(hgrd_gpu_ctx *c) { return c ? static_cast<void *>(c->st) : nullptr; }

int hgrd_gpu_shard_inter_scan(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch, const void *lo,
                              const void *hi, uint64_t elem_begin, uint64_t n_elems,
                              uint64_t *key_elem, uint32_t n_keys) {
  if (!c || !launch || !key_elem || (n_elems && (!lo || !hi)))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return shardInterScan(c, *launch, static_cast<const uint32_t *>(lo),
                        static_cast<const uint32_t *>(hi), elem_begin, n_elems, key_elem, n_keys);
}

int hgrd_gpu_shard_inter_records(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch,
                                 const hgrd_gpu_shard *shard, const uint64_t *key_elem,
                                 uint32_t n_keys, uint64_t *keys, uint32_t *vals, uint64_t cap,
                                 uint64_t *n) {
  if (!c || !launch || !shard || !key_elem || !n || (cap && (!keys || !vals)))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return shardInterRecords(c, *launch, shard, key_elem, n_keys, keys, vals, cap, n);
}

int hgrd_gpu_shard_inter(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch,
                         const hgrd_gpu_shard *shard, uint64_t *keys, uint32_t *vals,
                         uint64_t cap, uint64_t *n) {
  if (!c || !launch || !shard || !n || (cap && (!keys || !vals)))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return shardInter(c, *launch, shard, keys, vals, cap, n);
}

int hgrd_gpu_shard_detect(hgrd_gpu_ctx *c, const hgrd_gpu_launch *launch, const uint64_t *keys,
                          const uint32_t *vals, uint64_t n, hgrd_gpu_result *result) {
  if (!c || !launch || !result || (n && (!keys || !vals)) ||
      (!result->races && result->race_cap))
    return HGRD_GPU_EINVAL;
  std::string why;
  if (!validLaunch(*launch, why)) {
    c->err = why;
    return HGRD_GPU_EINVAL;
  }
  CK(cudaSetDevice(c->device));
  awaitUploads(c, launch);
  return shardDetect(c, *launch, keys, vals, n, result);
}

} // extern "C"

namespace hgrdgpu {
void setError(hgrd_gpu_ctx *c, const std::string &m) {
  if (c)
    c->err = m;
}

// Worker i (>= 1) of a context for parallel sweeps: a further context on
// the same device, created on first use and destroyed with its parent;
// worker 0 is the context itself.  nullptr when it cannot be created.
hgrd_gpu_ctx *sweepWorker(hgrd_gpu_ctx *c, int i) {
  if (i == 0)
    return c;
  while (static_cast<int>(c->workers.size()) < i) {
    hgrd_gpu_ctx *w = nullptr;
    if (hgrd_gpu_create(c->device, &w) != HGRD_GPU_OK)
      return nullptr;
    w->fusedEnabled = c->fusedEnabled;
    w->jitMode = c->jitMode;
    c->workers.push_back(w);
  }
  return c->workers[static_cast<size_t>(i - 1)];
}
// Per-check device timing (events around the check; device_ms).  Sweeps of
// tiny launches turn it off: the extra event round trip is ~12% of a check.
bool setTiming(hgrd_gpu_ctx *c, bool on) {
  const bool was = c->timing;
  c->timing = on && std::getenv("HGRD_NO_DEVICE_TIMING") == nullptr;
  return was;
}
} // namespace hgrdgpu

// K3/K4: conflict detection over key-sorted records.
//
// Reference semantics (src/oracle.cpp:745-769): for events a, b on one
// element from different threads, with at least one write, not both
// atomics whose scopes cover the pair, and not ordered by a barrier phase
// or a lock, the pair races with kind INTER-BLOCK (blocks differ),
// INTRA-BLOCK (same block, warps differ) or INTRA-WARP.
//
// Summary detector (no lock idioms).  After sorting by
//   element | block | blockPhase | warp | warpPhase | lane
// the three kinds are "two distinct ids inside one group":
//   INTER : group element,                             id block
//   INTRA-BLOCK : group (element, block, blockPhase),   id warp
//   INTRA-WARP  : group (element, block, bp, warp, wp), id lane
// and the write / atomic-scope rules are static per site pair (conf masks).
// So a site pair (s1, s2) realises a kind on an element iff the union of
// their ids in some group has two values: min(min1,min2) < max(max1,max2).
// One thread per element segment keeps per-site (min, max) at the three
// levels — O(g·S) instead of the reference's O(g²) pair loop — and
// publishes, per realised key, the minimum segment start (= minimum
// (handle, index), the reference's first-found element, :745).
//
// Witness (first pair in reference order inside that element): x is the
// earliest event (thread, seq) that has a later partner; "later" in event
// order inside a group is exactly "larger id" at that level, so x
// qualifies iff a partner site's max id in its group exceeds id(x); y is
// the earliest partner event with a larger id in x's group.
//
// Pairwise detector (kernels with fence + CAS/Exch lock idioms, whose
// lockInfo ordering (:678-728) is not a group property): records in
// canonical event order, stably sorted by element, brute-force pairs in
// the reference's x<y order, first pair per key via a packed atomicMin.
#pragma once

#include "device.cuh"

namespace hgrdgpu {
namespace dev {

struct DetectArgs {
  const uint64_t *keys;
  const uint32_t *vals;
  uint64_t n;
  KeyLayout kl;
  const SiteDev *sites;
  const uint64_t *confInter, *confIntra, *locMask;
  int nLocs, nSites;
  int64_t tpb, ws;
  // element -> (handle, index) over written buffers
  const uint64_t *wBase;
  const int32_t *wHandle;
  int nW;
  int kindMask; // kinds to report: bit 0 INTER-BLOCK, 1 INTRA-BLOCK, 2 INTRA-WARP
  // INTER-only detection: elements with more than kHotGroup records are
  // listed here and summarised by a warp each (k_detect_hot)
  uint32_t *hotList;
  unsigned *hotCount;
  uint32_t hotCap;
};

constexpr int kHotGroup = 64;

__device__ __forceinline__ void siteKey(const DetectArgs &A, int a, int b, int kind,
                                        uint32_t segStart, uint32_t *keySeg) {
  int la = A.sites[a].loc, lb = A.sites[b].loc;
  if (lb < la) {
    int t = la;
    la = lb;
    lb = t;
  }
  const int K = (la * A.nLocs + lb) * 3 + kind;
  if (keySeg[K] > segStart)
    atomicMin(&keySeg[K], segStart);
}

__device__ __forceinline__ void flushLevel(const DetectArgs &A, uint64_t pres,
                                           const uint32_t *mn, const uint32_t *mx,
                                           const uint64_t *conf, int kind,
                                           uint32_t segStart, uint32_t *keySeg) {
  uint64_t rem = pres;
  while (rem) {
    const int a = __ffsll(static_cast<long long>(rem)) - 1;
    rem &= rem - 1;
    uint64_t m = conf[a] & pres & ~((1ull << a) - 1);
    while (m) {
      const int b = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      const uint32_t lo = min(mn[a], mn[b]);
      const uint32_t hi = max(mx[a], mx[b]);
      if (lo < hi)
        siteKey(A, a, b, kind, segStart, keySeg);
    }
  }
}

__device__ __forceinline__ void note(uint64_t &pres, uint32_t *mn, uint32_t *mx,
                                     int s, uint32_t id) {
  const uint64_t bit = 1ull << s;
  if (!(pres & bit)) {
    pres |= bit;
    mn[s] = id;
    mx[s] = id;
  } else {
    mn[s] = min(mn[s], id);
    mx[s] = max(mx[s], id);
  }
}

__global__ void k_detect_summary(DetectArgs A, uint32_t *keySeg) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= A.n)
    return;
  const KeyLayout kl = A.kl;
  const uint64_t k0 = A.keys[i];
  if (k0 == kl.sentinel)
    return;
  const uint64_t elem = k0 >> kl.shE;
  if (i > 0 && (A.keys[i - 1] >> kl.shE) == elem)
    return; // not the first record of its element
  if (i + 1 >= A.n || (A.keys[i + 1] >> kl.shE) != elem)
    return; // a lone access cannot race
  if (A.hotList && A.kindMask == 1 && i + kHotGroup < A.n &&
      (A.keys[i + kHotGroup] >> kl.shE) == elem) { // a hot element: one warp (k_detect_hot)
    const unsigned slot = atomicAdd(A.hotCount, 1u);
    if (slot < A.hotCap) {
      A.hotList[slot] = static_cast<uint32_t>(i);
      return;
    }
  }
  const uint64_t mB = fieldMask(kl.bB), mW = fieldMask(kl.bW), mL = fieldMask(kl.bL);
  uint32_t mn1[kMaxSites], mx1[kMaxSites], mn2[kMaxSites], mx2[kMaxSites],
      mn3[kMaxSites], mx3[kMaxSites];
  uint64_t p1 = 0, p2 = 0, p3 = 0;
  uint64_t g2 = k0 >> kl.shP, g3 = k0 >> kl.shQ;
  const uint32_t seg = static_cast<uint32_t>(i);
  const bool lv1 = A.kindMask & 1, lv2 = A.kindMask & 2, lv3 = A.kindMask & 4;
  for (uint64_t j = i; j < A.n; ++j) {
    const uint64_t k = A.keys[j];
    if ((k >> kl.shE) != elem)
      break;
    const int s = static_cast<int>(A.vals[j] >> kl.bS);
    if (!(lv2 | lv3)) { // INTER only (fused pass 2): the block level alone
      note(p1, mn1, mx1, s, static_cast<uint32_t>((k >> kl.shB) & mB));
      continue;
    }
    if ((k >> kl.shP) != g2) {
      if (A.kindMask & 2)
        flushLevel(A, p2, mn2, mx2, A.confIntra, 1, seg, keySeg);
      p2 = 0;
      g2 = k >> kl.shP;
    }
    if ((k >> kl.shQ) != g3) {
      if (A.kindMask & 4)
        flushLevel(A, p3, mn3, mx3, A.confIntra, 2, seg, keySeg);
      p3 = 0;
      g3 = k >> kl.shQ;
    }
    if (lv1)
      note(p1, mn1, mx1, s, static_cast<uint32_t>((k >> kl.shB) & mB));
    if (lv2)
      note(p2, mn2, mx2, s, static_cast<uint32_t>((k >> kl.shW) & mW));
    if (lv3)
      note(p3, mn3, mx3, s, static_cast<uint32_t>(k & mL));
  }
  if (A.kindMask & 1)
    flushLevel(A, p1, mn1, mx1, A.confInter, 0, seg, keySeg);
  if (A.kindMask & 2)
    flushLevel(A, p2, mn2, mx2, A.confIntra, 1, seg, keySeg);
  if (A.kindMask & 4)
    flushLevel(A, p3, mn3, mx3, A.confIntra, 2, seg, keySeg);
}

// INTER level of the hot elements listed by k_detect_summary: the lanes of
// a warp stride over the element's records keeping per-site (min, max)
// block, the warp reduces them per present site and lane 0 flushes.
__global__ void k_detect_hot(DetectArgs A, uint32_t *keySeg) {
  const int lane = threadIdx.x & 31;
  const unsigned nHot = min(*A.hotCount, A.hotCap);
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nWarps = (gridDim.x * blockDim.x) >> 5;
  const KeyLayout kl = A.kl;
  const uint64_t mB = fieldMask(kl.bB);
  for (unsigned h = warp; h < nHot; h += nWarps) {
    const uint64_t i = A.hotList[h];
    const uint64_t elem = A.keys[i] >> kl.shE;
    uint32_t mn[kMaxSites], mx[kMaxSites];
    uint64_t p = 0;
    for (uint64_t j = i + lane; j < A.n; j += 32) {
      const uint64_t k = A.keys[j];
      if ((k >> kl.shE) != elem)
        break;
      note(p, mn, mx, static_cast<int>(A.vals[j] >> kl.bS),
           static_cast<uint32_t>((k >> kl.shB) & mB));
    }
    uint64_t all = p;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      all |= __shfl_xor_sync(0xffffffffu, all, o);
    uint64_t rem = all;
    while (rem) { // warp-uniform
      const int s = __ffsll(static_cast<long long>(rem)) - 1;
      rem &= rem - 1;
      const bool has = (p >> s) & 1ull;
      uint32_t a = has ? mn[s] : 0xffffffffu, b = has ? mx[s] : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
      }
      if (lane == 0) {
        mn[s] = a;
        mx[s] = b;
      }
    }
    if (lane == 0)
      flushLevel(A, all, mn, mx, A.confInter, 0, static_cast<uint32_t>(i), keySeg);
  }
}

__device__ __forceinline__ void elementOf(const DetectArgs &A, uint64_t elem,
                                          int32_t &handle, int64_t &index) {
  int w = 0;
  for (int q = 1; q < A.nW; ++q)
    if (A.wBase[q] <= elem)
      w = q;
  handle = A.wHandle[w];
  index = static_cast<int64_t>(elem - A.wBase[w]);
}

__device__ __forceinline__ uint64_t eventOrder(const DetectArgs &A, uint64_t k, uint32_t v) {
  const KeyLayout &kl = A.kl;
  const uint64_t block = (k >> kl.shB) & fieldMask(kl.bB);
  const uint64_t warp = (k >> kl.shW) & fieldMask(kl.bW);
  const uint64_t lane = k & fieldMask(kl.bL);
  const uint64_t thread = block * static_cast<uint64_t>(A.tpb) +
                          warp * static_cast<uint64_t>(A.ws) + lane;
  return (thread << kl.bS) | (v & seqMask(kl));
}

// Early stop of the prefix-wise INTER witness pass (fused pass 2b): for
// INTER key keyList[w] with first-found element target[w], done[w] = 1 once
// the earliest recorded event of that element at one of the key's locs, x,
// has a partner among the records so far — a later event of another block
// at the other loc whose site conflicts across blocks.  Records of later
// blocks come later in the reference order, so x and its first partner are
// then final.
__global__ void k_inter_done(const uint64_t *keys, const uint32_t *vals, uint64_t n,
                             KeyLayout kl, int64_t tpb, int64_t ws, const SiteDev *sites,
                             const uint64_t *confInter, int nLocs, const int *keyList,
                             const uint64_t *target, int nK, int *done) {
  const int w = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= nK)
    return;
  const int K = keyList[w];
  const int la = (K / 3) / nLocs, lb = (K / 3) % nLocs;
  const uint64_t e = target[w];
  const uint64_t mB = fieldMask(kl.bB), mW = fieldMask(kl.bW), mL = fieldMask(kl.bL);
  auto order = [&](uint64_t k, uint32_t v) {
    const uint64_t thread = ((k >> kl.shB) & mB) * static_cast<uint64_t>(tpb) +
                            ((k >> kl.shW) & mW) * static_cast<uint64_t>(ws) + (k & mL);
    return (thread << kl.bS) | (v & seqMask(kl));
  };
  uint64_t best = ~0ull; // earliest eligible event (order), its site and block
  int bs = -1;
  uint64_t bb = 0;
  for (uint64_t i = lane; i < n; i += 32) {
    const uint64_t k = keys[i];
    if (k == kl.sentinel || (k >> kl.shE) != e)
      continue;
    const int s = static_cast<int>(vals[i] >> kl.bS);
    const int loc = sites[s].loc;
    if (loc != la && loc != lb)
      continue;
    const uint64_t o = order(k, vals[i]);
    if (o < best) {
      best = o;
      bs = s;
      bb = (k >> kl.shB) & mB;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int os = __shfl_xor_sync(0xffffffffu, bs, off);
    const uint64_t obb = __shfl_xor_sync(0xffffffffu, bb, off);
    if (ob < best) {
      best = ob;
      bs = os;
      bb = obb;
    }
  }
  bool found = false;
  if (bs >= 0) {
    const int lx = sites[bs].loc;
    const int want = lx == la ? lb : la; // the partner's loc
    for (uint64_t i = lane; i < n && !found; i += 32) {
      const uint64_t k = keys[i];
      if (k == kl.sentinel || (k >> kl.shE) != e || ((k >> kl.shB) & mB) == bb)
        continue;
      const int s = static_cast<int>(vals[i] >> kl.bS);
      if (sites[s].loc != want || !((confInter[bs] >> s) & 1ull))
        continue;
      found = order(k, vals[i]) > best;
    }
  }
  found = __any_sync(0xffffffffu, found);
  if (lane == 0)
    done[w] = found ? 1 : 0;
}

__device__ __forceinline__ uint32_t levelId(const KeyLayout &kl, int kind, uint64_t k) {
  if (kind == 0)
    return static_cast<uint32_t>((k >> kl.shB) & fieldMask(kl.bB));
  if (kind == 1)
    return static_cast<uint32_t>((k >> kl.shW) & fieldMask(kl.bW));
  return static_cast<uint32_t>(k & fieldMask(kl.bL));
}

// One thread per race key; realised keys extract their witness pair.
__global__ void k_witness(DetectArgs A, const uint32_t *keySeg, int nKeys,
                          hgrd_gpu_race *races, Counters *ctr) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K >= nKeys)
    return;
  const uint32_t s = keySeg[K];
  if (s == 0xffffffffu)
    return;
  const KeyLayout kl = A.kl;
  const int kind = K % 3;
  if (!((A.kindMask >> kind) & 1))
    return;
  const int la = (K / 3) / A.nLocs, lb = (K / 3) % A.nLocs;
  const uint64_t *conf = kind == 0 ? A.confInter : A.confIntra;
  const int gsh = kind == 0 ? kl.shE : kind == 1 ? kl.shP : kl.shQ;
  const uint64_t elem = A.keys[s] >> kl.shE;
  uint64_t e = s;
  while (e < A.n && (A.keys[e] >> kl.shE) == elem)
    ++e;
  uint32_t mx[kMaxSites];
  uint64_t best = ~0ull, bestPm = 0;
  uint64_t bestI = s, bestG0 = s, bestG1 = e;
  for (uint64_t j = s; j < e;) {
    const uint64_t g = A.keys[j] >> gsh;
    uint64_t ge = j;
    uint64_t pres = 0;
    for (; ge < e && (A.keys[ge] >> gsh) == g; ++ge) {
      const int st = static_cast<int>(A.vals[ge] >> kl.bS);
      const uint32_t id = levelId(kl, kind, A.keys[ge]);
      const uint64_t bit = 1ull << st;
      if (!(pres & bit)) {
        pres |= bit;
        mx[st] = id;
      } else if (id > mx[st]) {
        mx[st] = id;
      }
    }
    for (uint64_t x = j; x < ge; ++x) {
      const int st = static_cast<int>(A.vals[x] >> kl.bS);
      const int loc = A.sites[st].loc;
      if (loc != la && loc != lb)
        continue;
      const int ploc = loc == la ? lb : la;
      const uint64_t pm = conf[st] & A.locMask[ploc] & pres;
      const uint32_t id = levelId(kl, kind, A.keys[x]);
      bool later = false;
      for (uint64_t m = pm; m && !later; m &= m - 1)
        later = mx[__ffsll(static_cast<long long>(m)) - 1] > id;
      if (!later)
        continue;
      const uint64_t ord = eventOrder(A, A.keys[x], A.vals[x]);
      if (ord < best) {
        best = ord;
        bestI = x;
        bestPm = pm;
        bestG0 = j;
        bestG1 = ge;
      }
    }
    j = ge;
  }
  if (best == ~0ull)
    return; // cannot happen for a realised key
  const uint32_t idx = levelId(kl, kind, A.keys[bestI]);
  uint64_t bestY = ~0ull, yI = bestI;
  for (uint64_t y = bestG0; y < bestG1; ++y) {
    const int st = static_cast<int>(A.vals[y] >> kl.bS);
    if (!((bestPm >> st) & 1ull) || levelId(kl, kind, A.keys[y]) <= idx)
      continue;
    const uint64_t ord = eventOrder(A, A.keys[y], A.vals[y]);
    if (ord < bestY) {
      bestY = ord;
      yI = y;
    }
  }
  const unsigned pos = atomicAdd(&ctr->nRaces, 1u);
  hgrd_gpu_race &o = races[pos];
  o.loc_a = la;
  o.loc_b = lb;
  o.kind = kind;
  o.site_x = static_cast<int32_t>(A.vals[bestI] >> kl.bS);
  o.site_y = static_cast<int32_t>(A.vals[yI] >> kl.bS);
  elementOf(A, elem, o.handle, o.index);
  o.thread_x = static_cast<int64_t>(best >> kl.bS);
  o.seq_x = static_cast<int32_t>(best & seqMask(kl));
  o.thread_y = static_cast<int64_t>(bestY >> kl.bS);
  o.seq_y = static_cast<int32_t>(bestY & seqMask(kl));
}

// INTER-BLOCK witness, one warp per key: the whole element segment is one
// group (level id = block), so the three passes of k_witness become warp
// reductions — hot elements (histogram bins) have thousands of events.
__global__ void k_witness_inter(DetectArgs A, const uint32_t *keySeg, int nKeys,
                                hgrd_gpu_race *races, Counters *ctr) {
  __shared__ uint32_t smx[8][kMaxSites];
  __shared__ unsigned long long spres[8];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = (blockIdx.x * (blockDim.x >> 5) + wid) * 3; // kind 0 keys only
  if (K >= nKeys)
    return;
  const uint32_t s = keySeg[K];
  if (s == 0xffffffffu)
    return;
  const KeyLayout kl = A.kl;
  const int la = (K / 3) / A.nLocs, lb = (K / 3) % A.nLocs;
  const uint64_t elem = A.keys[s] >> kl.shE;
  // segment end: lanes probe ahead in strides of 32
  uint64_t e = s;
  for (;;) {
    const uint64_t p = e + lane;
    const bool in = p < A.n && (A.keys[p] >> kl.shE) == elem;
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (m != 0xffffffffu) {
      e += __popc(m);
      break;
    }
    e += 32;
  }
  uint32_t *mx = smx[wid];
  if (lane == 0)
    spres[wid] = 0;
  for (int i = lane; i < kMaxSites; i += 32)
    mx[i] = 0;
  __syncwarp();
  for (uint64_t p = s + lane; p < e; p += 32) {
    const int st = static_cast<int>(A.vals[p] >> kl.bS);
    atomicMax(&mx[st], static_cast<uint32_t>((A.keys[p] >> kl.shB) & fieldMask(kl.bB)));
    atomicOr(&spres[wid], 1ull << st);
  }
  __syncwarp();
  const uint64_t pres = spres[wid];
  // x: earliest event with a partner in a later block
  uint64_t bx = ~0ull, bpm = 0, bxi = s;
  for (uint64_t p = s + lane; p < e; p += 32) {
    const int st = static_cast<int>(A.vals[p] >> kl.bS);
    const int loc = A.sites[st].loc;
    if (loc != la && loc != lb)
      continue;
    const uint64_t pm = A.confInter[st] & A.locMask[loc == la ? lb : la] & pres;
    const uint32_t id = static_cast<uint32_t>((A.keys[p] >> kl.shB) & fieldMask(kl.bB));
    bool later = false;
    for (uint64_t m = pm; m && !later; m &= m - 1)
      later = mx[__ffsll(static_cast<long long>(m)) - 1] > id;
    if (!later)
      continue;
    const uint64_t ord = eventOrder(A, A.keys[p], A.vals[p]);
    if (ord < bx) {
      bx = ord;
      bpm = pm;
      bxi = p;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ox = __shfl_down_sync(0xffffffffu, bx, o);
    const uint64_t om = __shfl_down_sync(0xffffffffu, bpm, o);
    const uint64_t oi = __shfl_down_sync(0xffffffffu, bxi, o);
    if (ox < bx) {
      bx = ox;
      bpm = om;
      bxi = oi;
    }
  }
  bx = __shfl_sync(0xffffffffu, bx, 0);
  bpm = __shfl_sync(0xffffffffu, bpm, 0);
  bxi = __shfl_sync(0xffffffffu, bxi, 0);
  if (bx == ~0ull)
    return;
  // y: earliest partner event in a later block
  const uint32_t idx = static_cast<uint32_t>((A.keys[bxi] >> kl.shB) & fieldMask(kl.bB));
  uint64_t by = ~0ull, byi = bxi;
  for (uint64_t p = s + lane; p < e; p += 32) {
    const int st = static_cast<int>(A.vals[p] >> kl.bS);
    if (!((bpm >> st) & 1ull) ||
        static_cast<uint32_t>((A.keys[p] >> kl.shB) & fieldMask(kl.bB)) <= idx)
      continue;
    const uint64_t ord = eventOrder(A, A.keys[p], A.vals[p]);
    if (ord < by) {
      by = ord;
      byi = p;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t oy = __shfl_down_sync(0xffffffffu, by, o);
    const uint64_t oi = __shfl_down_sync(0xffffffffu, byi, o);
    if (oy < by) {
      by = oy;
      byi = oi;
    }
  }
  if (lane != 0)
    return;
  const unsigned pos = atomicAdd(&ctr->nRaces, 1u);
  hgrd_gpu_race &o = races[pos];
  o.loc_a = la;
  o.loc_b = lb;
  o.kind = 0;
  o.site_x = static_cast<int32_t>(A.vals[bxi] >> kl.bS);
  o.site_y = static_cast<int32_t>(A.vals[byi] >> kl.bS);
  elementOf(A, elem, o.handle, o.index);
  o.thread_x = static_cast<int64_t>(bx >> kl.bS);
  o.seq_x = static_cast<int32_t>(bx & seqMask(kl));
  o.thread_y = static_cast<int64_t>(by >> kl.bS);
  o.seq_y = static_cast<int32_t>(by & seqMask(kl));
}

// ---------------------------------------------------------------------------
// Pairwise path (lock idioms).  Records are in canonical event order;
// order[] is the stable sort of record indices by element.

struct LockSet {
  int n;
  int32_t h[8];
  int64_t idx[8];
  int32_t scope[8];
};

__device__ __forceinline__ void lockInsert(LockSet &s, int32_t h, int64_t idx, int32_t sc,
                                           unsigned &flags) {
  for (int i = 0; i < s.n; ++i)
    if (s.h[i] == h && s.idx[i] == idx) {
      if (sc > s.scope[i])
        s.scope[i] = sc;
      return;
    }
  if (s.n < 8) {
    s.h[s.n] = h;
    s.idx[s.n] = idx;
    s.scope[s.n] = sc;
    ++s.n;
  } else {
    flags |= kFlagLockSet;
  }
}

struct LockInfo {
  LockSet acq, rel, cs;
};

// reference lockInfo, src/oracle.cpp:678-704
__device__ void lockInfoOf(const LaunchDev &L, uint64_t thread, int32_t seq,
                           LockInfo &li, unsigned &flags) {
  li.acq.n = li.rel.n = li.cs.n = 0;
  // (PARALLEL launches: fixed slots per thread, unused ones kind 15)
  const uint64_t b = L.opStride ? thread * L.opStride : L.opStart[thread];
  const uint64_t e = L.opStride ? b + L.opStride : L.opStart[thread + 1];
  for (uint64_t f = b; f < e; ++f) {
    const int32_t mf = L.opMeta[f];
    if ((mf & 15) != 2)
      continue;
    const int32_t fs = L.opSeq[f], fsc = (mf >> 4) & 15;
    for (uint64_t c = b; c < e; ++c) {
      const int32_t mc = L.opMeta[c];
      if ((mc & 15) != 0 || L.opSeq[c] >= fs)
        continue;
      if (fs < seq)
        lockInsert(li.acq, (mc >> 8) - 1, L.opIndex[c], min((mc >> 4) & 15, fsc), flags);
    }
    for (uint64_t x = b; x < e; ++x) {
      const int32_t mx = L.opMeta[x];
      if ((mx & 15) != 1 || L.opSeq[x] <= fs)
        continue;
      if (fs > seq)
        lockInsert(li.rel, (mx >> 8) - 1, L.opIndex[x], min((mx >> 4) & 15, fsc), flags);
    }
  }
  for (int i = 0; i < li.acq.n; ++i)
    for (int j = 0; j < li.rel.n; ++j)
      if (li.acq.h[i] == li.rel.h[j] && li.acq.idx[i] == li.rel.idx[j])
        lockInsert(li.cs, li.acq.h[i], li.acq.idx[i], min(li.acq.scope[i], li.rel.scope[j]),
                   flags);
}

__device__ __forceinline__ bool covers(int32_t s, bool sameBlock) {
  return s == HGRD_SCOPE_DEVICE || (s == HGRD_SCOPE_BLOCK && sameBlock);
}
__device__ __forceinline__ bool crossed(const LockSet &x, const LockSet &y, bool sameBlock) {
  for (int i = 0; i < x.n; ++i)
    for (int j = 0; j < y.n; ++j)
      if (x.h[i] == y.h[j] && x.idx[i] == y.idx[j] && covers(min(x.scope[i], y.scope[j]), sameBlock))
        return true;
  return false;
}

// Exact lockOrdered (reference :678-728) straight from two threads' sync-op
// lists, for events whose lock sets exceed LockSet's 8 entries (no limit;
// quadratic in the ops, so only the fallback).  Scopes: 0 absent, 1 block,
// 2 device; an acquire of lock (h, i) before event seq is a CAS on it
// before a fence before seq (scope: the narrower of the two, the widest
// such pair), a release an Exch after a fence after seq; a critical section
// both, scope the narrower.
__device__ int lockScopeOf(const LaunchDev &L, uint64_t thread, int32_t seq, int32_t h,
                           int64_t idx, bool acquire) {
  const uint64_t b = L.opStride ? thread * L.opStride : L.opStart[thread];
  const uint64_t e = L.opStride ? b + L.opStride : L.opStart[thread + 1];
  int best = 0;
  for (uint64_t f = b; f < e; ++f) {
    const int32_t mf = L.opMeta[f];
    if ((mf & 15) != 2)
      continue;
    const int32_t fs = L.opSeq[f], fsc = (mf >> 4) & 15;
    if (acquire ? !(fs < seq) : !(fs > seq))
      continue;
    for (uint64_t c = b; c < e; ++c) {
      const int32_t mc = L.opMeta[c];
      if ((mc & 15) != (acquire ? 0 : 1) || (mc >> 8) - 1 != h || L.opIndex[c] != idx)
        continue;
      if (acquire ? L.opSeq[c] >= fs : L.opSeq[c] <= fs)
        continue;
      best = max(best, min((mc >> 4) & 15, fsc));
    }
  }
  return best;
}

__device__ bool lockOrderedDirect(const LaunchDev &L, uint64_t ta, int32_t sa, uint64_t tb,
                                  int32_t sb, bool sameBlock) {
  const uint64_t b = L.opStride ? ta * L.opStride : L.opStart[ta];
  const uint64_t e = L.opStride ? b + L.opStride : L.opStart[ta + 1];
  for (uint64_t o = b; o < e; ++o) { // every lock of a's sets is one of a's CAS / Exch
    const int32_t m = L.opMeta[o];
    if ((m & 15) > 1)
      continue;
    const int32_t h = (m >> 8) - 1;
    const int64_t idx = L.opIndex[o];
    const int acqA = lockScopeOf(L, ta, sa, h, idx, true);
    const int relA = lockScopeOf(L, ta, sa, h, idx, false);
    const int acqB = lockScopeOf(L, tb, sb, h, idx, true);
    const int relB = lockScopeOf(L, tb, sb, h, idx, false);
    const int csA = (acqA && relA) ? min(acqA, relA) : 0;
    const int csB = (acqB && relB) ? min(acqB, relB) : 0;
    if ((csA && csB && covers(min(csA, csB), sameBlock)) ||
        (relA && acqB && covers(min(relA, acqB), sameBlock)) ||
        (relB && acqA && covers(min(relB, acqA), sameBlock)))
      return true;
  }
  return false;
}

// lockOrdered(a, b) from both events' lock facts (a's computed once per row);
// the exact direct evaluation when a set overflowed LockSet.
template <class E>
__device__ bool lockPairOrdered(const LaunchDev &L, const E &a, const E &b, bool sameBlock,
                                LockInfo &la, bool &laFull, bool &laWide, LockInfo &lb) {
  if (!laFull) {
    unsigned f = 0;
    lockInfoOf(L, a.thread, a.seq, la, f);
    laWide = (f & kFlagLockSet) != 0;
    laFull = true;
  }
  unsigned f = 0;
  lockInfoOf(L, b.thread, b.seq, lb, f);
  if (laWide || (f & kFlagLockSet))
    return lockOrderedDirect(L, a.thread, a.seq, b.thread, b.seq, sameBlock);
  return crossed(la.cs, lb.cs, sameBlock) || crossed(la.rel, lb.acq, sameBlock) ||
         crossed(lb.rel, la.acq, sameBlock);
}

// Per-event lock facts precomputed once (k_lock_info) instead of per pair:
// up to two entries per set, entry = (handle + 1) << 48 | scope << 46 |
// index, 0 = empty.  Wider sets, handles or indices mark the event
// kLockWide and pairRow recomputes its LockInfo.
struct LockC {
  uint64_t cs[2], acq[2], rel[2];
};
constexpr uint64_t kLockWide = ~0ull;
constexpr uint64_t kLockScopeBits = 3ull << 46;

__device__ __forceinline__ bool packSet(const LockSet &s, uint64_t *out) {
  if (s.n > 2)
    return false;
  for (int i = 0; i < 2; ++i) {
    out[i] = 0;
    if (i < s.n) {
      if (s.h[i] < 0 || s.h[i] >= 0xffff || s.idx[i] < 0 || s.idx[i] >= (int64_t(1) << 46) ||
          s.scope[i] < 0 || s.scope[i] > 3)
        return false;
      out[i] = (static_cast<uint64_t>(s.h[i] + 1) << 48) |
               (static_cast<uint64_t>(s.scope[i]) << 46) | static_cast<uint64_t>(s.idx[i]);
    }
  }
  return true;
}

__device__ __forceinline__ bool crossedC(const uint64_t *x, const uint64_t *y, bool sameBlock) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (x[i] && y[j] && ((x[i] ^ y[j]) & ~kLockScopeBits) == 0 &&
          covers(static_cast<int32_t>(min(x[i], y[j]) >> 46) & 3, sameBlock))
        return true;
  return false;
}

struct Ev {
  uint64_t block, warp, lane, bp, wp, thread;
  int site, seq;
};

__device__ __forceinline__ Ev decodeEv(const DetectArgs &A, uint64_t k, uint32_t v) {
  const KeyLayout &kl = A.kl;
  Ev e;
  e.block = (k >> kl.shB) & fieldMask(kl.bB);
  e.bp = (k >> kl.shP) & fieldMask(kl.bP);
  e.warp = (k >> kl.shW) & fieldMask(kl.bW);
  e.wp = (k >> kl.shQ) & fieldMask(kl.bQ);
  e.lane = k & fieldMask(kl.bL);
  e.thread = e.block * static_cast<uint64_t>(A.tpb) + e.warp * static_cast<uint64_t>(A.ws) + e.lane;
  e.site = static_cast<int>(v >> kl.bS);
  e.seq = static_cast<int>(v & seqMask(kl));
  return e;
}

// Pairs of one element group (sorted by element, canonical order within),
// the reference's detectRaces rule (:730-784) including lockOrdered.  The
// first-found pair per key is the minimum of (element, x, y): keyPair holds
// the least group start << 32 | x offset (the group start orders elements),
// and k_pair_first_y then finds the least y of that row with the key.
constexpr uint64_t kPairEventsMax = 1ull << 32; // (u32 sort order)
constexpr uint64_t kPairBig = 64; // larger groups: k_detect_pairwise_big

// The key of pair (a = event x, b = event y), or -1 when it is no race:
// one thread, two loads, covering atomics, separated phases or lock order.
__device__ __forceinline__ int pairKey(const DetectArgs &A, const LaunchDev &L,
                                       const uint32_t *order, bool locks, const LockC *lc,
                                       const Ev &a, const SiteDev &sa, const LockC &ca,
                                       uint64_t y, LockInfo &la, bool &laFull, bool &laWide,
                                       LockInfo &lb) {
  const Ev b = decodeEv(A, A.keys[order[y]], A.vals[order[y]]);
  if (a.thread == b.thread)
    return -1;
  const SiteDev sb = A.sites[b.site];
  if (sa.kind == HGRD_SITE_LOAD && sb.kind == HGRD_SITE_LOAD)
    return -1;
  const bool sameBlock = a.block == b.block;
  if (sa.kind == HGRD_SITE_ATOMIC && sb.kind == HGRD_SITE_ATOMIC &&
      covers(sa.scope, sameBlock) && covers(sb.scope, sameBlock))
    return -1;
  if (sameBlock && a.bp != b.bp)
    return -1;
  const bool sameWarp = sameBlock && a.warp == b.warp;
  if (sameWarp && a.wp != b.wp)
    return -1;
  if (locks) {
    bool ordered;
    const LockC cb = lc ? lc[y] : LockC{};
    if (lc && ca.cs[0] != kLockWide && cb.cs[0] != kLockWide) {
      ordered = crossedC(ca.cs, cb.cs, sameBlock) || crossedC(ca.rel, cb.acq, sameBlock) ||
                crossedC(cb.rel, ca.acq, sameBlock);
    } else {
      ordered = lockPairOrdered(L, a, b, sameBlock, la, laFull, laWide, lb);
    }
    if (ordered)
      return -1;
  }
  const int kind = !sameBlock ? 0 : !sameWarp ? 1 : 2;
  int l0 = sa.loc, l1 = sb.loc;
  if (l1 < l0) {
    const int t = l0;
    l0 = l1;
    l1 = t;
  }
  return (l0 * A.nLocs + l1) * 3 + kind;
}

__device__ __forceinline__ void pairRow(const DetectArgs &A, const LaunchDev &L,
                                        const uint32_t *order, bool locks, const LockC *lc,
                                        uint64_t i, uint64_t e, uint64_t x,
                                        unsigned long long *keyPair) {
  LockInfo la, lb;
  const Ev a = decodeEv(A, A.keys[order[x]], A.vals[order[x]]);
  const SiteDev sa = A.sites[a.site];
  const LockC ca = locks && lc ? lc[x] : LockC{};
  bool laFull = false, laWide = false;
  const unsigned long long packed = (static_cast<unsigned long long>(i) << 32) | (x - i);
  for (uint64_t y = x + 1; y < e; ++y) {
    const int K = pairKey(A, L, order, locks, lc, a, sa, ca, y, la, laFull, laWide, lb);
    if (K >= 0 && keyPair[K] > packed)
      atomicMin(&keyPair[K], packed);
  }
}

// keyY[K] = the least y offset of key K's first row (one CTA per key).
__global__ void k_pair_first_y(DetectArgs A, LaunchDev L, const uint64_t *elemSorted,
                               const uint32_t *order, bool locks, const LockC *lc,
                               const unsigned long long *keyPair, unsigned long long *keyY) {
  const int K = blockIdx.x;
  const unsigned long long p = keyPair[K];
  if (p == ~0ull)
    return;
  const uint64_t i = p >> 32, x = i + (p & 0xffffffffull);
  const uint64_t elem = elemSorted[i];
  LockInfo la, lb;
  const Ev a = decodeEv(A, A.keys[order[x]], A.vals[order[x]]);
  const SiteDev sa = A.sites[a.site];
  const LockC ca = locks && lc ? lc[x] : LockC{};
  bool laFull = false, laWide = false;
  for (uint64_t y = x + 1 + threadIdx.x; y < A.n && elemSorted[y] == elem; y += blockDim.x)
    if (pairKey(A, L, order, locks, lc, a, sa, ca, y, la, laFull, laWide, lb) == K) {
      atomicMin(&keyY[K], static_cast<unsigned long long>(y - i));
      break;
    }
}

// Lock facts of every event (sorted position x), once: lockInfoOf per pair
// was the pairwise pass's dominant cost on lock kernels.
__global__ void k_lock_info(DetectArgs A, LaunchDev L, const uint32_t *order, LockC *out) {
  const uint64_t x = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= A.n || A.keys[order[x]] == A.kl.sentinel)
    return;
  const Ev a = decodeEv(A, A.keys[order[x]], A.vals[order[x]]);
  LockInfo li;
  unsigned flags = 0;
  lockInfoOf(L, a.thread, a.seq, li, flags);
  LockC c;
  // (wide: more than two entries, or a set past LockSet's capacity — the
  // pair pass then evaluates lockOrdered exactly, lockPairOrdered)
  if ((flags & kFlagLockSet) || !packSet(li.cs, c.cs) || !packSet(li.acq, c.acq) ||
      !packSet(li.rel, c.rel))
    c.cs[0] = kLockWide;
  out[x] = c;
}

__global__ void k_detect_pairwise(DetectArgs A, LaunchDev L, const uint64_t *elemSorted,
                                  const uint32_t *order, bool locks, const LockC *lc,
                                  unsigned long long *keyPair) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= A.n)
    return;
  const uint64_t elem = elemSorted[i];
  if (i > 0 && elemSorted[i - 1] == elem)
    return;
  if (elem == fieldMask(A.kl.bE))
    return; // chunk padding of PARALLEL records (never a valid element)
  uint64_t e = i + 1;
  while (e < A.n && elemSorted[e] == elem)
    ++e;
  if (e - i < 2)
    return;
  if (A.n >= kPairEventsMax) {
    atomicOr(&L.ctr->flags, static_cast<unsigned>(kFlagSegment));
    return;
  }
  if (A.nSites <= 64) { // no statically conflicting pair of the group's sites: skip
    uint64_t pres = 0;
    for (uint64_t x = i; x < e; ++x)
      pres |= 1ull << (A.vals[order[x]] >> A.kl.bS);
    bool any = false;
    for (uint64_t rem = pres; rem && !any; rem &= rem - 1) {
      const int s = __ffsll(static_cast<long long>(rem)) - 1;
      any = ((A.confInter[s] | A.confIntra[s]) & pres) != 0;
    }
    if (!any)
      return;
  }
  if (e - i > kPairBig && A.hotList) { // a large group: all CTAs of k_detect_pairwise_big
    const unsigned slot = atomicAdd(A.hotCount, 1u);
    if (slot < A.hotCap) {
      A.hotList[2 * slot] = static_cast<uint32_t>(i);
      A.hotList[2 * slot + 1] = static_cast<uint32_t>(e);
      return;
    }
  }
  for (uint64_t x = i; x < e; ++x)
    pairRow(A, L, order, locks, lc, i, e, x, keyPair);
}

// The large groups listed by k_detect_pairwise, tiled like an n-body pass:
// a work item is (row chunk, column tile) of one group, 256 events each;
// the tile is decoded once into shared memory and every thread tests its
// row event against it, so a hot element (a lock word, a histogram bin, a
// shared counter) is spread over the whole GPU and each pair costs shared
// memory reads only.  Work items of a group are numbered column-tile major
// (tile t holds t + 1 row chunks).
struct EvT {
  unsigned long long thread;
  uint32_t block, warp, bp, wp;
  int32_t seq, loc;
  uint16_t site;
  uint8_t kind, scope;
  uint32_t pad;
};

__device__ __forceinline__ EvT loadEvT(const DetectArgs &A, const uint32_t *order, uint64_t x) {
  const Ev a = decodeEv(A, A.keys[order[x]], A.vals[order[x]]);
  const SiteDev sd = A.sites[a.site];
  EvT t;
  t.thread = a.thread;
  t.block = static_cast<uint32_t>(a.block);
  t.warp = static_cast<uint32_t>(a.warp);
  t.bp = static_cast<uint32_t>(a.bp);
  t.wp = static_cast<uint32_t>(a.wp);
  t.seq = a.seq;
  t.loc = sd.loc;
  t.site = static_cast<uint16_t>(a.site);
  t.kind = sd.kind;
  t.scope = sd.scope;
  return t;
}

__global__ void __launch_bounds__(256) k_detect_pairwise_big(DetectArgs A, LaunchDev L,
                                                             const uint64_t *elemSorted,
                                                             const uint32_t *order, bool locks,
                                                             const LockC *lc,
                                                             unsigned long long *keyPair) {
  constexpr int kT = 256;
  __shared__ EvT tEv[kT];
  __shared__ LockC tLc[kT];
  const unsigned nBig = min(*A.hotCount, A.hotCap);
  const int tid = threadIdx.x;
  unsigned flags = 0;
  uint64_t base = 0; // work items of the groups before this one
  for (unsigned h = 0; h < nBig; ++h) {
    const uint64_t i = A.hotList[2 * h], e = A.hotList[2 * h + 1];
    const uint64_t g = e - i;
    const uint64_t nC = (g + kT - 1) / kT;
    const uint64_t items = nC * (nC + 1) / 2;
    uint64_t w = base + ((blockIdx.x + gridDim.x - base % gridDim.x) % gridDim.x);
    for (; w < base + items; w += gridDim.x) {
      const uint64_t local = w - base;
      uint64_t tb = static_cast<uint64_t>((sqrt(8.0 * static_cast<double>(local) + 1.0) - 1.0) / 2.0);
      while (tb * (tb + 1) / 2 > local)
        --tb;
      while ((tb + 1) * (tb + 2) / 2 <= local)
        ++tb;
      const uint64_t rb = local - tb * (tb + 1) / 2;
      const uint64_t y0 = i + tb * kT, x = i + rb * kT + tid;
      const int nTile = e - y0 < static_cast<uint64_t>(kT) ? static_cast<int>(e - y0) : kT;
      __syncthreads(); // previous item's tile fully read
      if (tid < nTile) {
        tEv[tid] = loadEvT(A, order, y0 + tid);
        if (locks)
          tLc[tid] = lc[y0 + tid];
      }
      __syncthreads();
      if (x >= e)
        continue;
      const EvT a = loadEvT(A, order, x);
      LockC ca{};
      if (locks)
        ca = lc[x];
      LockInfo la, lb;
      bool laFull = false, laWide = false;
      const int jStart = rb == tb ? tid + 1 : 0;
      for (int j = jStart; j < nTile; ++j) {
        const EvT &b = tEv[j];
        if (a.thread == b.thread)
          continue;
        if (a.kind == HGRD_SITE_LOAD && b.kind == HGRD_SITE_LOAD)
          continue;
        const bool sameBlock = a.block == b.block;
        if (a.kind == HGRD_SITE_ATOMIC && b.kind == HGRD_SITE_ATOMIC &&
            covers(a.scope, sameBlock) && covers(b.scope, sameBlock))
          continue;
        if (sameBlock && a.bp != b.bp)
          continue;
        const bool sameWarp = sameBlock && a.warp == b.warp;
        if (sameWarp && a.wp != b.wp)
          continue;
        if (locks) {
          bool ordered;
          const LockC &cb = tLc[j];
          if (ca.cs[0] != kLockWide && cb.cs[0] != kLockWide) {
            ordered = crossedC(ca.cs, cb.cs, sameBlock) || crossedC(ca.rel, cb.acq, sameBlock) ||
                      crossedC(cb.rel, ca.acq, sameBlock);
          } else {
            ordered = lockPairOrdered(L, a, b, sameBlock, la, laFull, laWide, lb);
          }
          if (ordered)
            continue;
        }
        const int kind = !sameBlock ? 0 : !sameWarp ? 1 : 2;
        int l0 = a.loc, l1 = b.loc;
        if (l1 < l0) {
          const int t = l0;
          l0 = l1;
          l1 = t;
        }
        const int K = (l0 * A.nLocs + l1) * 3 + kind;
        const unsigned long long packed = (static_cast<unsigned long long>(i) << 32) | (x - i);
        if (keyPair[K] > packed)
          atomicMin(&keyPair[K], packed);
      }
    }
    base += items;
  }
  if (flags)
    atomicOr(&L.ctr->flags, flags);
}

__global__ void k_decode_pairwise(DetectArgs A, const uint64_t *elemSorted,
                                  const uint32_t *order,
                                  const unsigned long long *keyPair,
                                  const unsigned long long *keyY, int nKeys,
                                  hgrd_gpu_race *races, Counters *ctr) {
  const int K = blockIdx.x * blockDim.x + threadIdx.x;
  if (K >= nKeys)
    return;
  const unsigned long long p = keyPair[K];
  if (p == ~0ull)
    return;
  const uint64_t s = p >> 32;
  const uint64_t x = s + (p & 0xffffffffull), y = s + keyY[K];
  const Ev a = decodeEv(A, A.keys[order[x]], A.vals[order[x]]);
  const Ev b = decodeEv(A, A.keys[order[y]], A.vals[order[y]]);
  const unsigned pos = atomicAdd(&ctr->nRaces, 1u);
  hgrd_gpu_race &o = races[pos];
  o.kind = K % 3;
  o.loc_a = (K / 3) / A.nLocs;
  o.loc_b = (K / 3) % A.nLocs;
  o.site_x = a.site;
  o.site_y = b.site;
  elementOf(A, elemSorted[s], o.handle, o.index);
  o.thread_x = static_cast<int64_t>(a.thread);
  o.thread_y = static_cast<int64_t>(b.thread);
  o.seq_x = a.seq;
  o.seq_y = b.seq;
}

} // namespace dev
} // namespace hgrdgpu

// ===========================================================================
// TEST INFRASTRUCTURE — the CPU oracle the GPU race-check stage is checked
// against.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
// leg load this (as oracle/_ref/libhgrd_oracle.so); the product library
// (libhgrd_gpu.so) never links or calls it.
//
// What it is: a line-by-line CPU restatement of the reference's thread
// expansion and conflict detection, executed over the same lowered launch
// descriptor (include/hgrd_gpu.h) the GPU receives:
//   * canonical thread loop bz,by,bx,tz,ty,tx       reference src/oracle.cpp:440-465
//   * per-thread statement semantics, events, seq,   :482-646
//     barrier phases, sync ops
//   * lockInfo / lockOrdered / scopeCovers           :650-728
//   * detectRaces pair loop and first-insert keys    :730-784
// extended with the witness pair (the (x, y) that first realises each key),
// which the reference computes but does not report.
//
// Parity pin: driven by the shared host front end, this library must equal
// the unmodified reference (oracle/_ref/libhgrd_ref.so) on every field of
// OracleResult for the bundled corpus, the reference's unit-test programs
// and the reference's soundness-fuzz programs (tests/test_oracle_pin.py).
// ===========================================================================
#include "hgrd_gpu.h"
#include "host.hpp"

#include <cstring>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

using namespace hgrdgpu;

namespace {

int64_t wadd(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}

// reference applyBinOp, src/oracle.cpp:179-209
int64_t applyBin(int op, int64_t l, int64_t r) {
  switch (op) {
  case HGRD_ADD:
    return wadd(l, r);
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

// reference SyncOp (:25-31) and Event (:33-48)
struct SyncOp {
  enum Kind { Cas, Exch, Fence } kind = Fence;
  int scope = HGRD_SCOPE_DEVICE;
  int handle = -1;
  int64_t index = 0;
  int seq = 0;
};
struct Event {
  int site = 0;
  int loc = 0;
  int handle = -1;
  int64_t index = 0;
  bool isWrite = false, isAtomic = false;
  int atomicScope = HGRD_SCOPE_NONE;
  int64_t blockLin = 0, threadLin = 0, warp = 0, blockPhase = 0, warpPhase = 0;
  int64_t thread = 0;
  int seq = 0;
};

struct LockFact {
  int handle;
  int64_t index;
  int scope;
};
struct EventLockInfo {
  std::vector<LockFact> acqBefore, relAfter, insideCs;
};

void maxScopeInsert(std::vector<LockFact> &facts, int h, int64_t idx, int scope) {
  for (auto &f : facts)
    if (f.handle == h && f.index == idx) {
      if (scope > f.scope)
        f.scope = scope;
      return;
    }
  facts.push_back(LockFact{h, idx, scope});
}
int narrower(int a, int b) { return a <= b ? a : b; }

// reference lockInfo, src/oracle.cpp:678-704
EventLockInfo lockInfo(const Event &e, const std::vector<SyncOp> &ops) {
  EventLockInfo info;
  for (const auto &fence : ops) {
    if (fence.kind != SyncOp::Fence)
      continue;
    for (const auto &cas : ops) {
      if (cas.kind != SyncOp::Cas || cas.seq >= fence.seq)
        continue;
      if (fence.seq < e.seq)
        maxScopeInsert(info.acqBefore, cas.handle, cas.index, narrower(cas.scope, fence.scope));
    }
    for (const auto &ex : ops) {
      if (ex.kind != SyncOp::Exch || ex.seq <= fence.seq)
        continue;
      if (fence.seq > e.seq)
        maxScopeInsert(info.relAfter, ex.handle, ex.index, narrower(ex.scope, fence.scope));
    }
  }
  for (const auto &a : info.acqBefore)
    for (const auto &r : info.relAfter)
      if (a.handle == r.handle && a.index == r.index)
        maxScopeInsert(info.insideCs, a.handle, a.index, narrower(a.scope, r.scope));
  return info;
}

// reference scopeCovers :706-708, lockOrdered :710-728
bool scopeCovers(int s, bool sameBlock) {
  return s == HGRD_SCOPE_DEVICE || (s == HGRD_SCOPE_BLOCK && sameBlock);
}
bool crossed(const std::vector<LockFact> &x, const std::vector<LockFact> &y, bool sameBlock) {
  for (const auto &a : x)
    for (const auto &b : y)
      if (a.handle == b.handle && a.index == b.index &&
          scopeCovers(narrower(a.scope, b.scope), sameBlock))
        return true;
  return false;
}
bool lockOrdered(const EventLockInfo &a, const EventLockInfo &b, bool sameBlock) {
  return crossed(a.insideCs, b.insideCs, sameBlock) ||
         crossed(a.relAfter, b.acqBefore, sameBlock) ||
         crossed(b.relAfter, a.acqBefore, sameBlock);
}

struct AbortRun {};

class CpuOracle final : public LaunchBackend {
public:
  int reset() override {
    bufs_.clear();
    return 0;
  }
  int alloc(int64_t elems, int32_t *handle) override {
    *handle = static_cast<int32_t>(bufs_.size());
    bufs_.emplace_back(static_cast<size_t>(elems), 0);
    return 0;
  }
  int write(int32_t h, int64_t off, int64_t n, const int64_t *src) override {
    std::memcpy(bufs_[h].data() + off, src, static_cast<size_t>(n) * 8);
    return 0;
  }
  int read(int32_t h, int64_t off, int64_t n, int64_t *dst) override {
    std::memcpy(dst, bufs_[h].data() + off, static_cast<size_t>(n) * 8);
    return 0;
  }
  std::string lastError() override { return err_; }
  std::vector<std::vector<int64_t>> &buffers() { return bufs_; }

  // The batched check restated launch by launch (each with its own
  // buffers), with the batch's contract: launches that run out of budget
  // come back HGRD_RESULT_UNCHECKED (the caller re-checks them in order), so
  // the speculative sweep logic runs on CPU exactly as on GPU.
  int checkBatch(const hgrd_gpu_batch_launch *B, uint32_t n, hgrd_gpu_result *R) override {
    std::vector<std::vector<int64_t>> saved = std::move(bufs_);
    for (uint32_t i = 0; i < n; ++i) {
      bufs_.clear();
      for (uint32_t h = 0; h < B[i].n_buffers; ++h) {
        bufs_.emplace_back(static_cast<size_t>(std::max<int64_t>(B[i].buffer_elems[h], 0)), 0);
        if (B[i].buffer_data && B[i].buffer_data[h])
          std::memcpy(bufs_.back().data(), B[i].buffer_data[h],
                      8 * static_cast<size_t>(B[i].buffer_elems[h]));
      }
      hgrd_gpu_result &r = R[i];
      int rc = checkLaunch(B[i].launch, r);
      if (rc < 0)
        return rc;
      if (r.aborted || (B[i].launch.flags & (HGRD_LAUNCH_SEQUENTIAL | HGRD_LAUNCH_PAIRWISE)))
        r.mode = HGRD_RESULT_UNCHECKED;
    }
    bufs_ = std::move(saved);
    return 0;
  }
  bool hasBatch() const override { return batch_; }
  bool batch_ = false;

  int checkLaunch(const hgrd_gpu_launch &L, hgrd_gpu_result &R) override {
    L_ = &L;
    R.n_races = 0;
    R.n_traps = 0;
    R.n_traps_total = 0;
    R.steps = 0;
    R.instances = 0;
    R.records = 0;
    R.aborted = 0;
    R.abort_stmt = -1;
    R.mode = L.flags;
    R.device_ms = 0;
    R_ = &R;
    steps_ = 0;
    events_.clear();
    syncOps_.clear();
    written_.clear();
    for (uint32_t s = 0; s < L.n_sites; ++s)
      if (L.sites[s].kind != HGRD_SITE_LOAD && handleOf(static_cast<int>(s)) >= 0)
        written_.insert(handleOf(static_cast<int>(s)));
    bool aborted = false;
    try {
      expand();
    } catch (const AbortRun &) {
      aborted = true;
    }
    R.steps = steps_;
    R.instances = events_.size(); // executed up to the end or the abort
    for (const auto &e : events_)
      if (written_.count(e.handle))
        ++R.records;
    if (aborted) {
      R.aborted = 1;
      return 0; // the in-flight launch contributes no races (:71-76)
    }
    return detectRaces();
  }

private:
  int handleOf(int site) const {
    int p = L_->sites[site].param;
    return p >= 0 && static_cast<uint32_t>(p) < L_->n_params ? L_->param_handle[p] : -1;
  }

  void trapAt(int site, int kind, int64_t thread) {
    if (R_->n_traps < R_->trap_cap)
      R_->traps[R_->n_traps++] = hgrd_gpu_trap{site, kind, thread};
    ++R_->n_traps_total;
  }

  // reference execLaunch thread loop, src/oracle.cpp:440-465
  void expand() {
    const int64_t *g = L_->grid, *b = L_->block;
    int64_t thread = 0;
    for (int64_t bz = 0; bz < g[2]; ++bz)
      for (int64_t by = 0; by < g[1]; ++by)
        for (int64_t bx = 0; bx < g[0]; ++bx)
          for (int64_t tz = 0; tz < b[2]; ++tz)
            for (int64_t ty = 0; ty < b[1]; ++ty)
              for (int64_t tx = 0; tx < b[0]; ++tx) {
                int64_t bi[4][3] = {{tx, ty, tz}, {bx, by, bz}, {b[0], b[1], b[2]}, {g[0], g[1], g[2]}};
                int64_t blockLin = bx + by * g[0] + bz * g[0] * g[1];
                int64_t threadLin = tx + ty * b[0] + tz * b[0] * b[1];
                syncOps_.emplace_back();
                runThread(bi, blockLin, threadLin, threadLin / L_->warp_size, thread);
                ++thread;
              }
  }

  // reference runThreadStmt, src/oracle.cpp:560-646, over lowered code
  void runThread(const int64_t (&bi)[4][3], int64_t blockLin, int64_t threadLin,
                 int64_t warp, int64_t thread) {
    std::vector<int64_t> r(L_->reg_init, L_->reg_init + L_->n_regs);
    int64_t blockPhase = 0, warpPhase = 0;
    int seq = 0;
    std::vector<SyncOp> &ops = syncOps_.back();
    auto record = [&](int site, int h, int64_t idx, bool w, bool at, int scope) {
      Event e;
      e.site = site;
      e.loc = L_->sites[site].loc;
      e.handle = h;
      e.index = idx;
      e.isWrite = w;
      e.isAtomic = at;
      e.atomicScope = scope;
      e.blockLin = blockLin;
      e.threadLin = threadLin;
      e.warp = warp;
      e.blockPhase = blockPhase;
      e.warpPhase = warpPhase;
      e.thread = thread;
      e.seq = seq++;
      events_.push_back(e);
    };
    // reference checkBounds, :508-519
    auto inBounds = [&](int site, int h, int64_t idx) {
      if (h < 0) {
        trapAt(site, HGRD_TRAP_UNALLOCATED, thread);
        return false;
      }
      if (idx < 0 || idx >= static_cast<int64_t>(bufs_[h].size())) {
        trapAt(site, HGRD_TRAP_OOB, thread);
        return false;
      }
      return true;
    };
    for (uint32_t pc = 0; pc < L_->n_code;) {
      const hgrd_gpu_insn &I = L_->code[pc];
      switch (I.op) {
      case HGRD_OP_END:
        return;
      case HGRD_OP_STEP:
        if (++steps_ > L_->step_budget) {
          R_->abort_stmt = static_cast<int32_t>(I.imm);
          throw AbortRun{};
        }
        break;
      case HGRD_OP_CONST:
        r[I.a] = I.imm;
        break;
      case HGRD_OP_MOV:
        r[I.a] = r[I.b];
        break;
      case HGRD_OP_BUILTIN:
        r[I.a] = bi[I.sub / 3][I.sub % 3];
        break;
      case HGRD_OP_BIN:
        r[I.a] = applyBin(I.sub, r[I.b], r[I.c]);
        break;
      case HGRD_OP_LOAD: { // deviceLoad :542-549
        int site = static_cast<int>(I.imm);
        int h = handleOf(site);
        int64_t idx = r[I.b];
        if (!inBounds(site, h, idx)) {
          r[I.a] = 0;
          break;
        }
        record(site, h, idx, false, false, HGRD_SCOPE_NONE);
        r[I.a] = bufs_[h][idx];
        break;
      }
      case HGRD_OP_STORE: { // :567-577
        int site = static_cast<int>(I.imm);
        int h = handleOf(site);
        int64_t idx = r[I.a], val = r[I.b];
        if (!inBounds(site, h, idx))
          break;
        record(site, h, idx, true, false, HGRD_SCOPE_NONE);
        bufs_[h][idx] = val;
        break;
      }
      case HGRD_OP_ATOMIC: { // :578-605
        int site = static_cast<int>(I.imm);
        const hgrd_gpu_site &S = L_->sites[site];
        int h = handleOf(site);
        int64_t idx = r[I.a], val = r[I.b], cmp = r[I.c];
        if (!inBounds(site, h, idx))
          break;
        record(site, h, idx, true, true, S.scope);
        int64_t old = bufs_[h][idx];
        if (S.atomic_op == HGRD_ATOMIC_CAS) {
          if (old == cmp)
            bufs_[h][idx] = val;
          ops.push_back(SyncOp{SyncOp::Cas, S.scope, h, idx, seq - 1});
        } else if (S.atomic_op == HGRD_ATOMIC_EXCH) {
          bufs_[h][idx] = val;
          ops.push_back(SyncOp{SyncOp::Exch, S.scope, h, idx, seq - 1});
        } else {
          bufs_[h][idx] = wadd(old, val);
        }
        break;
      }
      case HGRD_OP_SYNCTHREADS: // :606-614
        ++blockPhase;
        ++warpPhase;
        break;
      case HGRD_OP_SYNCWARP:
        ++warpPhase;
        break;
      case HGRD_OP_FENCE: // :615-620
        ops.push_back(SyncOp{SyncOp::Fence, I.sub, -1, 0, seq++});
        break;
      case HGRD_OP_JZ:
        if (r[I.a] == 0) {
          pc = static_cast<uint32_t>(I.imm);
          continue;
        }
        break;
      case HGRD_OP_JMP:
        pc = static_cast<uint32_t>(I.imm);
        continue;
      }
      ++pc;
    }
  }

  // reference detectRaces, src/oracle.cpp:730-784 (+ witness)
  int detectRaces() {
    std::map<std::pair<int, int64_t>, std::vector<size_t>> byElement;
    for (size_t i = 0; i < events_.size(); ++i)
      byElement[{events_[i].handle, events_[i].index}].push_back(i);
    std::vector<EventLockInfo> locks(events_.size());
    std::vector<bool> have(events_.size(), false);
    auto lockOf = [&](size_t i) -> const EventLockInfo & {
      if (!have[i]) {
        locks[i] = lockInfo(events_[i], syncOps_[static_cast<size_t>(events_[i].thread)]);
        have[i] = true;
      }
      return locks[i];
    };
    std::set<std::tuple<int, int, int>> seen;
    for (const auto &[elem, idxs] : byElement) {
      for (size_t x = 0; x < idxs.size(); ++x) {
        for (size_t y = x + 1; y < idxs.size(); ++y) {
          const Event &a = events_[idxs[x]];
          const Event &b = events_[idxs[y]];
          if (a.thread == b.thread)
            continue;
          if (!a.isWrite && !b.isWrite)
            continue;
          bool sameBlock = a.blockLin == b.blockLin;
          if (a.isAtomic && b.isAtomic && scopeCovers(a.atomicScope, sameBlock) &&
              scopeCovers(b.atomicScope, sameBlock))
            continue;
          if (sameBlock && a.blockPhase != b.blockPhase)
            continue;
          bool sameWarp = sameBlock && a.warp == b.warp;
          if (sameWarp && a.warpPhase != b.warpPhase)
            continue;
          if (lockOrdered(lockOf(idxs[x]), lockOf(idxs[y]), sameBlock))
            continue;
          int kind = !sameBlock ? 0 : !sameWarp ? 1 : 2;
          int la = a.loc, lb = b.loc;
          if (lb < la)
            std::swap(la, lb);
          if (!seen.insert({la, lb, kind}).second)
            continue;
          if (R_->n_races >= R_->race_cap)
            return HGRD_GPU_E2BIG;
          hgrd_gpu_race &o = R_->races[R_->n_races++];
          o.loc_a = la;
          o.loc_b = lb;
          o.kind = kind;
          o.site_x = a.site;
          o.site_y = b.site;
          o.handle = a.handle;
          o.index = a.index;
          o.thread_x = a.thread;
          o.thread_y = b.thread;
          o.seq_x = a.seq;
          o.seq_y = b.seq;
        }
      }
    }
    return 0;
  }

  std::vector<std::vector<int64_t>> bufs_;
  const hgrd_gpu_launch *L_ = nullptr;
  hgrd_gpu_result *R_ = nullptr;
  int64_t steps_ = 0;
  std::vector<Event> events_;
  std::vector<std::vector<SyncOp>> syncOps_;
  std::set<int> written_;
  std::string err_;
};

char *dup(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

} // namespace

extern "C" {

void hgrd_oracle_free(char *p) { std::free(p); }

int hgrd_oracle_run_concrete_json(const char *src, const char *file,
                                  const char *cfg, char **out) {
  CpuOracle be;
  std::string s;
  int rc = runConcreteJson(be, src, file, cfg, s);
  *out = dup(s);
  return rc;
}

int hgrd_oracle_enumerate_verdict_json(const char *src, const char *file,
                                       const char *caps, char **out) {
  CpuOracle be;
  std::string s;
  int rc = enumerateVerdictJson(be, src, file, caps, s);
  *out = dup(s);
  return rc;
}

// enumerateVerdict through the speculative batched sweep (the product's
// sweep path) with the restatement as its batch backend.
int hgrd_oracle_enumerate_verdict_batched_json(const char *src, const char *file,
                                               const char *caps, char **out) {
  CpuOracle be;
  be.batch_ = true;
  std::string s;
  int rc = enumerateVerdictJson(be, src, file, caps, s);
  *out = dup(s);
  return rc;
}

// Many sweeps at once through the product's sweepManyJson (batched when
// `batched` is set) with the restatement as backend.
int hgrd_oracle_enumerate_verdict_many_json(const char *jobs, int rank, int world, int batched,
                                            char **out) {
  CpuOracle be;
  be.batch_ = batched != 0;
  std::string s;
  int rc = sweepManyJson([&](int i) -> LaunchBackend * { return i == 0 ? &be : nullptr; }, 1,
                         jobs, rank, world, s);
  *out = dup(s);
  return rc;
}

int hgrd_oracle_sweep_shard_json(const char *src, const char *file, const char *caps,
                                 int rank, int world, char **out) {
  CpuOracle be;
  std::string s;
  int rc = sweepShardJsonRun(be, src, file, caps, rank, world, s);
  *out = dup(s);
  return rc;
}

// Launch-level oracle for descriptors built outside the host interpreter
// (bench workloads): buffers are given by contents, then one check runs.
int hgrd_oracle_check_launch(const hgrd_gpu_launch *launch,
                             const int64_t *const *buffers, const int64_t *sizes,
                             int32_t n_buffers, hgrd_gpu_result *result) {
  CpuOracle be;
  for (int32_t i = 0; i < n_buffers; ++i) {
    int32_t h;
    be.alloc(sizes[i], &h);
    if (buffers && buffers[i])
      be.write(h, 0, sizes[i], buffers[i]);
  }
  return be.checkLaunch(*launch, *result);
}

} // extern "C"

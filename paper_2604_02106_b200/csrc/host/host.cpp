// Host interpreter of the race-check stage.  Mirrors the reference's
// Interpreter (reference src/oracle.cpp:55-437) so that every launch
// reaches the backend with exactly the parameters, dimensions, buffer
// contents, step budget and trap slots the reference would use, and folds
// the backend's per-launch result back the way the reference does
// (first-insert dedup across launches :776-780, final sort :76).
//
// Memory model.  The reference runs MiniCU threads to completion one after
// another (:440-465), so loads observe earlier threads' stores.  A launch is
// checked in one of two modes (chosen here, executed by the backend):
//  * PARALLEL: no loaded value that can reach an index / condition / loop
//    bound (LoweredKernel::siteValueNeeded) reads a buffer the launch
//    writes, so every instance's accesses are independent of the order
//    threads run in; the value-needed loads read the launch-entry buffers.
//    The launch's own stores are not materialised: its written buffers
//    become "stale".
//  * SEQUENTIAL: instances run in canonical order with memory effects.
// A stale buffer read by the host, or read by a later launch where the
// value matters, restarts the run in conservative mode, where every launch
// that writes memory runs SEQUENTIAL, so buffers are always exact.
#include "host.hpp"
#include "parallel_for.hpp"

#include <atomic>
#include <thread>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <tuple>

namespace hgrdgpu {

const LoweredKernel &CompiledProgram::kernel(const Function *k) {
  auto it = kernels.find(k);
  if (it == kernels.end())
    it = kernels.emplace(k, lowerKernel(*k)).first;
  return it->second;
}

// ---------------------------------------------------------------------------
// static scans (reference src/oracle.cpp:86-123 and :805-861)

bool hasIndirectIndexing(const Program &p) {
  bool found = false;
  std::function<void(const Expr &, bool)> scanE = [&](const Expr &e, bool inIndex) {
    if (e.kind == EK::Load) {
      if (inIndex)
        found = true;
      scanE(*e.index, true);
    } else if (e.kind == EK::Binary) {
      scanE(*e.lhs, inIndex);
      scanE(*e.rhs, inIndex);
    }
  };
  std::function<void(const Body &)> scanB = [&](const Body &b) {
    for (const auto &s : b) {
      switch (s->kind) {
      case SK::Store:
        scanE(*s->index, true);
        scanE(*s->value, false);
        break;
      case SK::Atomic:
        scanE(*s->index, true);
        break;
      case SK::Assign:
        if (s->value)
          scanE(*s->value, false);
        break;
      case SK::If:
        scanB(s->body);
        scanB(s->elseBody);
        break;
      case SK::For:
        scanB(s->body);
        break;
      default:
        break;
      }
    }
  };
  for (const auto &k : p.kernels)
    scanB(k.body);
  return found;
}

int countInputs(const Program &p) {
  int n = 0;
  std::function<void(const Expr &)> scanE = [&](const Expr &e) {
    if (e.kind == EK::Input)
      ++n;
    else if (e.kind == EK::Binary) {
      scanE(*e.lhs);
      scanE(*e.rhs);
    } else if (e.kind == EK::Load) {
      scanE(*e.index);
    }
  };
  std::function<void(const Body &)> scanB = [&](const Body &b) {
    for (const auto &sp : b) {
      const Stmt &s = *sp;
      switch (s.kind) {
      case SK::Assign:
        if (s.value)
          scanE(*s.value);
        break;
      case SK::Store:
        scanE(*s.index);
        scanE(*s.value);
        break;
      case SK::Assert:
        scanE(*s.cond);
        break;
      case SK::Alloc:
        scanE(*s.width);
        if (s.height)
          scanE(*s.height);
        break;
      case SK::If:
        scanE(*s.cond);
        scanB(s.body);
        scanB(s.elseBody);
        break;
      case SK::For:
        scanE(*s.init);
        scanE(*s.bound);
        scanB(s.body);
        break;
      case SK::Launch:
        for (const auto &d : s.grid)
          scanE(*d);
        for (const auto &d : s.block)
          scanE(*d);
        for (const auto &a : s.args)
          scanE(*a);
        break;
      case SK::Call:
        for (const auto &a : s.args)
          scanE(*a);
        break;
      case SK::Return:
        if (s.value)
          scanE(*s.value);
        break;
      default:
        break;
      }
    }
  };
  for (const auto &f : p.hosts)
    scanB(f.body);
  return n;
}

std::unique_ptr<CompiledProgram> compileProgram(std::unique_ptr<Program> p) {
  auto cp = std::make_unique<CompiledProgram>();
  cp->indirectIndexing = hasIndirectIndexing(*p);
  cp->inputs = countInputs(*p);
  cp->program = std::move(p);
  return cp;
}

const char *raceKindName(int kind) {
  switch (kind) {
  case 0:
    return "INTER-BLOCK";
  case 1:
    return "INTRA-BLOCK";
  case 2:
    return "INTRA-WARP";
  }
  return "?";
}

// ---------------------------------------------------------------------------

namespace {

// names assigned anywhere in a body (reference src/host_facts.cpp:101-121)
std::set<std::string> assignedNames(const Body &b) {
  std::set<std::string> names;
  std::function<void(const Body &)> walk = [&](const Body &body) {
    for (const auto &s : body) {
      if (s->kind == SK::Assign) {
        names.insert(s->name);
      } else if (s->kind == SK::If) {
        walk(s->body);
        walk(s->elseBody);
      } else if (s->kind == SK::For) {
        names.insert(s->aux);
        walk(s->body);
      } else if (s->kind == SK::Alloc) {
        names.insert(s->name);
        if (!s->aux.empty())
          names.insert(s->aux);
      }
    }
  };
  walk(b);
  return names;
}

int64_t wrapAdd(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}
int64_t wrapSub(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) - static_cast<uint64_t>(b));
}
int64_t wrapMul(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) * static_cast<uint64_t>(b));
}

// reference applyBinOp, src/oracle.cpp:179-209 (wrapping int64)
int64_t binop(Bin op, int64_t l, int64_t r) {
  switch (op) {
  case Bin::Add:
    return wrapAdd(l, r);
  case Bin::Sub:
    return wrapSub(l, r);
  case Bin::Mul:
    return wrapMul(l, r);
  case Bin::Div:
    return r == 0 ? 0 : (r == -1 ? wrapSub(0, l) : l / r);
  case Bin::Mod:
    return r == 0 || r == -1 ? 0 : l % r;
  case Bin::Lt:
    return l < r;
  case Bin::Le:
    return l <= r;
  case Bin::Gt:
    return l > r;
  case Bin::Ge:
    return l >= r;
  case Bin::Eq:
    return l == r;
  case Bin::Ne:
    return l != r;
  case Bin::And:
    return (l != 0 && r != 0) ? 1 : 0;
  case Bin::Or:
    return (l != 0 || r != 0) ? 1 : 0;
  }
  return 0;
}

struct Abort {};            // TrapAbort / assert stop
struct NeedConservative {}; // a stale buffer's value was needed
struct BackendFail {
  int code;
  std::string msg;
};

struct SpecFail {}; // a speculative host run needs what only a real check gives

// A launch of a speculative host run (enumerateVerdictBatched): everything
// hgrd_gpu_check_batch needs, kept until the batch is checked.
struct PendingLaunch {
  const LoweredKernel *lk = nullptr;
  int launchIndex = 0;
  std::array<int64_t, 3> grid{}, block{};
  int64_t warpSize = 32, budget = 0;
  size_t trapPos = 0; // host traps recorded before the launch
  std::vector<int64_t> regInit;
  std::vector<int32_t> paramHandle;
  std::vector<int64_t> bufElems;             // every buffer of the run
  std::vector<std::vector<int64_t>> bufData; // value-needed buffers' contents (empty: zeros)
};

using SeenKeys = std::set<std::tuple<int, int, int, int, int>>;

void decomposeThread(int64_t thread, const std::array<int64_t, 3> &grid,
                     const std::array<int64_t, 3> &block, int64_t tpb, int64_t (&b)[3],
                     int64_t (&t)[3]) {
  int64_t bl = thread / tpb, tl = thread % tpb;
  b[0] = bl % grid[0];
  b[1] = (bl / grid[0]) % grid[1];
  b[2] = bl / (grid[0] * grid[1]);
  t[0] = tl % block[0];
  t[1] = (tl / block[0]) % block[1];
  t[2] = tl / (block[0] * block[1]);
}

// detectRaces' tail (reference :766-780): a launch's races in the run's
// report, first insert of (locA, locB, kind) across the run's launches.
void mergeLaunchRaces(RunResult &res, SeenKeys &seen, const LoweredKernel &lk,
                      const std::array<int64_t, 3> &grid, const std::array<int64_t, 3> &block,
                      const hgrd_gpu_race *races, uint32_t n, int launchIndex) {
  const int64_t tpb = block[0] * block[1] * block[2];
  for (uint32_t i = 0; i < n; ++i) {
    const hgrd_gpu_race &g = races[i];
    Race r;
    r.locA = lk.locs[static_cast<size_t>(g.loc_a)];
    r.locB = lk.locs[static_cast<size_t>(g.loc_b)];
    r.kind = g.kind;
    r.array = lk.siteArray[static_cast<size_t>(g.site_x)];
    r.address = g.index;
    r.launch = launchIndex;
    r.threadX = g.thread_x;
    r.threadY = g.thread_y;
    r.seqX = g.seq_x;
    r.seqY = g.seq_y;
    decomposeThread(g.thread_x, grid, block, tpb, r.blockX, r.tidX);
    decomposeThread(g.thread_y, grid, block, tpb, r.blockY, r.tidY);
    auto key = std::make_tuple(r.locA.line, r.locA.col, r.locB.line, r.locB.col, r.kind);
    if (seen.insert(key).second)
      res.races.push_back(std::move(r));
  }
}

// reference operator< (src/oracle.cpp:9-19): the run's final order (:76)
void sortRaces(std::vector<Race> &races) {
  std::sort(races.begin(), races.end(), [](const Race &a, const Race &b) {
    if (!(a.locA == b.locA))
      return a.locA < b.locA;
    if (!(a.locB == b.locB))
      return a.locB < b.locB;
    if (a.kind != b.kind)
      return a.kind < b.kind;
    if (a.array != b.array)
      return a.array < b.array;
    return a.address < b.address;
  });
}

class HostRun {
public:
  // lean: a sweep's run — only the races count (enumerateVerdict,
  // :863-903), so launch records keep no defValues
  HostRun(CompiledProgram &cp, const ExecConfig &cfg, LaunchBackend &be,
          bool conservative, std::vector<PendingLaunch> *spec = nullptr, bool lean = false)
      : cp_(cp), prog_(*cp.program), cfg_(cfg), be_(be),
        conservative_(conservative), spec_(spec), lean_(lean) {}

  bool budgetAborted() const { return budgetAbort_; }
  int64_t steps() const { return steps_; }

  RunResult run() {
    res_.indirectIndexing = cp_.indirectIndexing;
    int rc = be_.reset();
    if (rc < 0)
      return fail(rc, be_.lastError());
    const Function *entry = prog_.findHost("main");
    if (!entry) {
      res_.traps.push_back("missing entry function");
      return std::move(res_);
    }
    Frame f;
    for (const auto &p : entry->params) {
      if (p.type == VarType::Int) {
        f.scalars[p.name] = 0;
        setDef(-entry->loc.line, 0, p.name, 0);
      } else {
        f.arrays[p.name] = -1;
      }
    }
    try {
      execBody(entry->body, f);
    } catch (const Abort &) {
    } catch (const BackendFail &bf) {
      return fail(bf.code, bf.msg);
    }
    sortRaces(res_.races);
    return std::move(res_);
  }

private:
  struct Frame {
    std::map<std::string, int64_t> scalars;
    std::map<std::string, int> arrays;
  };
  struct Buf {
    int64_t elems = 0;
    std::vector<int64_t> host; // lazily materialised mirror
    bool hostValid = true;     // mirror (or implicit zeros) == device
    int64_t dirtyLo = INT64_MAX, dirtyHi = -1;
    bool stale = false;        // device content not exact (PARALLEL writes)
  };

  RunResult fail(int code, const std::string &msg) {
    res_.error = code;
    res_.errorMessage = msg;
    return std::move(res_);
  }

  void setDef(int site, int aux, const std::string &name, int64_t v) {
    if (lean_)
      return;
    auto key = std::make_pair(site, aux);
    auto it = defs_.find(key);
    if (it == defs_.end())
      defs_.emplace(key, DefVal{name, v});
    else
      it->second.value = v; // DefKey identity ignores the name (host_facts.hpp:26-33)
  }

  void trap(const Loc &loc, const std::string &msg) {
    if (res_.traps.size() < 256)
      res_.traps.push_back(prog_.file + ":" + std::to_string(loc.line) + ": " + msg);
  }

  void step(const Loc &loc) {
    if (++steps_ > cfg_.maxSteps) {
      trap(loc, "step budget exhausted");
      budgetAbort_ = true;
      throw Abort{};
    }
  }

  void ensureHost(Buf &b, int h) {
    if (b.host.empty() && b.elems > 0 && b.hostValid) {
      b.host.assign(static_cast<size_t>(b.elems), 0);
      return;
    }
    if (!b.hostValid) {
      if (b.host.size() != static_cast<size_t>(b.elems))
        b.host.assign(static_cast<size_t>(b.elems), 0);
      int rc = be_.read(h, 0, b.elems, b.host.data());
      if (rc < 0)
        throw BackendFail{rc, be_.lastError()};
      b.hostValid = true;
    }
  }

  int64_t evalHost(const Expr &e, Frame &f) {
    switch (e.kind) {
    case EK::Lit:
      return e.value;
    case EK::Var: {
      auto it = f.scalars.find(e.name);
      return it == f.scalars.end() ? 0 : it->second;
    }
    case EK::Input: {
      int64_t v = 0;
      if (inputCursor_ < cfg_.inputs.size())
        v = cfg_.inputs[inputCursor_++];
      else
        trap(e.loc, "input exhausted; __input() defaults to 0");
      setDef(e.id, 0, "__input", v);
      return v;
    }
    case EK::Load: {
      auto it = f.arrays.find(e.name);
      int64_t idx = evalHost(*e.index, f);
      if (it == f.arrays.end() || it->second < 0) {
        trap(e.loc, "read from unallocated array " + e.name);
        return 0;
      }
      Buf &b = bufs_[it->second];
      if (idx < 0 || idx >= b.elems) {
        trap(e.loc, "host read out of bounds on " + e.name);
        return 0;
      }
      if (b.stale)
        throw NeedConservative{};
      ensureHost(b, it->second);
      return b.host[static_cast<size_t>(idx)];
    }
    case EK::Binary: {
      int64_t l = evalHost(*e.lhs, f); // host: left to right (:174-175)
      int64_t r = evalHost(*e.rhs, f);
      return binop(e.op, l, r);
    }
    default:
      return 0;
    }
  }

  bool execBody(const Body &b, Frame &f) {
    for (const auto &s : b)
      if (execStmt(*s, f))
        return true;
    return false;
  }

  void syncJoin(const Stmt &s, Frame &f) {
    std::set<std::string> names = assignedNames(s.body);
    std::set<std::string> e = assignedNames(s.elseBody);
    names.insert(e.begin(), e.end());
    for (const auto &n : names) {
      auto it = f.scalars.find(n);
      if (it != f.scalars.end())
        setDef(s.id, 3, n, it->second);
    }
  }

  bool execStmt(const Stmt &s, Frame &f) {
    step(s.loc);
    switch (s.kind) {
    case SK::Assign: {
      if (s.isDecl && isArray(s.declType)) {
        f.arrays[s.name] = -1;
        return false;
      }
      int64_t v = s.value ? evalHost(*s.value, f) : 0;
      f.scalars[s.name] = v;
      setDef(s.id, 0, s.name, v);
      return false;
    }
    case SK::Store: {
      int64_t idx = evalHost(*s.index, f);
      int64_t val = evalHost(*s.value, f);
      auto it = f.arrays.find(s.name);
      if (it == f.arrays.end() || it->second < 0) {
        trap(s.loc, "write to unallocated array " + s.name);
        return false;
      }
      Buf &b = bufs_[it->second];
      if (idx < 0 || idx >= b.elems) {
        trap(s.loc, "host write out of bounds on " + s.name);
        return false;
      }
      ensureHost(b, it->second);
      b.host[static_cast<size_t>(idx)] = val;
      b.dirtyLo = std::min(b.dirtyLo, idx);
      b.dirtyHi = std::max(b.dirtyHi, idx);
      return false;
    }
    case SK::Assert:
      if (evalHost(*s.cond, f) == 0) {
        res_.assertStopped = true;
        throw Abort{};
      }
      return false;
    case SK::Alloc: {
      int64_t elems = 0;
      if (!s.pitch) {
        elems = evalHost(*s.width, f);
      } else {
        int64_t w = evalHost(*s.width, f);
        int64_t h = evalHost(*s.height, f);
        if (w <= 0 || h <= 0) {
          trap(s.loc, "cudaMallocPitch with non-positive extent");
          f.scalars[s.aux] = 0;
          setDef(s.id, 1, s.aux, 0);
          f.arrays[s.name] = -1;
          return false;
        }
        int64_t pitch = wrapMul((w + 3) / 4, 4); // reference :271-275
        f.scalars[s.aux] = pitch;
        setDef(s.id, 1, s.aux, pitch);
        elems = wrapMul(pitch, h);
      }
      if (elems <= 0 || elems > cfg_.maxArrayElems) {
        trap(s.loc, "allocation size out of range for " + s.name);
        f.arrays[s.name] = -1;
        return false;
      }
      int32_t handle = -1;
      int rc = be_.alloc(elems, &handle);
      if (rc < 0)
        throw BackendFail{rc, be_.lastError()};
      if (handle != static_cast<int32_t>(bufs_.size()))
        throw BackendFail{HGRD_GPU_EINVAL, "backend handle order"};
      Buf b;
      b.elems = elems;
      bufs_.push_back(std::move(b));
      f.arrays[s.name] = handle;
      return false;
    }
    case SK::If: {
      bool taken = evalHost(*s.cond, f) != 0;
      bool returned = execBody(taken ? s.body : s.elseBody, f);
      syncJoin(s, f);
      return returned;
    }
    case SK::For: {
      int64_t i = evalHost(*s.init, f);
      std::set<std::string> assigned = assignedNames(s.body);
      assigned.erase(s.aux);
      for (;;) {
        step(s.loc);
        int64_t bound = evalHost(*s.bound, f);
        bool cont = s.inclusive ? (i <= bound) : (i < bound);
        if (!cont)
          break;
        f.scalars[s.aux] = i;
        setDef(s.id, 0, s.aux, i);
        for (const auto &n : assigned) {
          auto it = f.scalars.find(n);
          if (it != f.scalars.end())
            setDef(s.id, 1, n, it->second);
        }
        if (execBody(s.body, f))
          return true;
        i = wrapAdd(i, s.step);
      }
      f.scalars[s.aux] = i;
      setDef(s.id, 2, s.aux, i);
      for (const auto &n : assigned) {
        auto it = f.scalars.find(n);
        if (it != f.scalars.end())
          setDef(s.id, 2, n, it->second);
      }
      return false;
    }
    case SK::Launch:
      execLaunch(s, f);
      return false;
    case SK::Call: {
      const Function *callee = prog_.findHost(s.name);
      if (!callee) {
        trap(s.loc, "call to unknown function");
        return false;
      }
      if (callDepth_ > 64) {
        trap(s.loc, "host call depth exceeded");
        throw Abort{};
      }
      Frame cf;
      for (size_t i = 0; i < callee->params.size(); ++i) {
        const Param &p = callee->params[i];
        if (p.type == VarType::Int) {
          int64_t v = evalHost(*s.args[i], f);
          cf.scalars[p.name] = v;
          setDef(s.id, static_cast<int>(i) + 10, p.name, v);
        } else {
          int handle = -1;
          if (s.args[i]->kind == EK::Var) {
            auto it = f.arrays.find(s.args[i]->name);
            if (it != f.arrays.end())
              handle = it->second;
          }
          cf.arrays[p.name] = handle;
        }
      }
      ++callDepth_;
      execBody(callee->body, cf);
      --callDepth_;
      return false;
    }
    case SK::Return:
      return true;
    default:
      return false;
    }
  }

  // reference Interpreter::execLaunch, src/oracle.cpp:378-467: the host part
  // runs here; the thread loop and detectRaces run in the backend.
  void execLaunch(const Stmt &s, Frame &f) {
    const Function *kernel = prog_.findKernel(s.name);
    if (!kernel) {
      trap(s.loc, "launch of unknown kernel");
      return;
    }
    std::array<int64_t, 3> grid{}, block{};
    for (int d = 0; d < 3; ++d) {
      grid[d] = evalHost(*s.grid[d], f);
      block[d] = evalHost(*s.block[d], f);
    }
    for (int d = 0; d < 3; ++d) {
      if (grid[d] <= 0 || block[d] <= 0) {
        trap(s.loc, "non-positive launch dimension");
        ++res_.launchesSkipped;
        return;
      }
    }
    bool fits = true;
    for (int d = 0; d < 3; ++d)
      fits = fits && grid[d] <= cfg_.gridCap[d] && block[d] <= cfg_.blockCap[d];
    int64_t tpb = wrapMul(wrapMul(block[0], block[1]), block[2]);
    int64_t total = wrapMul(wrapMul(wrapMul(grid[0], grid[1]), grid[2]), tpb);
    if (!fits || total > cfg_.maxThreads) {
      ++res_.launchesSkipped;
      return;
    }
    LaunchRec rec;
    rec.site = s.id;
    rec.loc = s.loc;
    rec.grid = grid;
    rec.block = block;
    rec.defValues = defs_;
    std::vector<int32_t> paramHandle(kernel->params.size(), -1);
    std::vector<int64_t> scalarVal(kernel->params.size(), 0);
    for (size_t i = 0; i < kernel->params.size(); ++i) {
      const Param &p = kernel->params[i];
      if (p.type == VarType::Int) {
        int64_t v = evalHost(*s.args[i], f);
        scalarVal[i] = v;
        rec.scalarArgs.push_back(v);
        rec.isScalar.push_back(true);
      } else {
        int handle = -1;
        if (s.args[i]->kind == EK::Var) {
          auto it = f.arrays.find(s.args[i]->name);
          if (it != f.arrays.end())
            handle = it->second;
        }
        paramHandle[i] = handle;
        rec.scalarArgs.push_back(-1);
        rec.isScalar.push_back(false);
      }
    }
    res_.launchRecords.push_back(std::move(rec));
    ++res_.launchesRun;
    const int launchIndex = static_cast<int>(res_.launchRecords.size() - 1);
    checkLaunch(cp_.kernel(kernel), grid, block, paramHandle, scalarVal, launchIndex);
  }

  void checkLaunch(const LoweredKernel &lk, const std::array<int64_t, 3> &grid,
                   const std::array<int64_t, 3> &block,
                   const std::vector<int32_t> &paramHandle,
                   const std::vector<int64_t> &scalarVal, int launchIndex) {
    auto handleOf = [&](const hgrd_gpu_site &st) -> int32_t {
      return st.param >= 0 ? paramHandle[static_cast<size_t>(st.param)] : -1;
    };
    // Buffers this launch writes (aliasing resolved through handles).
    std::set<int32_t> written;
    for (const auto &st : lk.sites)
      if (st.kind != HGRD_SITE_LOAD && handleOf(st) >= 0)
        written.insert(handleOf(st));
    bool sequential = false;
    for (size_t i = 0; i < lk.sites.size(); ++i) {
      const auto &st = lk.sites[i];
      int32_t h = handleOf(st);
      if (st.kind != HGRD_SITE_LOAD || h < 0 || !lk.siteValueNeeded[i])
        continue;
      if (written.count(h))
        sequential = true;
      if (bufs_[static_cast<size_t>(h)].stale)
        throw NeedConservative{};
    }
    if (conservative_ && !written.empty())
      sequential = true;
    if (sequential) {
      for (const auto &st : lk.sites) {
        int32_t h = handleOf(st);
        if (st.kind == HGRD_SITE_LOAD && h >= 0 && bufs_[static_cast<size_t>(h)].stale)
          throw NeedConservative{};
      }
    }
    if (spec_) { // speculative run: keep the launch for the batch, assume no traps
      if (sequential || lk.hasLocks)
        throw SpecFail{};
      PendingLaunch p;
      p.lk = &lk;
      p.launchIndex = launchIndex;
      p.grid = grid;
      p.block = block;
      p.warpSize = cfg_.warpSize;
      p.budget = cfg_.maxSteps;
      p.trapPos = res_.traps.size();
      p.regInit.assign(lk.nRegs, 0);
      for (size_t i = 0; i < lk.paramReg.size(); ++i)
        if (lk.paramReg[i] >= 0)
          p.regInit[static_cast<size_t>(lk.paramReg[i])] = scalarVal[i];
      p.paramHandle = paramHandle;
      p.bufElems.resize(bufs_.size());
      p.bufData.resize(bufs_.size());
      for (size_t h = 0; h < bufs_.size(); ++h)
        p.bufElems[h] = bufs_[h].elems;
      for (size_t i = 0; i < lk.sites.size(); ++i) { // launch-entry contents of value-needed loads
        const int32_t h = handleOf(lk.sites[i]);
        if (lk.sites[i].kind == HGRD_SITE_LOAD && h >= 0 && lk.siteValueNeeded[i])
          p.bufData[static_cast<size_t>(h)] = bufs_[static_cast<size_t>(h)].host;
      }
      spec_->push_back(std::move(p));
      ++res_.stats.parLaunches;
      for (int32_t h : written)
        bufs_[static_cast<size_t>(h)].stale = true;
      return;
    }
    // Bring host-side writes to the device.
    for (size_t h = 0; h < bufs_.size(); ++h) {
      Buf &b = bufs_[h];
      if (b.dirtyHi >= b.dirtyLo) {
        int rc = be_.write(static_cast<int32_t>(h), b.dirtyLo, b.dirtyHi - b.dirtyLo + 1,
                           b.host.data() + b.dirtyLo);
        if (rc < 0)
          throw BackendFail{rc, be_.lastError()};
        b.dirtyLo = INT64_MAX;
        b.dirtyHi = -1;
      }
    }
    std::vector<int64_t> regInit(lk.nRegs, 0);
    for (size_t i = 0; i < lk.paramReg.size(); ++i)
      if (lk.paramReg[i] >= 0)
        regInit[static_cast<size_t>(lk.paramReg[i])] = scalarVal[i];

    hgrd_gpu_launch L{};
    L.code = lk.code.data();
    L.n_code = static_cast<uint32_t>(lk.code.size());
    L.n_regs = lk.nRegs;
    L.reg_init = regInit.data();
    L.sites = lk.sites.data();
    L.n_sites = static_cast<uint32_t>(lk.sites.size());
    L.n_locs = static_cast<uint32_t>(lk.locs.size());
    L.param_handle = paramHandle.data();
    L.n_params = static_cast<uint32_t>(paramHandle.size());
    L.flags = (sequential ? HGRD_LAUNCH_SEQUENTIAL : 0u) |
              (lk.hasLocks ? HGRD_LAUNCH_PAIRWISE : 0u);
    for (int d = 0; d < 3; ++d) {
      L.grid[d] = grid[d];
      L.block[d] = block[d];
    }
    L.warp_size = cfg_.warpSize;
    L.step_budget = cfg_.maxSteps - steps_;

    const size_t nl = std::max<size_t>(lk.locs.size(), 1);
    std::vector<hgrd_gpu_race> races(3 * nl * nl);
    const size_t trapCap = res_.traps.size() < 256 ? 256 - res_.traps.size() : 0;
    std::vector<hgrd_gpu_trap> traps(std::max<size_t>(trapCap, 1));
    hgrd_gpu_result R{};
    R.races = races.data();
    R.race_cap = static_cast<uint32_t>(races.size());
    R.traps = traps.data();
    R.trap_cap = static_cast<uint32_t>(trapCap);
    int rc = be_.checkLaunch(L, R);
    if (rc < 0)
      throw BackendFail{rc, be_.lastError()};

    res_.stats.instances += R.instances;
    res_.stats.records += R.records;
    res_.stats.kernelSteps += R.steps;
    res_.stats.deviceMs += R.device_ms;
    if (R.mode & HGRD_LAUNCH_SEQUENTIAL)
      ++res_.stats.seqLaunches;
    else
      ++res_.stats.parLaunches;

    for (uint32_t i = 0; i < R.n_traps && i < trapCap; ++i) {
      const hgrd_gpu_trap &t = traps[i];
      const auto si = static_cast<size_t>(t.site);
      trap(lk.siteLoc[si], std::string(t.kind == HGRD_TRAP_OOB
                                            ? "kernel access out of bounds on "
                                            : "kernel access to unallocated array ") +
                               lk.siteArray[si]);
    }
    steps_ += R.steps;
    if (R.aborted) {
      trap(lk.stmtLocs[static_cast<size_t>(R.abort_stmt)], "step budget exhausted");
      throw Abort{};
    }
    // Memory state after the launch.
    for (int32_t h : written) {
      Buf &b = bufs_[static_cast<size_t>(h)];
      if (sequential)
        b.hostValid = false;
      else
        b.stale = true;
    }
    mergeLaunchRaces(res_, seen_, lk, grid, block, races.data(), R.n_races, launchIndex);
  }

  CompiledProgram &cp_;
  const Program &prog_;
  const ExecConfig &cfg_;
  LaunchBackend &be_;
  const bool conservative_;
  std::vector<PendingLaunch> *spec_;
  const bool lean_;
  bool budgetAbort_ = false;
  RunResult res_;
  std::vector<Buf> bufs_;
  std::map<std::pair<int, int>, DefVal> defs_;
  SeenKeys seen_;
  size_t inputCursor_ = 0;
  int64_t steps_ = 0;
  int callDepth_ = 0;
};

} // namespace

RunResult runConcrete(CompiledProgram &prog, const ExecConfig &cfg,
                      LaunchBackend &backend, bool lean) {
  try {
    return HostRun(prog, cfg, backend, false, nullptr, lean).run();
  } catch (const NeedConservative &) {
  }
  RunResult r;
  try {
    r = HostRun(prog, cfg, backend, true, nullptr, lean).run();
  } catch (const NeedConservative &) {
    r.error = HGRD_GPU_EINVAL;
    r.errorMessage = "stale buffer in conservative mode";
  }
  r.stats.restarts = 1;
  return r;
}

// reference enumerateVerdict, src/oracle.cpp:863-903
SweepResult enumerateVerdict(CompiledProgram &prog, const SweepCaps &caps,
                             LaunchBackend &backend) {
  SweepResult out;
  const int inputs = prog.inputs;
  std::set<std::tuple<int, int, int, int, int, int64_t>> seen;
  uint64_t configs = 0;
  std::vector<size_t> cursor(static_cast<size_t>(inputs), 0);
  for (int64_t ws : caps.warpSizes) {
    std::fill(cursor.begin(), cursor.end(), 0);
    for (;;) {
      if (configs++ > caps.maxConfigs) {
        out.configs = configs - 1;
        return out;
      }
      ExecConfig c;
      c.gridCap = caps.gridCap;
      c.blockCap = caps.blockCap;
      c.warpSize = ws;
      c.maxThreads = caps.maxThreads;
      for (int i = 0; i < inputs; ++i)
        c.inputs.push_back(caps.inputSet[cursor[static_cast<size_t>(i)]]);
      RunResult r = runConcrete(prog, c, backend, true);
      if (r.error) {
        out.error = r.error;
        out.errorMessage = r.errorMessage;
        return out;
      }
      out.stats.instances += r.stats.instances;
      out.stats.records += r.stats.records;
      out.stats.deviceMs += r.stats.deviceMs;
      out.stats.parLaunches += r.stats.parLaunches;
      out.stats.seqLaunches += r.stats.seqLaunches;
      out.stats.restarts += r.stats.restarts;
      for (const auto &race : r.races) {
        auto key = std::make_tuple(race.locA.line, race.locA.col, race.locB.line,
                                   race.locB.col, race.kind, ws);
        if (seen.insert(key).second)
          out.races.push_back(SweepRace{race.locA, race.locB, race.kind, ws});
      }
      int pos = inputs - 1;
      while (pos >= 0) {
        if (++cursor[static_cast<size_t>(pos)] < caps.inputSet.size())
          break;
        cursor[static_cast<size_t>(pos)] = 0;
        --pos;
      }
      if (pos < 0)
        break;
    }
  }
  out.configs = configs;
  return out;
}

namespace {

// enumerateVerdict's configurations in canonical order (warp sizes outer,
// input odometer inner, last input fastest; at most maxConfigs + 1),
// reference src/oracle.cpp:863-903.
std::vector<ExecConfig> sweepConfigs(const CompiledProgram &prog, const SweepCaps &caps) {
  std::vector<ExecConfig> out;
  const int inputs = prog.inputs;
  uint64_t configs = 0;
  std::vector<size_t> cursor(static_cast<size_t>(inputs), 0);
  for (int64_t ws : caps.warpSizes) {
    std::fill(cursor.begin(), cursor.end(), 0);
    for (;;) {
      if (configs++ > caps.maxConfigs)
        return out;
      ExecConfig c;
      c.gridCap = caps.gridCap;
      c.blockCap = caps.blockCap;
      c.warpSize = ws;
      c.maxThreads = caps.maxThreads;
      for (int i = 0; i < inputs; ++i)
        c.inputs.push_back(caps.inputSet[cursor[static_cast<size_t>(i)]]);
      out.push_back(std::move(c));
      int pos = inputs - 1;
      while (pos >= 0) {
        if (++cursor[static_cast<size_t>(pos)] < caps.inputSet.size())
          break;
        cursor[static_cast<size_t>(pos)] = 0;
        --pos;
      }
      if (pos < 0)
        break;
    }
  }
  return out;
}

// Host-only backend of a speculative run: handles and sizes, no device.
class SpecBackend final : public LaunchBackend {
public:
  int reset() override {
    n_ = 0;
    return 0;
  }
  int alloc(int64_t, int32_t *handle) override {
    *handle = n_++;
    return 0;
  }
  int write(int32_t, int64_t, int64_t, const int64_t *) override { return 0; }
  int read(int32_t, int64_t, int64_t, int64_t *) override { return HGRD_GPU_EINVAL; }
  int checkLaunch(const hgrd_gpu_launch &, hgrd_gpu_result &) override { return HGRD_GPU_EINVAL; }
  std::string lastError() override { return "speculative run"; }

private:
  int32_t n_ = 0;
};

struct SpecRun {
  bool ok = false;
  RunResult res;
  std::vector<PendingLaunch> launches;
  int64_t hostSteps = 0;
};

SpecRun speculate(CompiledProgram &prog, const ExecConfig &cfg) {
  SpecRun out;
  SpecBackend be;
  try {
    HostRun run(prog, cfg, be, false, &out.launches, true);
    out.res = run.run();
    out.ok = !run.budgetAborted() && out.res.error == 0;
    out.hostSteps = run.steps();
  } catch (const SpecFail &) {
  } catch (const NeedConservative &) {
  }
  return out;
}

} // namespace

namespace {

// A configuration of one program's sweep (several programs' sweeps can be
// batched together).
struct ConfigJob {
  CompiledProgram *prog;
  ExecConfig cfg;
};

// runConcrete of every configuration in `jobs` (results in order): host
// runs speculated on host threads, their launches checked in batches, the
// configurations whose speculation fails re-run exactly.  ENOTSUP when the
// backend has no batched path.
// Exact runs of configurations `which` (runConcrete), spread over worker
// backends 1..n-1 (backend 0 is the batch's), one host thread each.
struct ExactPool {
  const std::function<LaunchBackend *(int)> *workers;
  int n;
  std::vector<std::thread> threads;
  std::atomic<size_t> next{0};
  std::atomic<int> error{0};
  std::string err;

  void start(const std::vector<ConfigJob> &jobs, const std::vector<size_t> &which,
             std::vector<RunResult> &out) {
    const int nt = static_cast<int>(std::min<size_t>(static_cast<size_t>(std::max(n - 1, 0)),
                                                     which.size()));
    for (int t = 1; t <= nt; ++t) {
      LaunchBackend *be = (*workers)(t);
      if (!be)
        break;
      threads.emplace_back([&, be] {
        for (size_t k; (k = next.fetch_add(1)) < which.size();) {
          const ConfigJob &j = jobs[which[k]];
          RunResult r = runConcrete(*j.prog, j.cfg, *be, true);
          if (r.error) {
            error = r.error;
            err = r.errorMessage;
          }
          ++r.stats.restarts;
          out[which[k]] = std::move(r);
        }
      });
    }
  }
  // remaining configurations on the caller's backend, then wait
  int finish(const std::vector<ConfigJob> &jobs, const std::vector<size_t> &which,
             std::vector<RunResult> &out, LaunchBackend &be) {
    for (size_t k; (k = next.fetch_add(1)) < which.size();) {
      const ConfigJob &j = jobs[which[k]];
      RunResult r = runConcrete(*j.prog, j.cfg, be, true);
      if (r.error) {
        error = r.error;
        err = r.errorMessage;
      }
      ++r.stats.restarts;
      out[which[k]] = std::move(r);
    }
    for (auto &t : threads)
      t.join();
    threads.clear();
    return error;
  }
};

int runConfigsBatched(const std::vector<ConfigJob> &jobs, LaunchBackend &backend,
                      int hostThreads, std::vector<RunResult> &outRuns, std::string &err,
                      const std::function<LaunchBackend *(int)> *workers, int nWorkers) {
  const size_t nc = jobs.size();
  const auto tA = std::chrono::steady_clock::now();
  // lower every kernel up front (the cache is not thread-safe)
  {
    std::set<CompiledProgram *> progs;
    for (const ConfigJob &j : jobs)
      if (progs.insert(j.prog).second)
        for (const Function &k : j.prog->program->kernels)
          j.prog->kernel(&k);
  }
  // 1. speculative host runs, spread over host threads
  std::vector<SpecRun> spec(nc);
  if (hostThreads > 1)
    parallelFor(nc, [&](size_t i) { spec[i] = speculate(*jobs[i].prog, jobs[i].cfg); }, 16);
  else
    for (size_t i = 0; i < nc; ++i)
      spec[i] = speculate(*jobs[i].prog, jobs[i].cfg);
  // configurations whose speculation failed (sequential or lock-idiom
  // launches, host reads of device results, the host's step budget) run
  // exactly on the worker backends while the batch is checked
  outRuns.assign(nc, RunResult{});
  std::vector<size_t> failed;
  for (size_t i = 0; i < nc; ++i)
    if (!spec[i].ok)
      failed.push_back(i);
  ExactPool pool{workers, workers ? nWorkers : 0};
  if (workers && !failed.empty())
    pool.start(jobs, failed, outRuns);
  const auto tB = std::chrono::steady_clock::now();
  // 2. every pending launch of every configuration in one batched check
  std::vector<hgrd_gpu_batch_launch> bl;
  std::vector<std::vector<const int64_t *>> dataPtrs;
  std::vector<std::pair<size_t, size_t>> owner; // batch entry -> (config, launch)
  size_t nRaceSlots = 0;
  for (size_t i = 0; i < nc; ++i)
    if (spec[i].ok)
      for (size_t k = 0; k < spec[i].launches.size(); ++k) {
        owner.emplace_back(i, k);
        const size_t nl = std::max<size_t>(spec[i].launches[k].lk->locs.size(), 1);
        nRaceSlots += 3 * nl * nl;
      }
  bl.resize(owner.size());
  dataPtrs.resize(owner.size());
  std::vector<hgrd_gpu_race> raceStore(std::max<size_t>(nRaceSlots, 1));
  std::vector<hgrd_gpu_result> results(owner.size());
  constexpr uint32_t kTrapsPerLaunch = 64; // more: the configuration is re-run exactly
  std::unique_ptr<hgrd_gpu_trap[]> trapStore(
      new hgrd_gpu_trap[std::max<size_t>(owner.size(), 1) * kTrapsPerLaunch]);
  std::vector<size_t> raceAt(owner.size() + 1, 0);
  for (size_t e = 0; e < owner.size(); ++e) {
    const size_t nl = std::max<size_t>(spec[owner[e].first].launches[owner[e].second].lk->locs.size(), 1);
    raceAt[e + 1] = raceAt[e] + 3 * nl * nl;
  }
  parallelFor(owner.size(), [&](size_t e) {
    const PendingLaunch &p = spec[owner[e].first].launches[owner[e].second];
    const LoweredKernel &lk = *p.lk;
    hgrd_gpu_launch &L = bl[e].launch;
    L = hgrd_gpu_launch{};
    L.code = lk.code.data();
    L.n_code = static_cast<uint32_t>(lk.code.size());
    L.n_regs = lk.nRegs;
    L.reg_init = p.regInit.data();
    L.sites = lk.sites.data();
    L.n_sites = static_cast<uint32_t>(lk.sites.size());
    L.n_locs = static_cast<uint32_t>(lk.locs.size());
    L.param_handle = p.paramHandle.data();
    L.n_params = static_cast<uint32_t>(p.paramHandle.size());
    L.flags = 0;
    for (int d = 0; d < 3; ++d) {
      L.grid[d] = p.grid[d];
      L.block[d] = p.block[d];
    }
    L.warp_size = p.warpSize;
    L.step_budget = p.budget;
    dataPtrs[e].resize(p.bufData.size());
    for (size_t h = 0; h < p.bufData.size(); ++h)
      dataPtrs[e][h] = p.bufData[h].empty() ? nullptr : p.bufData[h].data();
    bl[e].buffer_elems = p.bufElems.data();
    bl[e].buffer_data = dataPtrs[e].data();
    bl[e].n_buffers = static_cast<uint32_t>(p.bufElems.size());
    results[e] = hgrd_gpu_result{};
    results[e].races = raceStore.data() + raceAt[e];
    results[e].race_cap = static_cast<uint32_t>(raceAt[e + 1] - raceAt[e]);
    results[e].traps = trapStore.get() + e * kTrapsPerLaunch;
    results[e].trap_cap = kTrapsPerLaunch;
  });
  const auto tC = std::chrono::steady_clock::now();
  if (!bl.empty()) {
    constexpr size_t kChunk = 1 << 16; // launches per batched check
    for (size_t b = 0; b < bl.size(); b += kChunk) {
      const uint32_t m = static_cast<uint32_t>(std::min(kChunk, bl.size() - b));
      const int rc = backend.checkBatch(bl.data() + b, m, results.data() + b);
      if (rc < 0) {
        pool.finish(jobs, failed, outRuns, backend);
        err = backend.lastError();
        return rc;
      }
    }
  }
  const auto tD = std::chrono::steady_clock::now();
  // 3. per configuration in canonical order: the speculation's report, or an
  //    exact re-run
  std::vector<char> exact(nc, 0);
  for (size_t i = 0; i < nc; ++i)
    exact[i] = !spec[i].ok;
  std::vector<int64_t> kernelSteps(nc, 0);
  size_t nSpecFail = 0, nUnchecked = 0;
  for (size_t i = 0; i < nc; ++i)
    nSpecFail += !spec[i].ok;
  for (size_t e = 0; e < owner.size(); ++e) {
    const size_t i = owner[e].first;
    if (results[e].mode & HGRD_RESULT_UNCHECKED) {
      nUnchecked += !exact[i];
      exact[i] = 1;
    }
    kernelSteps[i] += results[e].steps;
  }
  if (pool.finish(jobs, failed, outRuns, backend) < 0) {
    err = pool.err;
    return pool.error;
  }
  const auto tE = std::chrono::steady_clock::now();
  // the configurations' first batch entries (entries are in config order)
  std::vector<size_t> firstEntry(nc + 1, owner.size());
  for (size_t e = owner.size(); e-- > 0;)
    firstEntry[owner[e].first] = e;
  // 3a. the speculation's report per configuration (independent: host threads)
  parallelFor(
      nc,
      [&](size_t i) {
        if (!spec[i].ok)
          return; // (run exactly by the pool)
        if (!exact[i] && spec[i].hostSteps + kernelSteps[i] > jobs[i].cfg.maxSteps)
          exact[i] = 1; // the budget runs out somewhere: the exact run finds where
        if (exact[i])
          return;
        const size_t e0 = firstEntry[i], e = e0 + spec[i].launches.size();
        // kernel traps go between the host traps recorded before and after
        // their launch; the run keeps the first 256 (reference :125-130)
        std::vector<std::string> traps;
        const std::vector<std::string> &hostTraps = spec[i].res.traps;
        size_t hostAt = 0;
        for (size_t q = e0; q < e; ++q) {
          const PendingLaunch &p = spec[i].launches[q - e0];
          while (hostAt < p.trapPos && hostAt < hostTraps.size())
            traps.push_back(hostTraps[hostAt++]);
          const hgrd_gpu_result &kr = results[q];
          const uint64_t want = std::min<uint64_t>(kr.n_traps_total,
                                                   traps.size() < 256 ? 256 - traps.size() : 0);
          if (want > kr.n_traps) {
            exact[i] = 1; // more traps than the batch handed back
            return;
          }
          for (uint64_t t = 0; t < want; ++t) {
            const auto si = static_cast<size_t>(kr.traps[t].site);
            traps.push_back(jobs[i].prog->program->file + ":" +
                            std::to_string(p.lk->siteLoc[si].line) + ": " +
                            (kr.traps[t].kind == HGRD_TRAP_OOB
                                 ? "kernel access out of bounds on "
                                 : "kernel access to unallocated array ") +
                            p.lk->siteArray[si]);
          }
        }
        while (hostAt < hostTraps.size())
          traps.push_back(hostTraps[hostAt++]);
        if (traps.size() > 256)
          traps.resize(256);
        RunResult &r = outRuns[i];
        r = std::move(spec[i].res);
        r.traps = std::move(traps);
        SeenKeys keys;
        for (size_t q = e0; q < e; ++q) {
          const PendingLaunch &p = spec[i].launches[q - e0];
          mergeLaunchRaces(r, keys, *p.lk, p.grid, p.block, results[q].races,
                           results[q].n_races, p.launchIndex);
          r.stats.instances += results[q].instances;
          r.stats.records += results[q].records;
          r.stats.kernelSteps += results[q].steps;
          ++r.stats.batchedLaunches;
        }
        sortRaces(r.races);
      },
      64);
  // 3b. exact re-runs of what the batch could not decide (traps beyond the
  //     batch's trap slots, the step budget, unchecked launches)
  std::vector<size_t> redo;
  for (size_t i = 0; i < nc; ++i)
    if (spec[i].ok && exact[i])
      redo.push_back(i);
  if (!redo.empty()) {
    ExactPool pool2{workers, workers ? nWorkers : 0};
    if (workers)
      pool2.start(jobs, redo, outRuns);
    if (pool2.finish(jobs, redo, outRuns, backend) < 0) {
      err = pool2.err;
      return pool2.error;
    }
  }
  // the speculation state (tens of thousands of small allocations) is freed
  // off the caller's critical path
  std::thread([s = std::move(spec), b = std::move(bl), d = std::move(dataPtrs),
               r = std::move(results), rs = std::move(raceStore)]() mutable {}).detach();
  // development: HGRD_SWEEP_TRACE=1 prints why configurations were re-run
  // and where the time went
  static const bool trace = std::getenv("HGRD_SWEEP_TRACE") != nullptr;
  if (trace) {
    const auto tF = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    std::fprintf(stderr, "[hgrd sweep] %zu configs, %zu launches batched, %zu speculation "
                 "failures, %zu with unchecked launches; speculate %.0f prepare %.0f batch %.0f "
                 "exact-wait %.0f merge %.0f (us)\n", nc, owner.size(), nSpecFail, nUnchecked,
                 us(tA, tB), us(tB, tC), us(tC, tD), us(tD, tE), us(tE, tF));
  }
  return 0;
}

} // namespace

int sweepHostThreads() {
  if (const char *e = std::getenv("HGRD_SWEEP_THREADS"))
    return std::max(1, std::atoi(e));
  return static_cast<int>(std::min(32u, std::max(1u, std::thread::hardware_concurrency())));
}

SweepResult enumerateVerdictBatched(CompiledProgram &prog, const SweepCaps &caps,
                                    LaunchBackend &backend, int hostThreads,
                                    const std::function<LaunchBackend *(int)> *workers,
                                    int nWorkers) {
  const std::vector<ExecConfig> cfgs = sweepConfigs(prog, caps);
  std::vector<ConfigJob> jobs;
  for (const ExecConfig &c : cfgs)
    jobs.push_back(ConfigJob{&prog, c});
  std::vector<RunResult> runs;
  std::string err;
  const int rc = runConfigsBatched(jobs, backend, hostThreads, runs, err, workers, nWorkers);
  if (rc == HGRD_GPU_ENOTSUP)
    return enumerateVerdict(prog, caps, backend);
  SweepResult out;
  if (rc < 0) {
    out.error = rc;
    out.errorMessage = err;
    return out;
  }
  out.configs = cfgs.size();
  std::set<std::tuple<int, int, int, int, int, int64_t>> seen; // first wins, :883-889
  for (size_t i = 0; i < cfgs.size(); ++i) {
    const RunResult &r = runs[i];
    out.stats.instances += r.stats.instances;
    out.stats.records += r.stats.records;
    out.stats.parLaunches += r.stats.parLaunches;
    out.stats.seqLaunches += r.stats.seqLaunches;
    out.stats.restarts += r.stats.restarts;
    out.stats.batchedLaunches += r.stats.batchedLaunches;
    for (const auto &race : r.races) {
      auto key = std::make_tuple(race.locA.line, race.locA.col, race.locB.line, race.locB.col,
                                 race.kind, cfgs[i].warpSize);
      if (seen.insert(key).second)
        out.races.push_back(SweepRace{race.locA, race.locB, race.kind, cfgs[i].warpSize});
    }
  }
  return out;
}

SweepShard sweepShardBatched(CompiledProgram &prog, const SweepCaps &caps, int rank, int world,
                             LaunchBackend &backend, int hostThreads) {
  const std::vector<ExecConfig> all = sweepConfigs(prog, caps);
  std::vector<ExecConfig> mine;
  std::vector<uint64_t> index;
  for (size_t k = 0; k < all.size(); ++k)
    if (static_cast<int>(k % static_cast<size_t>(world)) == rank) {
      mine.push_back(all[k]);
      index.push_back(k);
    }
  std::vector<ConfigJob> jobs;
  for (const ExecConfig &c : mine)
    jobs.push_back(ConfigJob{&prog, c});
  std::vector<RunResult> runs;
  std::string err;
  const int rc = runConfigsBatched(jobs, backend, hostThreads, runs, err, nullptr, 0);
  if (rc == HGRD_GPU_ENOTSUP)
    return sweepShard(prog, caps, rank, world, backend);
  SweepShard out;
  out.total = all.size();
  if (rc < 0) {
    out.error = rc;
    out.errorMessage = err;
    return out;
  }
  for (size_t i = 0; i < mine.size(); ++i) {
    RunResult &r = runs[i];
    out.stats.instances += r.stats.instances;
    out.stats.records += r.stats.records;
    out.stats.parLaunches += r.stats.parLaunches;
    out.stats.seqLaunches += r.stats.seqLaunches;
    out.stats.restarts += r.stats.restarts;
    out.stats.batchedLaunches += r.stats.batchedLaunches;
    out.configs.push_back(ShardConfig{index[i], mine[i].warpSize, std::move(r.races)});
  }
  return out;
}


SweepShard sweepShard(CompiledProgram &prog, const SweepCaps &caps, int rank, int world,
                      LaunchBackend &backend) {
  SweepShard out;
  const int inputs = prog.inputs;
  uint64_t configs = 0;
  std::vector<size_t> cursor(static_cast<size_t>(inputs), 0);
  for (int64_t ws : caps.warpSizes) {
    std::fill(cursor.begin(), cursor.end(), 0);
    for (;;) {
      if (configs > caps.maxConfigs) { // reference :873 (configs++ > maxConfigs)
        out.total = configs;
        return out;
      }
      const uint64_t index = configs++;
      if (static_cast<int>(index % static_cast<uint64_t>(world)) == rank) {
        ExecConfig c;
        c.gridCap = caps.gridCap;
        c.blockCap = caps.blockCap;
        c.warpSize = ws;
        c.maxThreads = caps.maxThreads;
        for (int i = 0; i < inputs; ++i)
          c.inputs.push_back(caps.inputSet[cursor[static_cast<size_t>(i)]]);
        RunResult r = runConcrete(prog, c, backend, true);
        if (r.error) {
          out.error = r.error;
          out.errorMessage = r.errorMessage;
          return out;
        }
        out.stats.instances += r.stats.instances;
        out.stats.records += r.stats.records;
        out.stats.deviceMs += r.stats.deviceMs;
        out.stats.parLaunches += r.stats.parLaunches;
        out.stats.seqLaunches += r.stats.seqLaunches;
        out.stats.restarts += r.stats.restarts;
        out.configs.push_back(ShardConfig{index, ws, std::move(r.races)});
      }
      int pos = inputs - 1;
      while (pos >= 0) {
        if (++cursor[static_cast<size_t>(pos)] < caps.inputSet.size())
          break;
        cursor[static_cast<size_t>(pos)] = 0;
        --pos;
      }
      if (pos < 0)
        break;
    }
  }
  out.total = configs;
  return out;
}

// ---------------------------------------------------------------------------
// JSON

namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0;
  bool isInt = true;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal *get(const char *k) const {
    for (const auto &kv : obj)
      if (kv.first == k)
        return &kv.second;
    return nullptr;
  }
};

class JParse {
public:
  explicit JParse(const char *s) : p_(s) {}
  JVal value() {
    ws();
    JVal v;
    char c = *p_;
    if (c == '{') {
      ++p_;
      v.kind = JVal::Obj;
      ws();
      if (*p_ == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        expect(':');
        JVal x = value();
        v.obj.emplace_back(std::move(k), std::move(x));
        ws();
        if (*p_ == ',') {
          ++p_;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      ++p_;
      v.kind = JVal::Arr;
      ws();
      if (*p_ == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (*p_ == ',') {
          ++p_;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.s = str();
      return v;
    }
    if (!std::strncmp(p_, "true", 4)) {
      p_ += 4;
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (!std::strncmp(p_, "false", 5)) {
      p_ += 5;
      v.kind = JVal::Bool;
      return v;
    }
    if (!std::strncmp(p_, "null", 4)) {
      p_ += 4;
      return v;
    }
    const char *start = p_;
    if (*p_ == '-' || *p_ == '+')
      ++p_;
    bool isInt = true;
    while ((*p_ >= '0' && *p_ <= '9') || *p_ == '.' || *p_ == 'e' || *p_ == 'E' ||
           *p_ == '-' || *p_ == '+') {
      if (*p_ == '.' || *p_ == 'e' || *p_ == 'E')
        isInt = false;
      ++p_;
    }
    if (p_ == start)
      throw std::runtime_error("bad JSON value");
    std::string num(start, p_);
    v.kind = JVal::Num;
    v.isInt = isInt;
    if (isInt) {
      v.i = std::stoll(num);
      v.d = static_cast<double>(v.i);
    } else {
      v.d = std::stod(num);
      v.i = static_cast<int64_t>(v.d);
    }
    return v;
  }

private:
  void ws() {
    while (*p_ == ' ' || *p_ == '\n' || *p_ == '\t' || *p_ == '\r')
      ++p_;
  }
  void expect(char c) {
    if (*p_ != c)
      throw std::runtime_error(std::string("JSON: expected ") + c);
    ++p_;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (*p_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        char e = *p_++;
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
      } else {
        out.push_back(*p_++);
      }
    }
    expect('"');
    return out;
  }
  const char *p_;
};

bool readI64(const JVal &o, const char *k, int64_t &dst) {
  const JVal *v = o.get(k);
  if (!v || v->kind != JVal::Num)
    return false;
  dst = v->i;
  return true;
}
void readArr3(const JVal &o, const char *k, std::array<int64_t, 3> &dst) {
  const JVal *v = o.get(k);
  if (!v || v->kind != JVal::Arr)
    return;
  for (size_t i = 0; i < 3 && i < v->arr.size(); ++i)
    dst[i] = v->arr[i].i;
}
void readVec(const JVal &o, const char *k, std::vector<int64_t> &dst) {
  const JVal *v = o.get(k);
  if (!v || v->kind != JVal::Arr)
    return;
  dst.clear();
  for (const auto &x : v->arr)
    dst.push_back(x.i);
}

std::string esc(const std::string &s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
    case '"':
      o += "\\\"";
      break;
    case '\\':
      o += "\\\\";
      break;
    case '\n':
      o += "\\n";
      break;
    case '\t':
      o += "\\t";
      break;
    default:
      if (static_cast<unsigned char>(c) < 0x20) {
        char buf[8];
        std::snprintf(buf, sizeof buf, "\\u%04x", c);
        o += buf;
      } else {
        o.push_back(c);
      }
    }
  }
  return o + "\"";
}

std::string locJ(const Loc &l, const std::string &file) {
  return "{\"file\":" + esc(file) + ",\"line\":" + std::to_string(l.line) +
         ",\"column\":" + std::to_string(l.col) + "}";
}

template <class V> std::string arrJ(const V &v) {
  std::string o = "[";
  bool first = true;
  for (const auto &x : v) {
    if (!first)
      o += ",";
    first = false;
    o += std::to_string(x);
  }
  return o + "]";
}

std::string statsJ(const RunStats &s) {
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"instances\":%" PRIu64 ",\"records\":%" PRIu64
                ",\"kernelSteps\":%" PRId64 ",\"deviceMs\":%.6f,\"parallelLaunches\":%d,"
                "\"sequentialLaunches\":%d,\"restarts\":%d,\"batchedLaunches\":%d}",
                s.instances, s.records, s.kernelSteps, s.deviceMs, s.parLaunches,
                s.seqLaunches, s.restarts, s.batchedLaunches);
  return buf;
}

} // namespace

bool parseExecConfigJson(const char *json, ExecConfig &c, std::string &err) {
  try {
    JVal o = JParse(json && *json ? json : "{}").value();
    readArr3(o, "gridCap", c.gridCap);
    readArr3(o, "blockCap", c.blockCap);
    readI64(o, "warpSize", c.warpSize);
    readVec(o, "inputs", c.inputs);
    readI64(o, "maxThreads", c.maxThreads);
    readI64(o, "maxArrayElems", c.maxArrayElems);
    readI64(o, "maxSteps", c.maxSteps);
  } catch (const std::exception &e) {
    err = e.what();
    return false;
  }
  return true;
}

void capsFromJson(const JVal &o, SweepCaps &c) {
  readArr3(o, "gridCap", c.gridCap);
  readArr3(o, "blockCap", c.blockCap);
  readVec(o, "inputSet", c.inputSet);
  readVec(o, "warpSizes", c.warpSizes);
  readI64(o, "maxThreads", c.maxThreads);
  int64_t mc;
  if (readI64(o, "maxConfigs", mc))
    c.maxConfigs = static_cast<uint64_t>(mc);
}

bool parseSweepCapsJson(const char *json, SweepCaps &c, std::string &err) {
  try {
    capsFromJson(JParse(json && *json ? json : "{}").value(), c);
  } catch (const std::exception &e) {
    err = e.what();
    return false;
  }
  return true;
}

std::string errorJson(const std::vector<std::string> &diags) {
  std::string o = "{\"error\":[";
  for (size_t i = 0; i < diags.size(); ++i)
    o += (i ? "," : "") + esc(diags[i]);
  return o + "]}";
}

std::string runResultJson(const RunResult &r, const std::string &file) {
  std::ostringstream o;
  o << "{\"races\":[";
  for (size_t i = 0; i < r.races.size(); ++i) {
    const Race &x = r.races[i];
    o << (i ? "," : "") << "{\"kind\":" << esc(raceKindName(x.kind))
      << ",\"locA\":" << locJ(x.locA, file) << ",\"locB\":" << locJ(x.locB, file)
      << ",\"array\":" << esc(x.array) << ",\"address\":" << x.address << "}";
  }
  o << "],\"traps\":[";
  for (size_t i = 0; i < r.traps.size(); ++i)
    o << (i ? "," : "") << esc(r.traps[i]);
  o << "],\"launchesRun\":" << r.launchesRun
    << ",\"launchesSkipped\":" << r.launchesSkipped
    << ",\"assertStopped\":" << (r.assertStopped ? "true" : "false")
    << ",\"indirectIndexing\":" << (r.indirectIndexing ? "true" : "false")
    << ",\"launchRecords\":[";
  for (size_t i = 0; i < r.launchRecords.size(); ++i) {
    const LaunchRec &l = r.launchRecords[i];
    o << (i ? "," : "") << "{\"site\":" << l.site << ",\"line\":" << l.loc.line
      << ",\"column\":" << l.loc.col << ",\"grid\":" << arrJ(l.grid)
      << ",\"block\":" << arrJ(l.block) << ",\"scalarArgs\":" << arrJ(l.scalarArgs)
      << ",\"isScalar\":[";
    for (size_t k = 0; k < l.isScalar.size(); ++k)
      o << (k ? "," : "") << (l.isScalar[k] ? 1 : 0);
    o << "],\"defValues\":[";
    bool first = true;
    for (const auto &[key, dv] : l.defValues) {
      o << (first ? "" : ",") << "[" << key.first << "," << key.second << ","
        << esc(dv.name) << "," << dv.value << "]";
      first = false;
    }
    o << "]}";
  }
  o << "],\"witnesses\":[";
  for (size_t i = 0; i < r.races.size(); ++i) {
    const Race &x = r.races[i];
    o << (i ? "," : "") << "{\"launch\":" << x.launch << ",\"threadA\":" << x.threadX
      << ",\"seqA\":" << x.seqX << ",\"blockIdxA\":" << arrJ(x.blockX)
      << ",\"threadIdxA\":" << arrJ(x.tidX) << ",\"threadB\":" << x.threadY
      << ",\"seqB\":" << x.seqY << ",\"blockIdxB\":" << arrJ(x.blockY)
      << ",\"threadIdxB\":" << arrJ(x.tidY) << "}";
  }
  o << "],\"stats\":" << statsJ(r.stats) << "}";
  return o.str();
}

std::string sweepResultJson(const SweepResult &r, const std::string &file) {
  // (direct appends: a config-5 sweep reports thousands of races per call)
  const std::string fileJ = esc(file);
  std::string o;
  o.reserve(96 + r.races.size() * (112 + 2 * fileJ.size()));
  o += "{\"races\":[";
  char num[24];
  auto put = [&](int64_t v) {
    const auto res = std::to_chars(num, num + sizeof num, v);
    o.append(num, static_cast<size_t>(res.ptr - num));
  };
  auto loc = [&](const Loc &l) {
    o += "{\"file\":";
    o += fileJ;
    o += ",\"line\":";
    put(l.line);
    o += ",\"column\":";
    put(l.col);
    o += "}";
  };
  for (size_t i = 0; i < r.races.size(); ++i) {
    const SweepRace &x = r.races[i];
    o += i ? ",{\"kind\":\"" : "{\"kind\":\"";
    o += raceKindName(x.kind);
    o += "\",\"locA\":";
    loc(x.locA);
    o += ",\"locB\":";
    loc(x.locB);
    o += ",\"warpSize\":";
    put(x.warpSize);
    o += "}";
  }
  o += "],\"configs\":";
  put(static_cast<int64_t>(r.configs));
  o += ",\"stats\":";
  o += statsJ(r.stats);
  o += "}";
  return o;
}

std::string sweepShardJson(const SweepShard &r, const std::string &file) {
  std::ostringstream o;
  o << "{\"total\":" << r.total << ",\"configs\":[";
  for (size_t i = 0; i < r.configs.size(); ++i) {
    const ShardConfig &c = r.configs[i];
    o << (i ? "," : "") << "{\"index\":" << c.index << ",\"warpSize\":" << c.warpSize
      << ",\"races\":[";
    for (size_t k = 0; k < c.races.size(); ++k) {
      const Race &x = c.races[k];
      o << (k ? "," : "") << "{\"kind\":" << esc(raceKindName(x.kind))
        << ",\"locA\":" << locJ(x.locA, file) << ",\"locB\":" << locJ(x.locB, file) << "}";
    }
    o << "]}";
  }
  o << "],\"stats\":" << statsJ(r.stats) << "}";
  return o.str();
}

int sweepShardJsonRun(LaunchBackend &be, const char *src, const char *file,
                      const char *capsJson, int rank, int world, std::string &out) {
  SweepCaps caps;
  std::string err;
  if (world < 1 || rank < 0 || rank >= world) {
    out = errorJson({"bad rank/world"});
    return HGRD_GPU_EINVAL;
  }
  if (!parseSweepCapsJson(capsJson, caps, err)) {
    out = errorJson({"caps: " + err});
    return HGRD_GPU_EINVAL;
  }
  ParseOutcome po = parseMiniCU(src ? src : "", file ? file : "");
  if (!po.program) {
    out = errorJson(po.diagnostics);
    return HGRD_GPU_OK;
  }
  std::string fileName = po.program->file;
  auto cp = compileProgram(std::move(po.program));
  SweepShard r = be.hasBatch() ? sweepShardBatched(*cp, caps, rank, world, be, sweepHostThreads())
                               : sweepShard(*cp, caps, rank, world, be);
  if (r.error) {
    out = errorJson({"backend: " + r.errorMessage});
    return r.error;
  }
  out = sweepShardJson(r, fileName);
  return HGRD_GPU_OK;
}

int runConcreteJson(LaunchBackend &be, const char *src, const char *file,
                    const char *cfgJson, std::string &out) {
  ExecConfig cfg;
  std::string err;
  if (!parseExecConfigJson(cfgJson, cfg, err)) {
    out = errorJson({"config: " + err});
    return HGRD_GPU_EINVAL;
  }
  // development: HGRD_HOST_TRACE=1 prints the host phases of the call
  static const bool trace = std::getenv("HGRD_HOST_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  ParseOutcome po = parseMiniCU(src ? src : "", file ? file : "");
  if (!po.program) {
    out = errorJson(po.diagnostics);
    return HGRD_GPU_OK;
  }
  std::string fileName = po.program->file;
  auto cp = compileProgram(std::move(po.program));
  const auto t1 = std::chrono::steady_clock::now();
  RunResult r = runConcrete(*cp, cfg, be);
  const auto t2 = std::chrono::steady_clock::now();
  if (r.error) {
    out = errorJson({"backend: " + r.errorMessage});
    return r.error;
  }
  out = runResultJson(r, fileName);
  if (trace) {
    const auto t3 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "[hgrd run_concrete] parse+compile %.1f run %.1f json %.1f (us)\n",
                 us(t0, t1), us(t1, t2), us(t2, t3));
  }
  return HGRD_GPU_OK;
}

uint64_t sweepSize(const CompiledProgram &prog, const SweepCaps &caps) {
  long double per = 1;
  for (int i = 0; i < prog.inputs; ++i)
    per *= static_cast<long double>(caps.inputSet.size());
  const long double all = per * static_cast<long double>(caps.warpSizes.size());
  const long double cap = static_cast<long double>(caps.maxConfigs) + 1;
  return static_cast<uint64_t>(all < cap ? all : cap);
}

SweepResult enumerateVerdictParallel(CompiledProgram &prog, const SweepCaps &caps,
                                     const std::vector<LaunchBackend *> &backends) {
  // lower every kernel first: the shards then only read the program
  for (const auto &k : prog.program->kernels)
    prog.kernel(&k);
  const int world = static_cast<int>(backends.size());
  std::vector<SweepShard> shards(static_cast<size_t>(world));
  std::vector<std::thread> threads;
  for (int r = 0; r < world; ++r)
    threads.emplace_back([&, r] {
      shards[static_cast<size_t>(r)] = sweepShard(prog, caps, r, world, *backends[static_cast<size_t>(r)]);
    });
  for (auto &t : threads)
    t.join();
  SweepResult out;
  std::vector<const ShardConfig *> all;
  for (const auto &sh : shards) {
    if (sh.error) {
      out.error = sh.error;
      out.errorMessage = sh.errorMessage;
      return out;
    }
    out.configs = std::max<uint64_t>(out.configs, sh.total);
    out.stats.instances += sh.stats.instances;
    out.stats.records += sh.stats.records;
    out.stats.deviceMs += sh.stats.deviceMs;
    out.stats.parLaunches += sh.stats.parLaunches;
    out.stats.seqLaunches += sh.stats.seqLaunches;
    out.stats.restarts += sh.stats.restarts;
    for (const auto &c : sh.configs)
      all.push_back(&c);
  }
  std::sort(all.begin(), all.end(),
            [](const ShardConfig *a, const ShardConfig *b) { return a->index < b->index; });
  std::set<std::tuple<int, int, int, int, int, int64_t>> seen; // reference :883-889
  for (const ShardConfig *c : all)
    for (const auto &race : c->races) {
      auto key = std::make_tuple(race.locA.line, race.locA.col, race.locB.line, race.locB.col,
                                 race.kind, c->warpSize);
      if (seen.insert(key).second)
        out.races.push_back(SweepRace{race.locA, race.locB, race.kind, c->warpSize});
    }
  return out;
}

SweepResult enumerateVerdictOnWorkers(const std::function<LaunchBackend *(int)> &workers, int n,
                                      CompiledProgram &cp, const SweepCaps &caps) {
  if (LaunchBackend *b0 = workers(0); b0 && b0->hasBatch())
    return enumerateVerdictBatched(cp, caps, *b0, sweepHostThreads(), &workers, n);
  const uint64_t size = sweepSize(cp, caps);
  // one configuration per worker at least: a configuration costs a few
  // GPU round trips (~30 us each), more than spawning its worker thread
  int use = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(std::max(n, 1)), size));
  std::vector<LaunchBackend *> bes;
  for (int i = 0; i < std::max(use, 1); ++i) {
    LaunchBackend *b = workers(i);
    if (!b)
      break;
    bes.push_back(b);
  }
  if (bes.empty()) {
    SweepResult r;
    r.error = HGRD_GPU_ENODEV;
    r.errorMessage = "no sweep worker";
    return r;
  }
  return bes.size() > 1 ? enumerateVerdictParallel(cp, caps, bes)
                        : enumerateVerdict(cp, caps, *bes[0]);
}

int enumerateVerdictJsonParallel(const std::function<LaunchBackend *(int)> &workers, int n,
                                 const char *src, const char *file, const char *capsJson,
                                 std::string &out) {
  SweepCaps caps;
  std::string err;
  if (!parseSweepCapsJson(capsJson, caps, err)) {
    out = errorJson({"caps: " + err});
    return HGRD_GPU_EINVAL;
  }
  ParseOutcome po = parseMiniCU(src ? src : "", file ? file : "");
  if (!po.program) {
    out = errorJson(po.diagnostics);
    return HGRD_GPU_OK;
  }
  std::string fileName = po.program->file;
  auto cp = compileProgram(std::move(po.program));
  SweepResult r = enumerateVerdictOnWorkers(workers, n, *cp, caps);
  if (r.error) {
    out = errorJson({"backend: " + r.errorMessage});
    return r.error;
  }
  out = sweepResultJson(r, fileName);
  return HGRD_GPU_OK;
}

int sweepManyJson(const std::function<LaunchBackend *(int)> &workers, int n,
                  const char *jobsJson, int rank, int world, std::string &out) {
  if (world < 1 || rank < 0 || rank >= world) {
    out = errorJson({"bad rank / world"});
    return HGRD_GPU_EINVAL;
  }
  struct Job {
    std::string file, error;
    std::unique_ptr<CompiledProgram> cp;
    SweepCaps caps;
    std::vector<ExecConfig> cfgs; // this rank's configurations
    std::vector<uint64_t> index;  // their canonical indices
    uint64_t total = 0;
    size_t first = 0;             // first entry in the combined list
  };
  static const bool trace = std::getenv("HGRD_SWEEP_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto tJson = t0;
  std::vector<Job> jobs;
  try {
    JVal arr = JParse(jobsJson ? jobsJson : "[]").value();
    if (arr.kind != JVal::Arr)
      throw std::runtime_error("jobs: expected an array");
    tJson = std::chrono::steady_clock::now();
    jobs.resize(arr.arr.size());
    for (size_t q = 0; q < arr.arr.size(); ++q) {
      const JVal *file = arr.arr[q].get("file");
      jobs[q].file = file && file->kind == JVal::Str ? file->s : "prog.mcu";
      if (const JVal *c = arr.arr[q].get("caps"))
        capsFromJson(*c, jobs[q].caps);
    }
    // front end of every job (independent programs: host threads)
    parallelFor(
        jobs.size(),
        [&](size_t q) {
          Job &job = jobs[q];
          const JVal *src = arr.arr[q].get("source");
          ParseOutcome po = parseMiniCU(src && src->kind == JVal::Str ? src->s : "", job.file);
          if (!po.program) {
            job.error = errorJson(po.diagnostics);
            return;
          }
          job.cp = compileProgram(std::move(po.program));
          for (const Function &k : job.cp->program->kernels)
            job.cp->kernel(&k); // lowered here, in parallel
          const std::vector<ExecConfig> all = sweepConfigs(*job.cp, job.caps);
          job.total = all.size();
          for (size_t k = 0; k < all.size(); ++k)
            if (static_cast<int>(k % static_cast<size_t>(world)) == rank) {
              job.cfgs.push_back(all[k]);
              job.index.push_back(k);
            }
        },
        8);
  } catch (const std::exception &e) {
    out = errorJson({std::string("jobs: ") + e.what()});
    return HGRD_GPU_EINVAL;
  }
  const auto t1 = std::chrono::steady_clock::now();
  // every job's configurations in one batched run
  std::vector<ConfigJob> all;
  for (Job &j : jobs) {
    j.first = all.size();
    for (const ExecConfig &c : j.cfgs)
      all.push_back(ConfigJob{j.cp.get(), c});
  }
  LaunchBackend *b0 = workers(0);
  if (!b0) {
    out = errorJson({"no backend"});
    return HGRD_GPU_ENODEV;
  }
  std::vector<RunResult> runs;
  std::string err;
  int rc = b0->hasBatch() ? runConfigsBatched(all, *b0, sweepHostThreads(), runs, err, &workers, n)
                          : HGRD_GPU_ENOTSUP;
  if (rc == HGRD_GPU_ENOTSUP) {
    runs.clear();
    for (const ConfigJob &c : all) {
      runs.push_back(runConcrete(*c.prog, c.cfg, *b0, true));
      if (runs.back().error) {
        rc = runs.back().error;
        err = runs.back().errorMessage;
        break;
      }
    }
    if (rc == HGRD_GPU_ENOTSUP)
      rc = 0;
  }
  if (rc < 0) {
    out = errorJson({"backend: " + err});
    return rc;
  }
  const auto t2 = std::chrono::steady_clock::now();
  const size_t nJobs = jobs.size();
  // each job's report on host threads, then concatenated in job order
  std::vector<std::string> parts(nJobs);
  parallelFor(
      nJobs,
      [&](size_t q) {
    Job &j = jobs[q];
    std::string &part = parts[q];
    if (!j.error.empty()) {
      part = j.error;
      return;
    }
    if (world == 1) { // the job's enumerateVerdict result
      SweepResult sr;
      sr.configs = j.total;
      std::set<std::tuple<int, int, int, int, int, int64_t>> seen; // first wins, :883-889
      for (size_t k = 0; k < j.cfgs.size(); ++k) {
        const RunResult &r = runs[j.first + k];
        sr.stats.instances += r.stats.instances;
        sr.stats.records += r.stats.records;
        sr.stats.parLaunches += r.stats.parLaunches;
        sr.stats.seqLaunches += r.stats.seqLaunches;
        sr.stats.restarts += r.stats.restarts;
        sr.stats.batchedLaunches += r.stats.batchedLaunches;
        for (const auto &race : r.races) {
          auto key = std::make_tuple(race.locA.line, race.locA.col, race.locB.line,
                                     race.locB.col, race.kind, j.cfgs[k].warpSize);
          if (seen.insert(key).second)
            sr.races.push_back(SweepRace{race.locA, race.locB, race.kind, j.cfgs[k].warpSize});
        }
      }
      part = sweepResultJson(sr, j.file);
    } else { // this rank's share (parallel.merge_shards combines them)
      SweepShard sh;
      sh.total = j.total;
      for (size_t k = 0; k < j.cfgs.size(); ++k) {
        RunResult &r = runs[j.first + k];
        sh.stats.instances += r.stats.instances;
        sh.stats.records += r.stats.records;
        sh.stats.parLaunches += r.stats.parLaunches;
        sh.stats.seqLaunches += r.stats.seqLaunches;
        sh.stats.restarts += r.stats.restarts;
        sh.stats.batchedLaunches += r.stats.batchedLaunches;
        sh.configs.push_back(ShardConfig{j.index[k], j.cfgs[k].warpSize, std::move(r.races)});
      }
      part = sweepShardJson(sh, j.file);
    }
      },
      8);
  size_t bytes = 2;
  for (const std::string &p : parts)
    bytes += p.size() + 1;
  out.clear();
  out.reserve(bytes);
  out += "[";
  for (size_t q = 0; q < nJobs; ++q) {
    if (q)
      out += ",";
    out += parts[q];
  }
  out += "]";
  // the jobs' programs and runs are freed off the caller's critical path
  std::thread([j = std::move(jobs), r = std::move(runs), a = std::move(all)]() mutable {})
      .detach();
  if (trace) {
    auto us = [](auto a, auto b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    std::fprintf(stderr, "[hgrd many] %zu jobs: json %.0f front end %.0f run %.0f report %.0f "
                 "(us)\n", nJobs, us(t0, tJson), us(tJson, t1), us(t1, t2),
                 us(t2, std::chrono::steady_clock::now()));
  }
  return HGRD_GPU_OK;
}

int enumerateVerdictJson(LaunchBackend &be, const char *src, const char *file,
                         const char *capsJson, std::string &out) {
  SweepCaps caps;
  std::string err;
  if (!parseSweepCapsJson(capsJson, caps, err)) {
    out = errorJson({"caps: " + err});
    return HGRD_GPU_EINVAL;
  }
  ParseOutcome po = parseMiniCU(src ? src : "", file ? file : "");
  if (!po.program) {
    out = errorJson(po.diagnostics);
    return HGRD_GPU_OK;
  }
  std::string fileName = po.program->file;
  auto cp = compileProgram(std::move(po.program));
  SweepResult r = be.hasBatch() ? enumerateVerdictBatched(*cp, caps, be, sweepHostThreads())
                                : enumerateVerdict(*cp, caps, be);
  if (r.error) {
    out = errorJson({"backend: " + r.errorMessage});
    return r.error;
  }
  out = sweepResultJson(r, fileName);
  return HGRD_GPU_OK;
}

} // namespace hgrdgpu

// Reference-side binding of the B200 race-check stage (see gpu_adapter.hpp).
// Walks the reference AST (include/hgrd/ast.hpp:84-209) into the flat node
// tables of include/hgrd_gpu_program.h, calls libhgrd_gpu.so, and rebuilds
// the reference's result types (include/hgrd/oracle.hpp:27-72).
#include "gpu_adapter.hpp"
#include "gpu_adapter_flat.hpp"

#include "hgrd_gpu_program.h"

#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <variant>

namespace hgrd_gpu {

// ------------------------------------------------------------------ flatten
FlatProgram::FlatProgram(const hgrd::Program &program) : file_(program.fileName) {
  auto function = [&](const std::string &name, const std::vector<hgrd::Param> &ps,
                      const hgrd::StmtList &b, const hgrd::SourceLoc &loc, bool kernel) {
    hgrd_gpu_function f{};
    f.name = str(name);
    f.kernel = kernel ? 1 : 0;
    f.line = loc.line;
    f.col = loc.column;
    f.params_begin = static_cast<int32_t>(params_.size());
    for (const hgrd::Param &p : ps)
      params_.push_back(hgrd_gpu_param{str(p.name), static_cast<int32_t>(p.type), p.loc.line,
                                       p.loc.column});
    f.n_params = static_cast<int32_t>(ps.size());
    body(b, f.body_begin, f.n_body);
    fns_.push_back(f);
  };
  for (const hgrd::FunctionDecl &f : program.hostFunctions)
    function(f.name, f.params, f.body, f.loc, false);
  for (const hgrd::KernelDecl &k : program.kernels)
    function(k.name, k.params, k.body, k.loc, true);
  for (const std::string &s : strings_)
    strPtrs_.push_back(s.c_str());
  prog_.file_name = file_.c_str();
  prog_.strings = strPtrs_.data();
  prog_.n_strings = static_cast<uint32_t>(strPtrs_.size());
  prog_.exprs = exprs_.data();
  prog_.n_exprs = static_cast<uint32_t>(exprs_.size());
  prog_.stmts = stmts_.data();
  prog_.n_stmts = static_cast<uint32_t>(stmts_.size());
  prog_.expr_list = exprList_.data();
  prog_.n_expr_list = static_cast<uint32_t>(exprList_.size());
  prog_.stmt_list = stmtList_.data();
  prog_.n_stmt_list = static_cast<uint32_t>(stmtList_.size());
  prog_.params = params_.data();
  prog_.n_params = static_cast<uint32_t>(params_.size());
  prog_.functions = fns_.data();
  prog_.n_functions = static_cast<uint32_t>(fns_.size());
}

const hgrd::Stmt *FlatProgram::stmtById(int nodeId) const {
  auto it = byId_.find(nodeId);
  return it == byId_.end() ? nullptr : it->second;
}

int FlatProgram::str(const std::string &s) {
  auto it = strIndex_.find(s);
  if (it != strIndex_.end())
    return it->second;
  const int i = static_cast<int>(strings_.size());
  strings_.push_back(s);
  strIndex_.emplace(s, i);
  return i;
}

int FlatProgram::expr(const hgrd::Expr *e) {
  if (!e)
    return -1;
  hgrd_gpu_expr x{};
  x.line = e->loc.line;
  x.col = e->loc.column;
  x.node_id = e->nodeId;
  x.name = x.lhs = x.rhs = x.index = -1;
  std::visit(
      [&](const auto &n) {
        using T = std::decay_t<decltype(n)>;
        if constexpr (std::is_same_v<T, hgrd::IntLit>) {
          x.kind = HGRD_EXPR_INT;
          x.value = n.value;
        } else if constexpr (std::is_same_v<T, hgrd::VarRef>) {
          x.kind = HGRD_EXPR_VAR;
          x.name = str(n.name);
        } else if constexpr (std::is_same_v<T, hgrd::BuiltinRef>) {
          x.kind = HGRD_EXPR_BUILTIN;
          x.builtin = static_cast<int32_t>(n.builtin);
          x.axis = static_cast<int32_t>(n.axis);
        } else if constexpr (std::is_same_v<T, hgrd::BinaryExpr>) {
          x.kind = HGRD_EXPR_BINARY;
          x.op = static_cast<int32_t>(n.op);
          x.lhs = expr(n.lhs.get());
          x.rhs = expr(n.rhs.get());
        } else if constexpr (std::is_same_v<T, hgrd::ArrayLoad>) {
          x.kind = HGRD_EXPR_LOAD;
          x.name = str(n.array);
          x.index = expr(n.index.get());
        } else {
          x.kind = HGRD_EXPR_INPUT;
        }
      },
      e->node);
  exprs_.push_back(x);
  return static_cast<int>(exprs_.size()) - 1;
}

void FlatProgram::args(const std::vector<hgrd::ExprPtr> &a, int32_t &begin, int32_t &n) {
  std::vector<int32_t> ids;
  for (const auto &e : a)
    ids.push_back(expr(e.get()));
  begin = static_cast<int32_t>(exprList_.size());
  n = static_cast<int32_t>(ids.size());
  exprList_.insert(exprList_.end(), ids.begin(), ids.end());
}

void FlatProgram::body(const hgrd::StmtList &b, int32_t &begin, int32_t &n) {
  std::vector<int32_t> ids; // children first: a body's indices are contiguous
  for (const auto &s : b)
    ids.push_back(stmt(*s));
  begin = static_cast<int32_t>(stmtList_.size());
  n = static_cast<int32_t>(ids.size());
  stmtList_.insert(stmtList_.end(), ids.begin(), ids.end());
}

int FlatProgram::stmt(const hgrd::Stmt &s) {
  hgrd_gpu_stmt x{};
  x.line = s.loc.line;
  x.col = s.loc.column;
  x.node_id = s.nodeId;
  x.name = x.aux = -1;
  x.value = x.index = x.cmp = x.cond = x.init = x.bound = x.width = x.height = -1;
  for (int d = 0; d < 3; ++d)
    x.grid[d] = x.block[d] = -1;
  byId_[s.nodeId] = &s;
  std::visit(
      [&](const auto &n) {
        using T = std::decay_t<decltype(n)>;
        if constexpr (std::is_same_v<T, hgrd::AssignStmt>) {
          x.kind = HGRD_STMT_ASSIGN;
          x.name = str(n.name);
          x.flags = n.isDecl ? HGRD_STMT_IS_DECL : 0;
          x.decl_type = static_cast<int32_t>(n.declType);
          x.value = expr(n.value.get());
        } else if constexpr (std::is_same_v<T, hgrd::ArrayStoreStmt>) {
          x.kind = HGRD_STMT_STORE;
          x.name = str(n.array);
          x.index = expr(n.index.get());
          x.value = expr(n.value.get());
        } else if constexpr (std::is_same_v<T, hgrd::IfStmt>) {
          x.kind = HGRD_STMT_IF;
          x.cond = expr(n.cond.get());
          body(n.thenBody, x.body_begin, x.n_body);
          body(n.elseBody, x.else_begin, x.n_else);
        } else if constexpr (std::is_same_v<T, hgrd::ForStmt>) {
          x.kind = HGRD_STMT_FOR;
          x.aux = str(n.iter);
          x.flags = (n.declaresIter ? HGRD_STMT_DECLARES_ITER : 0) |
                    (n.inclusiveBound ? HGRD_STMT_INCLUSIVE : 0);
          x.step = n.step;
          x.init = expr(n.init.get());
          x.bound = expr(n.bound.get());
          body(n.body, x.body_begin, x.n_body);
        } else if constexpr (std::is_same_v<T, hgrd::BarrierStmt>) {
          x.kind = HGRD_STMT_BARRIER;
          x.sub = static_cast<int32_t>(n.kind);
        } else if constexpr (std::is_same_v<T, hgrd::FenceStmt>) {
          x.kind = HGRD_STMT_FENCE;
          x.scope = static_cast<int32_t>(n.scope);
        } else if constexpr (std::is_same_v<T, hgrd::AtomicStmt>) {
          x.kind = HGRD_STMT_ATOMIC;
          x.sub = static_cast<int32_t>(n.op);
          x.scope = static_cast<int32_t>(n.scope);
          x.name = str(n.array);
          x.index = expr(n.index.get());
          x.cmp = expr(n.compare.get());
          x.value = expr(n.value.get());
        } else if constexpr (std::is_same_v<T, hgrd::AssertStmt>) {
          x.kind = HGRD_STMT_ASSERT;
          x.cond = expr(n.cond.get());
        } else if constexpr (std::is_same_v<T, hgrd::AllocStmt>) {
          x.kind = HGRD_STMT_ALLOC;
          x.sub = static_cast<int32_t>(n.kind);
          x.name = str(n.array);
          if (n.kind == hgrd::AllocKind::MallocPitch)
            x.aux = str(n.pitchVar);
          x.width = expr(n.width.get());
          x.height = expr(n.height.get());
        } else if constexpr (std::is_same_v<T, hgrd::LaunchStmt>) {
          x.kind = HGRD_STMT_LAUNCH;
          x.name = str(n.kernel);
          for (int d = 0; d < 3; ++d) {
            x.grid[d] = expr(n.grid[static_cast<size_t>(d)].get());
            x.block[d] = expr(n.block[static_cast<size_t>(d)].get());
          }
          args(n.args, x.args_begin, x.n_args);
        } else if constexpr (std::is_same_v<T, hgrd::CallStmt>) {
          x.kind = HGRD_STMT_CALL;
          x.name = str(n.callee);
          args(n.args, x.args_begin, x.n_args);
        } else {
          x.kind = HGRD_STMT_RETURN;
          x.value = expr(n.value.get());
        }
      },
      s.node);
  stmts_.push_back(x);
  return static_cast<int>(stmts_.size()) - 1;
}

// ------------------------------------------------------------------ context
namespace {
std::mutex g_mu;
hgrd_gpu_ctx *g_ctx = nullptr;

[[noreturn]] void fail(hgrd_gpu_ctx *c, const char *what, int rc) {
  throw std::runtime_error(std::string(what) + " failed (" + std::to_string(rc) +
                           "): " + (c ? hgrd_gpu_last_error(c) : ""));
}
} // namespace

hgrd_gpu_ctx *context() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx) {
    const int rc = hgrd_gpu_create(0, &g_ctx);
    if (rc != HGRD_GPU_OK) {
      g_ctx = nullptr;
      fail(nullptr, "hgrd_gpu_create (no sm_100 device; there is no CPU fallback)", rc);
    }
  }
  return g_ctx;
}

void setContext(hgrd_gpu_ctx *ctx) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ctx = ctx;
}

// ------------------------------------------------------------------- calls
hgrd::OracleResult runConcrete(const hgrd::Program &program, const hgrd::ExecConfig &config,
                               unsigned long long *instances) {
  FlatProgram flat(program);
  hgrd_gpu_exec_config c{};
  for (int d = 0; d < 3; ++d) {
    c.grid_cap[d] = config.gridCap[static_cast<size_t>(d)];
    c.block_cap[d] = config.blockCap[static_cast<size_t>(d)];
  }
  c.warp_size = config.warpSize;
  std::vector<int64_t> inputs(config.inputs.begin(), config.inputs.end());
  c.inputs = inputs.data();
  c.n_inputs = static_cast<uint32_t>(inputs.size());
  c.max_threads = config.maxThreads;
  c.max_array_elems = config.maxArrayElems;
  c.max_steps = config.maxSteps;
  hgrd_gpu_ctx *ctx = context();
  hgrd_gpu_oracle_result *r = nullptr;
  const int rc = hgrd_gpu_run_concrete_program(ctx, flat.get(), &c, &r);
  if (rc != HGRD_GPU_OK)
    fail(ctx, "hgrd_gpu_run_concrete_program", rc);
  std::unique_ptr<hgrd_gpu_oracle_result, void (*)(hgrd_gpu_oracle_result *)> keep(
      r, hgrd_gpu_oracle_result_free);
  hgrd::OracleResult out;
  auto loc = [&](int line, int col) { return hgrd::SourceLoc{program.fileName, line, col}; };
  for (uint32_t i = 0; i < r->n_races; ++i) {
    const hgrd_gpu_observed_race &x = r->races[i];
    hgrd::ObservedRace o;
    o.locA = loc(x.line_a, x.col_a);
    o.locB = loc(x.line_b, x.col_b);
    o.kind = static_cast<hgrd::RaceKind>(x.kind);
    o.array = x.array;
    o.address = x.address;
    out.races.push_back(o);
  }
  for (uint32_t i = 0; i < r->n_traps; ++i)
    out.traps.emplace_back(r->traps[i]);
  out.launchesRun = r->launches_run;
  out.launchesSkipped = r->launches_skipped;
  out.assertStopped = r->assert_stopped != 0;
  out.indirectIndexing = r->indirect_indexing != 0;
  for (uint32_t i = 0; i < r->n_launch_records; ++i) {
    const hgrd_gpu_launch_record &x = r->launch_records[i];
    hgrd::LaunchRecord rec;
    rec.launchStmt = flat.stmtById(x.launch_node_id);
    for (int d = 0; d < 3; ++d) {
      rec.grid[static_cast<size_t>(d)] = x.grid[d];
      rec.block[static_cast<size_t>(d)] = x.block[d];
    }
    for (uint32_t k = 0; k < x.n_args; ++k) {
      rec.scalarArgs.push_back(x.scalar_args[k]);
      rec.isScalar.push_back(x.is_scalar[k] != 0);
    }
    for (uint32_t k = 0; k < x.n_defs; ++k) {
      hgrd::DefKey key;
      key.site = x.defs[k].site;
      key.aux = x.defs[k].aux;
      key.name = x.defs[k].name;
      rec.defValues.emplace(key, x.defs[k].value);
    }
    out.launchRecords.push_back(std::move(rec));
  }
  if (instances)
    *instances = r->instances;
  return out;
}

std::vector<hgrd::SweepRace> enumerateVerdict(const hgrd::Program &program,
                                              const hgrd::SweepCaps &caps) {
  FlatProgram flat(program);
  hgrd_gpu_sweep_caps c{};
  for (int d = 0; d < 3; ++d) {
    c.grid_cap[d] = caps.gridCap[static_cast<size_t>(d)];
    c.block_cap[d] = caps.blockCap[static_cast<size_t>(d)];
  }
  std::vector<int64_t> in(caps.inputSet.begin(), caps.inputSet.end());
  std::vector<int64_t> ws(caps.warpSizes.begin(), caps.warpSizes.end());
  c.input_set = in.data();
  c.n_input_set = static_cast<uint32_t>(in.size());
  c.warp_sizes = ws.data();
  c.n_warp_sizes = static_cast<uint32_t>(ws.size());
  c.max_threads = caps.maxThreads;
  c.max_configs = caps.maxConfigs;
  hgrd_gpu_ctx *ctx = context();
  hgrd_gpu_sweep_result *r = nullptr;
  const int rc = hgrd_gpu_enumerate_verdict_program(ctx, flat.get(), &c, &r);
  if (rc != HGRD_GPU_OK)
    fail(ctx, "hgrd_gpu_enumerate_verdict_program", rc);
  std::vector<hgrd::SweepRace> out;
  for (uint32_t i = 0; i < r->n_races; ++i) {
    const hgrd_gpu_sweep_race &x = r->races[i];
    hgrd::SweepRace o;
    o.locA = hgrd::SourceLoc{program.fileName, x.line_a, x.col_a};
    o.locB = hgrd::SourceLoc{program.fileName, x.line_b, x.col_b};
    o.kind = static_cast<hgrd::RaceKind>(x.kind);
    o.warpSize = x.warp_size;
    out.push_back(o);
  }
  hgrd_gpu_sweep_result_free(r);
  return out;
}

int countInputs(const hgrd::Program &program) {
  FlatProgram flat(program);
  return hgrd_gpu_count_inputs_program(flat.get());
}

} // namespace hgrd_gpu

// The reference's oracle API over the C ABI (include/hgrd_gpu_program.h):
// a caller's parsed Program (reference include/hgrd/ast.hpp), passed as flat
// node tables, is rebuilt as the host front end's AST with the caller's own
// SourceLocs and node ids, resolved (reference parser.cpp:1017-1180), and run
// through the same host mirror + B200 race-check stage as the source-text
// entry points.  Results come back as C structs owned by the library.
#include "gpu_backend.hpp"
#include "hgrd_gpu_program.h"
#include "host.hpp"
#include "minicu.hpp"

#include <cstdlib>
#include <cstring>
#include <deque>
#include <sstream>
#include <string>
#include <vector>

using namespace hgrdgpu;

namespace {

// ---------------------------------------------------------------- flat -> AST
struct Flat {
  const hgrd_gpu_program &P;
  std::vector<uint8_t> usedE, usedS; // every node is used once: the tables form a tree
  std::string err;

  explicit Flat(const hgrd_gpu_program &p)
      : P(p), usedE(p.n_exprs, 0), usedS(p.n_stmts, 0) {}

  bool fail(const std::string &m) {
    if (err.empty())
      err = m;
    return false;
  }
  bool str(int32_t i, std::string &out, bool required, const char *what) {
    if (i < 0) {
      out.clear();
      return !required || fail(std::string("missing ") + what);
    }
    if (static_cast<uint32_t>(i) >= P.n_strings || !P.strings || !P.strings[i])
      return fail(std::string("bad string index for ") + what);
    out = P.strings[i];
    return true;
  }

  ExprP expr(int32_t i, bool required, const char *what) {
    if (i < 0) {
      if (required)
        fail(std::string("missing expression: ") + what);
      return nullptr;
    }
    if (static_cast<uint32_t>(i) >= P.n_exprs || !P.exprs) {
      fail(std::string("bad expression index: ") + what);
      return nullptr;
    }
    if (usedE[static_cast<size_t>(i)]++) {
      fail("expression node used twice (the tables must form a tree)");
      return nullptr;
    }
    const hgrd_gpu_expr &x = P.exprs[i];
    auto e = std::make_unique<Expr>();
    e->loc = Loc{x.line, x.col};
    e->id = x.node_id;
    switch (x.kind) {
    case HGRD_EXPR_INT:
      e->kind = EK::Lit;
      e->value = x.value;
      break;
    case HGRD_EXPR_VAR:
      e->kind = EK::Var;
      str(x.name, e->name, true, "variable name");
      break;
    case HGRD_EXPR_BUILTIN:
      e->kind = EK::Builtin;
      if (x.builtin < 0 || x.builtin > 3 || x.axis < 0 || x.axis > 2)
        fail("bad builtin");
      e->builtin = static_cast<uint8_t>(x.builtin);
      e->axis = static_cast<uint8_t>(x.axis);
      break;
    case HGRD_EXPR_BINARY:
      e->kind = EK::Binary;
      if (x.op < HGRD_ADD || x.op > HGRD_OR)
        fail("bad binary operator");
      e->op = static_cast<Bin>(x.op);
      e->lhs = expr(x.lhs, true, "binary lhs");
      e->rhs = expr(x.rhs, true, "binary rhs");
      break;
    case HGRD_EXPR_LOAD:
      e->kind = EK::Load;
      str(x.name, e->name, true, "array name");
      e->index = expr(x.index, true, "load index");
      break;
    case HGRD_EXPR_INPUT:
      e->kind = EK::Input;
      break;
    default:
      fail("bad expression kind");
    }
    return e;
  }

  std::vector<ExprP> exprList(int32_t begin, int32_t n, const char *what) {
    std::vector<ExprP> v;
    if (n < 0 || begin < 0 || static_cast<uint64_t>(begin) + static_cast<uint64_t>(n) >
                                  static_cast<uint64_t>(P.n_expr_list)) {
      if (n != 0)
        fail(std::string("bad argument range: ") + what);
      return v;
    }
    for (int32_t k = 0; k < n; ++k)
      v.push_back(expr(P.expr_list[begin + k], true, what));
    return v;
  }

  Body body(int32_t begin, int32_t n) {
    Body b;
    if (n == 0)
      return b;
    if (n < 0 || begin < 0 ||
        static_cast<uint64_t>(begin) + static_cast<uint64_t>(n) >
            static_cast<uint64_t>(P.n_stmt_list)) {
      fail("bad statement-list range");
      return b;
    }
    for (int32_t k = 0; k < n && err.empty(); ++k)
      if (StmtP s = stmt(P.stmt_list[begin + k]))
        b.push_back(std::move(s));
    return b;
  }

  StmtP stmt(int32_t i) {
    if (i < 0 || static_cast<uint32_t>(i) >= P.n_stmts || !P.stmts) {
      fail("bad statement index");
      return nullptr;
    }
    if (usedS[static_cast<size_t>(i)]++) {
      fail("statement node used twice (the tables must form a tree)");
      return nullptr;
    }
    const hgrd_gpu_stmt &x = P.stmts[i];
    auto s = std::make_unique<Stmt>();
    s->loc = Loc{x.line, x.col};
    s->id = x.node_id;
    switch (x.kind) {
    case HGRD_STMT_ASSIGN:
      s->kind = SK::Assign;
      str(x.name, s->name, true, "assignment target");
      s->isDecl = (x.flags & HGRD_STMT_IS_DECL) != 0;
      if (x.decl_type < 0 || x.decl_type > 3)
        fail("bad declaration type");
      s->declType = static_cast<VarType>(x.decl_type);
      s->value = expr(x.value, false, "assigned value");
      break;
    case HGRD_STMT_STORE:
      s->kind = SK::Store;
      str(x.name, s->name, true, "store array");
      s->index = expr(x.index, true, "store index");
      s->value = expr(x.value, true, "stored value");
      break;
    case HGRD_STMT_IF:
      s->kind = SK::If;
      s->cond = expr(x.cond, true, "if condition");
      s->body = body(x.body_begin, x.n_body);
      s->elseBody = body(x.else_begin, x.n_else);
      break;
    case HGRD_STMT_FOR:
      s->kind = SK::For;
      str(x.aux, s->aux, true, "loop iterator");
      s->declaresIter = (x.flags & HGRD_STMT_DECLARES_ITER) != 0;
      s->inclusive = (x.flags & HGRD_STMT_INCLUSIVE) != 0;
      s->step = x.step;
      if (x.step <= 0)
        fail("loop step must be positive");
      s->init = expr(x.init, true, "loop init");
      s->bound = expr(x.bound, true, "loop bound");
      s->body = body(x.body_begin, x.n_body);
      break;
    case HGRD_STMT_BARRIER:
      if (x.sub != 0 && x.sub != 1)
        fail("bad barrier kind");
      s->kind = x.sub == 0 ? SK::SyncThreads : SK::SyncWarp;
      break;
    case HGRD_STMT_FENCE:
      s->kind = SK::Fence;
      if (x.scope < 1 || x.scope > 2)
        fail("bad fence scope");
      s->scope = static_cast<Scope>(x.scope);
      break;
    case HGRD_STMT_ATOMIC:
      s->kind = SK::Atomic;
      if (x.sub < 0 || x.sub > 2 || x.scope < 1 || x.scope > 2)
        fail("bad atomic");
      s->aop = static_cast<AtomicOp>(x.sub);
      s->scope = static_cast<Scope>(x.scope);
      str(x.name, s->name, true, "atomic array");
      s->index = expr(x.index, true, "atomic index");
      if (s->aop == AtomicOp::Cas)
        s->cmp = expr(x.cmp, true, "CAS compare");
      s->value = expr(x.value, true, "atomic value");
      break;
    case HGRD_STMT_ASSERT:
      s->kind = SK::Assert;
      s->cond = expr(x.cond, true, "assert condition");
      break;
    case HGRD_STMT_ALLOC:
      s->kind = SK::Alloc;
      if (x.sub != 0 && x.sub != 1)
        fail("bad allocation kind");
      s->pitch = x.sub == 1;
      str(x.name, s->name, true, "allocation target");
      str(x.aux, s->aux, s->pitch, "pitch variable");
      s->width = expr(x.width, true, "allocation width");
      if (s->pitch)
        s->height = expr(x.height, true, "allocation height");
      break;
    case HGRD_STMT_LAUNCH:
      s->kind = SK::Launch;
      str(x.name, s->name, true, "launched kernel");
      for (int d = 0; d < 3; ++d) {
        s->grid[d] = expr(x.grid[d], true, "grid dimension");
        s->block[d] = expr(x.block[d], true, "block dimension");
      }
      s->args = exprList(x.args_begin, x.n_args, "launch argument");
      break;
    case HGRD_STMT_CALL:
      s->kind = SK::Call;
      str(x.name, s->name, true, "callee");
      s->args = exprList(x.args_begin, x.n_args, "call argument");
      break;
    case HGRD_STMT_RETURN:
      s->kind = SK::Return;
      s->value = expr(x.value, false, "return value");
      break;
    default:
      fail("bad statement kind");
    }
    return s;
  }
};

std::unique_ptr<Program> buildProgram(const hgrd_gpu_program *p, std::string &err) {
  if (!p || (!p->functions && p->n_functions)) {
    err = "no program";
    return nullptr;
  }
  Flat F(*p);
  auto prog = std::make_unique<Program>();
  prog->file = p->file_name ? p->file_name : "";
  for (uint32_t i = 0; i < p->n_functions && F.err.empty(); ++i) {
    const hgrd_gpu_function &x = p->functions[i];
    Function f;
    F.str(x.name, f.name, true, "function name");
    f.kernel = x.kernel != 0;
    f.loc = Loc{x.line, x.col};
    if (x.n_params < 0 || x.params_begin < 0 ||
        static_cast<uint64_t>(x.params_begin) + static_cast<uint64_t>(x.n_params) >
            static_cast<uint64_t>(p->n_params)) {
      F.fail("bad parameter range");
      break;
    }
    for (int32_t k = 0; k < x.n_params; ++k) {
      const hgrd_gpu_param &q = p->params[x.params_begin + k];
      Param prm;
      F.str(q.name, prm.name, true, "parameter name");
      if (q.type < 0 || q.type > 3)
        F.fail("bad parameter type");
      prm.type = static_cast<VarType>(q.type);
      prm.loc = Loc{q.line, q.col};
      f.params.push_back(std::move(prm));
    }
    f.body = F.body(x.body_begin, x.n_body);
    (f.kernel ? prog->kernels : prog->hosts).push_back(std::move(f));
  }
  if (!F.err.empty()) {
    err = F.err;
    return nullptr;
  }
  std::vector<std::string> diags = resolveMiniCU(*prog);
  if (!diags.empty()) {
    err = diags.front();
    return nullptr;
  }
  return prog;
}

// ------------------------------------------------------------- canonical dump
void dumpExpr(std::ostringstream &o, const Expr *e) {
  if (!e) {
    o << "_";
    return;
  }
  o << "(E" << static_cast<int>(e->kind) << "#" << e->id << "@" << e->loc.line << ":"
    << e->loc.col;
  switch (e->kind) {
  case EK::Lit:
    o << " " << e->value;
    break;
  case EK::Var:
    o << " " << e->name;
    break;
  case EK::Builtin:
    o << " b" << int(e->builtin) << "." << int(e->axis);
    break;
  case EK::Binary:
    o << " op" << int(e->op) << " ";
    dumpExpr(o, e->lhs.get());
    o << " ";
    dumpExpr(o, e->rhs.get());
    break;
  case EK::Load:
    o << " " << e->name << "[";
    dumpExpr(o, e->index.get());
    o << "]";
    break;
  case EK::Input:
    break;
  }
  o << ")";
}

void dumpBody(std::ostringstream &o, const Body &b);

void dumpStmt(std::ostringstream &o, const Stmt &s) {
  o << "(S" << static_cast<int>(s.kind) << "#" << s.id << "@" << s.loc.line << ":" << s.loc.col
    << " n=" << s.name << " a=" << s.aux << " d" << s.isDecl << " t" << int(s.declType) << " p"
    << s.pitch << " i" << s.inclusive << " di" << s.declaresIter << " st" << s.step << " op"
    << int(s.aop) << " sc" << int(s.scope);
  const Expr *xs[] = {s.value.get(), s.index.get(), s.cmp.get(),   s.cond.get(),
                      s.init.get(),  s.bound.get(), s.width.get(), s.height.get()};
  for (const Expr *x : xs) {
    o << " ";
    dumpExpr(o, x);
  }
  if (s.kind == SK::Launch)
    for (int d = 0; d < 3; ++d) {
      o << " g";
      dumpExpr(o, s.grid[d].get());
      o << " b";
      dumpExpr(o, s.block[d].get());
    }
  o << " args[";
  for (const auto &a : s.args) {
    dumpExpr(o, a.get());
    o << ",";
  }
  o << "] {";
  dumpBody(o, s.body);
  o << "} else {";
  dumpBody(o, s.elseBody);
  o << "})";
}

void dumpBody(std::ostringstream &o, const Body &b) {
  for (const auto &s : b) {
    dumpStmt(o, *s);
    o << "\n";
  }
}

std::string dumpProgram(const Program &p) {
  std::ostringstream o;
  o << "file " << p.file << "\n";
  for (const auto *fs : {&p.hosts, &p.kernels})
    for (const Function &f : *fs) {
      o << (f.kernel ? "kernel " : "host ") << f.name << "@" << f.loc.line << ":" << f.loc.col
        << "(";
      for (const Param &q : f.params)
        o << q.name << ":" << int(q.type) << "@" << q.loc.line << ":" << q.loc.col << ",";
      o << ") {\n";
      dumpBody(o, f.body);
      o << "}\n";
    }
  return o.str();
}

char *dupStr(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  if (p)
    std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// ------------------------------------------------------------ result storage
struct OracleHolder {
  hgrd_gpu_oracle_result pub{}; // first member: the pointer handed out
  std::deque<std::string> strs; // stable c_str() pointers
  std::vector<hgrd_gpu_observed_race> races;
  std::vector<const char *> traps;
  std::vector<hgrd_gpu_launch_record> recs;
  std::deque<std::vector<int64_t>> args;
  std::deque<std::vector<uint8_t>> isScalar;
  std::deque<std::vector<hgrd_gpu_def_value>> defs;

  const char *keep(const std::string &s) {
    strs.push_back(s);
    return strs.back().c_str();
  }
};

struct SweepHolder {
  hgrd_gpu_sweep_result pub{};
  std::vector<hgrd_gpu_sweep_race> races;
};

ExecConfig execConfig(const hgrd_gpu_exec_config &c) {
  ExecConfig e;
  for (int d = 0; d < 3; ++d) {
    e.gridCap[d] = c.grid_cap[d];
    e.blockCap[d] = c.block_cap[d];
  }
  e.warpSize = c.warp_size;
  e.inputs.assign(c.inputs, c.inputs + (c.inputs ? c.n_inputs : 0));
  e.maxThreads = c.max_threads;
  e.maxArrayElems = c.max_array_elems;
  e.maxSteps = c.max_steps;
  return e;
}

} // namespace

extern "C" {

int hgrd_gpu_run_concrete_program(hgrd_gpu_ctx *ctx, const hgrd_gpu_program *program,
                                  const hgrd_gpu_exec_config *config,
                                  hgrd_gpu_oracle_result **out) {
  if (!ctx || !config || !out)
    return HGRD_GPU_EINVAL;
  *out = nullptr;
  std::string err;
  std::unique_ptr<Program> prog = buildProgram(program, err);
  if (!prog) {
    setError(ctx, "program: " + err);
    return HGRD_GPU_EINVAL;
  }
  auto cp = compileProgram(std::move(prog));
  GpuBackend be(ctx);
  RunResult r = runConcrete(*cp, execConfig(*config), be);
  if (r.error) {
    setError(ctx, "backend: " + r.errorMessage);
    return r.error;
  }
  auto *h = new OracleHolder();
  for (const Race &x : r.races) {
    hgrd_gpu_observed_race o{};
    o.line_a = x.locA.line;
    o.col_a = x.locA.col;
    o.line_b = x.locB.line;
    o.col_b = x.locB.col;
    o.kind = x.kind;
    o.array = h->keep(x.array);
    o.address = x.address;
    o.thread_a = x.threadX;
    o.thread_b = x.threadY;
    o.launch = x.launch;
    h->races.push_back(o);
  }
  for (const std::string &t : r.traps)
    h->traps.push_back(h->keep(t));
  for (const LaunchRec &l : r.launchRecords) {
    hgrd_gpu_launch_record o{};
    o.launch_node_id = l.site;
    for (int d = 0; d < 3; ++d) {
      o.grid[d] = l.grid[d];
      o.block[d] = l.block[d];
    }
    h->args.push_back(l.scalarArgs);
    h->isScalar.emplace_back(l.isScalar.begin(), l.isScalar.end());
    o.scalar_args = h->args.back().data();
    o.is_scalar = h->isScalar.back().data();
    o.n_args = static_cast<uint32_t>(l.scalarArgs.size());
    std::vector<hgrd_gpu_def_value> dv;
    for (const auto &[key, v] : l.defValues)
      dv.push_back(hgrd_gpu_def_value{key.first, key.second, h->keep(v.name), v.value});
    h->defs.push_back(std::move(dv));
    o.defs = h->defs.back().data();
    o.n_defs = static_cast<uint32_t>(h->defs.back().size());
    h->recs.push_back(o);
  }
  hgrd_gpu_oracle_result &p = h->pub;
  p.races = h->races.data();
  p.n_races = static_cast<uint32_t>(h->races.size());
  p.traps = h->traps.data();
  p.n_traps = static_cast<uint32_t>(h->traps.size());
  p.launches_run = r.launchesRun;
  p.launches_skipped = r.launchesSkipped;
  p.assert_stopped = r.assertStopped;
  p.indirect_indexing = r.indirectIndexing;
  p.launch_records = h->recs.data();
  p.n_launch_records = static_cast<uint32_t>(h->recs.size());
  p.instances = r.stats.instances;
  *out = &h->pub;
  return HGRD_GPU_OK;
}

void hgrd_gpu_oracle_result_free(hgrd_gpu_oracle_result *r) {
  delete reinterpret_cast<OracleHolder *>(r);
}

int hgrd_gpu_enumerate_verdict_program(hgrd_gpu_ctx *ctx, const hgrd_gpu_program *program,
                                       const hgrd_gpu_sweep_caps *caps,
                                       hgrd_gpu_sweep_result **out) {
  if (!ctx || !caps || !out)
    return HGRD_GPU_EINVAL;
  *out = nullptr;
  std::string err;
  std::unique_ptr<Program> prog = buildProgram(program, err);
  if (!prog) {
    setError(ctx, "program: " + err);
    return HGRD_GPU_EINVAL;
  }
  auto cp = compileProgram(std::move(prog));
  SweepCaps sc;
  for (int d = 0; d < 3; ++d) {
    sc.gridCap[d] = caps->grid_cap[d];
    sc.blockCap[d] = caps->block_cap[d];
  }
  sc.inputSet.assign(caps->input_set, caps->input_set + (caps->input_set ? caps->n_input_set : 0));
  sc.warpSizes.assign(caps->warp_sizes,
                      caps->warp_sizes + (caps->warp_sizes ? caps->n_warp_sizes : 0));
  sc.maxThreads = caps->max_threads;
  sc.maxConfigs = caps->max_configs;
  SweepWorkers pool(ctx); // (batched unless HGRD_SWEEP_BATCH=0, as the JSON entry point)
  SweepResult r = enumerateVerdictOnWorkers(pool.getter(), pool.n, *cp, sc);
  if (r.error) {
    setError(ctx, "backend: " + r.errorMessage);
    return r.error;
  }
  auto *h = new SweepHolder();
  for (const SweepRace &x : r.races)
    h->races.push_back(hgrd_gpu_sweep_race{x.locA.line, x.locA.col, x.locB.line, x.locB.col,
                                           x.kind, x.warpSize});
  h->pub.races = h->races.data();
  h->pub.n_races = static_cast<uint32_t>(h->races.size());
  h->pub.configs = r.configs;
  *out = &h->pub;
  return HGRD_GPU_OK;
}

void hgrd_gpu_sweep_result_free(hgrd_gpu_sweep_result *r) {
  delete reinterpret_cast<SweepHolder *>(r);
}

int hgrd_gpu_count_inputs_program(const hgrd_gpu_program *program) {
  std::string err;
  std::unique_ptr<Program> prog = buildProgram(program, err);
  return prog ? countInputs(*prog) : HGRD_GPU_EINVAL;
}

int hgrd_gpu_program_dump(const hgrd_gpu_program *program, char **out) {
  if (!out)
    return HGRD_GPU_EINVAL;
  std::string err;
  std::unique_ptr<Program> prog = buildProgram(program, err);
  *out = dupStr(prog ? dumpProgram(*prog) : "error: " + err);
  return prog ? HGRD_GPU_OK : HGRD_GPU_EINVAL;
}

int hgrd_gpu_source_dump(const char *source, const char *file_name, char **out) {
  if (!out)
    return HGRD_GPU_EINVAL;
  ParseOutcome po = parseMiniCU(source ? source : "", file_name ? file_name : "");
  if (!po.program) {
    *out = dupStr("error: " + (po.diagnostics.empty() ? std::string("?") : po.diagnostics[0]));
    return HGRD_GPU_EINVAL;
  }
  *out = dupStr(dumpProgram(*po.program));
  return HGRD_GPU_OK;
}

} // extern "C"

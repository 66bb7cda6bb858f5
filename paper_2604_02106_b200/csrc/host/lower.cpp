// MiniCU kernel -> register bytecode (include/hgrd_gpu.h).
//
// Semantics follow the reference thread interpreter
// (reference src/oracle.cpp:482-646) statement by statement:
//  * every executed statement charges one step, every loop test one more
//    (:561, :630);
//  * kernel binary operators evaluate the RIGHT operand first (:500, GCC
//    argument order), comparisons/logic yield 0/1 without short circuit;
//  * stores: index, value, bounds check, record (:569-575);
//    atomics: index, value, compare, bounds check, record (:580-586);
//  * for: init once; each iteration step + bound re-evaluated, iterator
//    variable set from a hidden counter, counter += step; afterwards the
//    iterator holds the final counter (:627-641);
//  * return stops the thread without evaluating its value (:643-644);
//  * unknown / never-assigned names read 0 (:485-487).
#include "lower.hpp"

#include <algorithm>
#include <functional>
#include <set>

namespace hgrdgpu {

namespace {

class Lowerer {
public:
  explicit Lowerer(const Function &k) : k_(k) {}

  LoweredKernel run() {
    out_.fn = &k_;
    collectNames();
    tempBase_ = static_cast<int>(slots_.size());
    out_.paramReg.assign(k_.params.size(), -1);
    for (size_t i = 0; i < k_.params.size(); ++i)
      if (k_.params[i].type == VarType::Int)
        out_.paramReg[i] = slots_.at(k_.params[i].name);
    for (const auto &s : k_.body)
      stmt(*s);
    emit(HGRD_OP_END);
    // Patch returns to the final END.
    for (size_t at : returnJumps_)
      out_.code[at].imm = static_cast<int64_t>(out_.code.size() - 1);
    out_.nRegs = static_cast<uint32_t>(tempBase_ + maxTemps_);
    finalizeLocs();
    analyzeRelevance();
    for (auto &insn : out_.code)
      if (insn.op == HGRD_OP_LOAD && out_.siteValueNeeded[insn.imm])
        insn.sub |= 1;
    return std::move(out_);
  }

private:
  // ---- named registers ----
  void nameSlot(const std::string &n) {
    if (!slots_.count(n))
      slots_.emplace(n, static_cast<int>(slots_.size()));
  }
  void collectNamesExpr(const Expr &e) {
    switch (e.kind) {
    case EK::Var:
      nameSlot(e.name);
      break;
    case EK::Binary:
      collectNamesExpr(*e.lhs);
      collectNamesExpr(*e.rhs);
      break;
    case EK::Load:
      collectNamesExpr(*e.index);
      break;
    default:
      break;
    }
  }
  void collectNamesBody(const Body &b) {
    for (const auto &sp : b) {
      const Stmt &s = *sp;
      switch (s.kind) {
      case SK::Assign:
        nameSlot(s.name);
        if (s.value)
          collectNamesExpr(*s.value);
        break;
      case SK::Store:
      case SK::Atomic:
        collectNamesExpr(*s.index);
        collectNamesExpr(*s.value);
        if (s.cmp)
          collectNamesExpr(*s.cmp);
        break;
      case SK::If:
        collectNamesExpr(*s.cond);
        collectNamesBody(s.body);
        collectNamesBody(s.elseBody);
        break;
      case SK::For:
        nameSlot(s.aux);
        nameSlot("\x01for" + std::to_string(s.id)); // hidden counter
        collectNamesExpr(*s.init);
        collectNamesExpr(*s.bound);
        collectNamesBody(s.body);
        break;
      default:
        break;
      }
    }
  }
  void collectNames() {
    for (const auto &p : k_.params)
      if (p.type == VarType::Int)
        nameSlot(p.name);
    collectNamesBody(k_.body);
  }

  // ---- emission ----
  size_t emit(uint8_t op, uint8_t sub = 0, int a = 0, int b = 0, int c = 0,
              int64_t imm = 0) {
    hgrd_gpu_insn i{};
    i.op = op;
    i.sub = sub;
    i.a = static_cast<uint16_t>(a);
    i.b = static_cast<uint16_t>(b);
    i.c = static_cast<uint16_t>(c);
    i.imm = imm;
    out_.code.push_back(i);
    return out_.code.size() - 1;
  }
  int temp() {
    int r = tempBase_ + tempTop_++;
    maxTemps_ = std::max(maxTemps_, tempTop_);
    return r;
  }
  int newSite(const Loc &loc, const std::string &array, uint8_t kind,
              uint8_t aop, Scope scope) {
    hgrd_gpu_site s{};
    s.loc = -1;
    int param = -1;
    for (size_t i = 0; i < k_.params.size(); ++i)
      if (k_.params[i].name == array && isArray(k_.params[i].type))
        param = static_cast<int>(i);
    s.param = param;
    s.kind = kind;
    s.atomic_op = aop;
    s.scope = static_cast<uint8_t>(scope);
    out_.sites.push_back(s);
    out_.siteArray.push_back(array);
    out_.siteLoc.push_back(loc);
    return static_cast<int>(out_.sites.size() - 1);
  }

  int expr(const Expr &e) {
    switch (e.kind) {
    case EK::Lit: {
      int r = temp();
      emit(HGRD_OP_CONST, 0, r, 0, 0, e.value);
      return r;
    }
    case EK::Var:
      return slots_.at(e.name);
    case EK::Builtin: {
      int r = temp();
      emit(HGRD_OP_BUILTIN, static_cast<uint8_t>(e.builtin * 3 + e.axis), r);
      return r;
    }
    case EK::Binary: {
      int rr = expr(*e.rhs); // right operand first (reference :500 under GCC)
      int lr = expr(*e.lhs);
      int r = temp();
      emit(HGRD_OP_BIN, static_cast<uint8_t>(e.op), r, lr, rr);
      return r;
    }
    case EK::Load: {
      int ir = expr(*e.index);
      int site = newSite(e.loc, e.name, HGRD_SITE_LOAD, 0, Scope::None);
      loadSite_[&e] = site;
      int r = temp();
      emit(HGRD_OP_LOAD, 0, r, ir, 0, site);
      return r;
    }
    case EK::Input:
    default: {
      int r = temp(); // rejected in kernels by the resolver
      emit(HGRD_OP_CONST, 0, r, 0, 0, 0);
      return r;
    }
    }
  }

  int stepId(const Loc &l) {
    out_.stmtLocs.push_back(l);
    return static_cast<int>(out_.stmtLocs.size() - 1);
  }

  void body(const Body &b) {
    for (const auto &s : b)
      stmt(*s);
  }

  void stmt(const Stmt &s) {
    const int savedTop = tempTop_;
    const int sid = stepId(s.loc);
    emit(HGRD_OP_STEP, 0, 0, 0, 0, sid);
    switch (s.kind) {
    case SK::Assign: {
      int v;
      if (s.value) {
        v = expr(*s.value);
      } else {
        v = temp();
        emit(HGRD_OP_CONST, 0, v, 0, 0, 0);
      }
      emit(HGRD_OP_MOV, 0, slots_.at(s.name), v);
      break;
    }
    case SK::Store: {
      int ir = expr(*s.index);
      int vr = expr(*s.value);
      int site = newSite(s.loc, s.name, HGRD_SITE_STORE, 0, Scope::None);
      stmtSite_[&s] = site;
      emit(HGRD_OP_STORE, 0, ir, vr, 0, site);
      break;
    }
    case SK::Atomic: {
      int ir = expr(*s.index);
      int vr = expr(*s.value);
      int cr;
      if (s.cmp) {
        cr = expr(*s.cmp);
      } else {
        cr = temp();
        emit(HGRD_OP_CONST, 0, cr, 0, 0, 0);
      }
      int site = newSite(s.loc, s.name, HGRD_SITE_ATOMIC,
                         static_cast<uint8_t>(s.aop), s.scope);
      stmtSite_[&s] = site;
      emit(HGRD_OP_ATOMIC, 0, ir, vr, cr, site);
      break;
    }
    case SK::SyncThreads:
      emit(HGRD_OP_SYNCTHREADS);
      break;
    case SK::SyncWarp:
      emit(HGRD_OP_SYNCWARP);
      break;
    case SK::Fence:
      emit(HGRD_OP_FENCE, static_cast<uint8_t>(s.scope));
      break;
    case SK::If: {
      int cr = expr(*s.cond);
      size_t jz = emit(HGRD_OP_JZ, 0, cr);
      tempTop_ = savedTop;
      body(s.body);
      size_t jmp = emit(HGRD_OP_JMP);
      out_.code[jz].imm = static_cast<int64_t>(out_.code.size());
      body(s.elseBody);
      out_.code[jmp].imm = static_cast<int64_t>(out_.code.size());
      break;
    }
    case SK::For: {
      const int ctr = slots_.at("\x01for" + std::to_string(s.id));
      const int iter = slots_.at(s.aux);
      int ir = expr(*s.init);
      emit(HGRD_OP_MOV, 0, ctr, ir);
      tempTop_ = savedTop;
      const size_t top = out_.code.size();
      emit(HGRD_OP_STEP, 0, 0, 0, 0, sid); // loop test (reference :630)
      int br = expr(*s.bound);
      int cr = temp();
      emit(HGRD_OP_BIN, static_cast<uint8_t>(s.inclusive ? Bin::Le : Bin::Lt),
           cr, ctr, br);
      size_t jz = emit(HGRD_OP_JZ, 0, cr);
      emit(HGRD_OP_MOV, 0, iter, ctr);
      tempTop_ = savedTop;
      body(s.body);
      int st = temp();
      emit(HGRD_OP_CONST, 0, st, 0, 0, s.step);
      emit(HGRD_OP_BIN, static_cast<uint8_t>(Bin::Add), ctr, ctr, st);
      emit(HGRD_OP_JMP, 0, 0, 0, 0, static_cast<int64_t>(top));
      out_.code[jz].imm = static_cast<int64_t>(out_.code.size());
      emit(HGRD_OP_MOV, 0, iter, ctr);
      break;
    }
    case SK::Return:
      returnJumps_.push_back(emit(HGRD_OP_JMP));
      break;
    default:
      break; // host-only statements are rejected in kernels by the parser
    }
    tempTop_ = savedTop;
  }

  void finalizeLocs() {
    std::vector<Loc> all(out_.siteLoc.begin(), out_.siteLoc.end());
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    out_.locs = all;
    for (size_t i = 0; i < out_.sites.size(); ++i)
      out_.sites[i].loc = static_cast<int32_t>(
          std::lower_bound(all.begin(), all.end(), out_.siteLoc[i]) - all.begin());
  }

  // ---- value relevance (flow-insensitive fixpoint over named locals) ----
  using Sites = std::set<int>;
  Sites valueLoads(const Expr &e) {
    switch (e.kind) {
    case EK::Var: {
      auto it = varLoads_.find(e.name);
      return it == varLoads_.end() ? Sites{} : it->second;
    }
    case EK::Binary: {
      Sites a = valueLoads(*e.lhs), b = valueLoads(*e.rhs);
      a.insert(b.begin(), b.end());
      return a;
    }
    case EK::Load:
      return Sites{loadSite_.at(&e)};
    default:
      return {};
    }
  }
  bool flowAssign(const std::string &name, const Sites &from) {
    Sites &dst = varLoads_[name];
    size_t before = dst.size();
    dst.insert(from.begin(), from.end());
    return dst.size() != before;
  }
  bool propagateBody(const Body &b) {
    bool changed = false;
    for (const auto &sp : b) {
      const Stmt &s = *sp;
      if (s.kind == SK::Assign && s.value)
        changed |= flowAssign(s.name, valueLoads(*s.value));
      else if (s.kind == SK::If)
        changed |= propagateBody(s.body) | propagateBody(s.elseBody);
      else if (s.kind == SK::For)
        changed |= flowAssign(s.aux, valueLoads(*s.init)) | propagateBody(s.body);
    }
    return changed;
  }
  void sink(const Expr &e, Sites &rel) {
    Sites s = valueLoads(e);
    rel.insert(s.begin(), s.end());
  }
  void sinksInExpr(const Expr &e, Sites &rel) {
    if (e.kind == EK::Binary) {
      sinksInExpr(*e.lhs, rel);
      sinksInExpr(*e.rhs, rel);
    } else if (e.kind == EK::Load) {
      sink(*e.index, rel);
      sinksInExpr(*e.index, rel);
    }
  }
  void sinksInBody(const Body &b, Sites &rel) {
    for (const auto &sp : b) {
      const Stmt &s = *sp;
      switch (s.kind) {
      case SK::Assign:
        if (s.value)
          sinksInExpr(*s.value, rel);
        break;
      case SK::Store:
      case SK::Atomic:
        sink(*s.index, rel);
        sinksInExpr(*s.index, rel);
        sinksInExpr(*s.value, rel);
        if (s.cmp)
          sinksInExpr(*s.cmp, rel);
        break;
      case SK::If:
        sink(*s.cond, rel);
        sinksInExpr(*s.cond, rel);
        sinksInBody(s.body, rel);
        sinksInBody(s.elseBody, rel);
        break;
      case SK::For:
        sink(*s.init, rel);
        sink(*s.bound, rel);
        sinksInExpr(*s.init, rel);
        sinksInExpr(*s.bound, rel);
        sinksInBody(s.body, rel);
        break;
      case SK::Fence:
        hasFence_ = true;
        break;
      default:
        break;
      }
      if (s.kind == SK::Atomic && s.aop != AtomicOp::Add)
        hasCasExch_ = true;
    }
  }
  void analyzeRelevance() {
    while (propagateBody(k_.body)) {
    }
    Sites rel;
    sinksInBody(k_.body, rel);
    out_.siteValueNeeded.assign(out_.sites.size(), false);
    for (int s : rel)
      out_.siteValueNeeded[s] = true;
    out_.hasLocks = hasFence_ && hasCasExch_;
  }

  const Function &k_;
  LoweredKernel out_;
  std::map<std::string, int> slots_;
  int tempBase_ = 0, tempTop_ = 0, maxTemps_ = 0;
  std::vector<size_t> returnJumps_;
  std::map<const Expr *, int> loadSite_;
  std::map<const Stmt *, int> stmtSite_;
  std::map<std::string, Sites> varLoads_;
  bool hasFence_ = false, hasCasExch_ = false;
};

} // namespace

LoweredKernel lowerKernel(const Function &kernel) { return Lowerer(kernel).run(); }

} // namespace hgrdgpu

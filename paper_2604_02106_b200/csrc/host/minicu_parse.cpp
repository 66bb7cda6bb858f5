// MiniCU tokenizer, recursive-descent parser and resolver.
// Grammar: reference docs/minicu-grammar.md:9-68.  Node-id / location rules
// that race reports depend on are listed in minicu.hpp.
#include "minicu.hpp"

#include <cctype>
#include <map>
#include <set>
#include <stdexcept>

namespace hgrdgpu {

const Function *Program::findKernel(const std::string &n) const {
  for (const auto &k : kernels)
    if (k.name == n)
      return &k;
  return nullptr;
}
const Function *Program::findHost(const std::string &n) const {
  for (const auto &f : hosts)
    if (f.name == n)
      return &f;
  return nullptr;
}

namespace {

enum class T : uint8_t {
  End, Ident, Num, LPar, RPar, LBrace, RBrace, LBrack, RBrack, Comma, Semi,
  Amp, Assign, Plus, Minus, Star, Slash, Percent, Lt, Le, Gt, Ge, Eq, Ne,
  AndAnd, OrOr, Dot, Inc, LaunchL, LaunchR
};

struct Tok {
  T t = T::End;
  std::string s;
  int64_t n = 0;
  Loc loc;
};

// Whole-input tokenization.  A character outside the alphabet ends the
// token stream exactly like end of input (the reference lexer returns its
// End token for it, parser.cpp:225-228).
// ASCII classes (the "C" locale's, without the libc calls)
inline bool isSpace(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }
inline bool isAlpha(char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z'); }
inline bool isDigit(char c) { return c >= '0' && c <= '9'; }

std::vector<Tok> tokenize(const std::string &src) {
  std::vector<Tok> out;
  out.reserve(src.size() / 3 + 8);
  size_t i = 0;
  int line = 1, col = 1;
  auto bump = [&] {
    if (i < src.size()) {
      if (src[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
      ++i;
    }
  };
  auto at = [&](size_t k) -> char { return k < src.size() ? src[k] : '\0'; };
  for (;;) {
    // whitespace and comments
    for (;;) {
      if (i >= src.size())
        break;
      char c = src[i];
      if (isSpace(c)) {
        bump();
      } else if (c == '/' && at(i + 1) == '/') {
        while (i < src.size() && src[i] != '\n')
          bump();
      } else if (c == '/' && at(i + 1) == '*') {
        bump();
        bump();
        while (i + 1 < src.size() && !(src[i] == '*' && src[i + 1] == '/'))
          bump();
        bump();
        bump();
      } else {
        break;
      }
    }
    Tok tk;
    tk.loc = Loc{line, col};
    if (i >= src.size()) {
      out.push_back(std::move(tk));
      return out;
    }
    char c = src[i];
    if (isAlpha(c) || c == '_') {
      size_t b = i;
      while (i < src.size() &&
             (isAlpha(src[i]) || isDigit(src[i]) || src[i] == '_'))
        bump();
      tk.t = T::Ident;
      tk.s = src.substr(b, i - b);
      out.push_back(std::move(tk));
      continue;
    }
    if (isDigit(c)) {
      size_t b = i;
      while (i < src.size() && isDigit(src[i]))
        bump();
      tk.t = T::Num;
      tk.s = src.substr(b, i - b);
      tk.n = std::stoll(tk.s);
      out.push_back(std::move(tk));
      continue;
    }
    struct Multi {
      const char *text;
      T t;
    };
    static const Multi multis[] = {{"<<<", T::LaunchL}, {">>>", T::LaunchR},
                                   {"<=", T::Le},       {">=", T::Ge},
                                   {"==", T::Eq},       {"!=", T::Ne},
                                   {"&&", T::AndAnd},   {"||", T::OrOr},
                                   {"++", T::Inc}};
    bool matched = false;
    for (const auto &m : multis) {
      if (m.text[0] != c)
        continue; // cheap first-character filter
      size_t len = std::char_traits<char>::length(m.text);
      if (src.compare(i, len, m.text) == 0) {
        for (size_t k = 0; k < len; ++k)
          bump();
        tk.t = m.t;
        matched = true;
        break;
      }
    }
    if (matched) {
      out.push_back(std::move(tk));
      continue;
    }
    static const std::string singles = "(){}[],;&=+-*/%<>.";
    static const T singleT[] = {T::LPar,  T::RPar,   T::LBrace,  T::RBrace,
                                T::LBrack, T::RBrack, T::Comma,   T::Semi,
                                T::Amp,   T::Assign, T::Plus,    T::Minus,
                                T::Star,  T::Slash,  T::Percent, T::Lt,
                                T::Gt,    T::Dot};
    size_t p = singles.find(c);
    if (p == std::string::npos) {
      out.push_back(std::move(tk)); // End
      return out;
    }
    bump();
    tk.t = singleT[p];
    out.push_back(std::move(tk));
  }
}

struct SyntaxFail {
  Loc loc;
  std::string msg;
};

class Parser {
public:
  Parser(const std::string &src, std::string file)
      : toks_(tokenize(src)), file_(std::move(file)) {}

  ParseOutcome run() {
    ParseOutcome out;
    auto prog = std::make_unique<Program>();
    prog->file = file_;
    try {
      while (cur().t != T::End)
        topLevel(*prog);
      resolveProgram(*prog);
    } catch (const SyntaxFail &f) {
      out.diagnostics.push_back(diag(f.loc, "syntax error", f.msg));
      return out;
    }
    if (!diags_.empty()) {
      out.diagnostics = diags_;
      return out;
    }
    out.program = std::move(prog);
    return out;
  }

  // The resolver alone, over a program built elsewhere (the flat-program
  // ABI, include/hgrd_gpu_program.h).
  std::vector<std::string> resolveOnly(Program &p) {
    resolveProgram(p);
    return diags_;
  }

private:
  std::string diag(const Loc &l, const char *kind, const std::string &m) {
    return file_ + ":" + std::to_string(l.line) + ":" + std::to_string(l.col) +
           ": " + kind + ": " + m;
  }
  const Tok &cur() const { return toks_[pos_]; }
  bool is(T t) const { return cur().t == t; }
  bool isWord(const char *w) const { return cur().t == T::Ident && cur().s == w; }
  const Tok &take() {
    const Tok &t = toks_[pos_];
    if (pos_ + 1 < toks_.size())
      ++pos_;
    return t;
  }
  [[noreturn]] void failAt(const Loc &l, const std::string &m) {
    throw SyntaxFail{l, m};
  }
  [[noreturn]] void fail(const std::string &m) { failAt(cur().loc, m); }
  const Tok &need(T t, const char *what) {
    if (!is(t))
      fail(std::string("expected ") + what);
    return take();
  }
  bool eat(T t) {
    if (!is(t))
      return false;
    take();
    return true;
  }
  int nextId() { return ++ids_; }

  ExprP expr(EK k, Loc l) {
    auto e = std::make_unique<Expr>();
    e->kind = k;
    e->loc = l;
    return e;
  }
  ExprP seal(ExprP e) {
    e->id = nextId();
    return e;
  }
  ExprP lit(Loc l, int64_t v) {
    auto e = expr(EK::Lit, l);
    e->value = v;
    return seal(std::move(e));
  }
  StmtP stmt(SK k, Loc l) {
    auto s = std::make_unique<Stmt>();
    s->kind = k;
    s->loc = l;
    return s;
  }
  StmtP seal(StmtP s) {
    s->id = nextId();
    return s;
  }

  static bool typeWord(const std::string &w) {
    return w == "int" || w == "float" || w == "lock";
  }
  static bool varType(const std::string &ty, bool ptr, VarType &out) {
    if (ty == "int")
      out = ptr ? VarType::IntArray : VarType::Int;
    else if (ty == "float" && ptr)
      out = VarType::FloatArray;
    else if (ty == "lock" && ptr)
      out = VarType::LockArray;
    else
      return false;
    return true;
  }

  // ---- top level ----
  void topLevel(Program &prog) {
    Function f;
    if (isWord("__global__")) {
      take();
      if (!isWord("void"))
        fail("expected 'void' after '__global__'");
      take();
      f.kernel = true;
    } else if (isWord("void") || isWord("int")) {
      bool isInt = cur().s == "int";
      take();
      if (isInt && is(T::Star))
        fail("top-level array declarations are not supported");
    } else {
      fail("expected a kernel or host function declaration");
    }
    f.loc = cur().loc;
    f.name = need(T::Ident, f.kernel ? "kernel name" : "function name").s;
    f.params = params();
    f.body = block(f.kernel);
    (f.kernel ? prog.kernels : prog.hosts).push_back(std::move(f));
  }

  std::vector<Param> params() {
    need(T::LPar, "'('");
    std::vector<Param> ps;
    if (eat(T::RPar))
      return ps;
    do {
      Param p;
      p.loc = cur().loc;
      if (!is(T::Ident))
        fail("expected parameter type");
      std::string ty = take().s;
      bool ptr = eat(T::Star);
      if (!varType(ty, ptr, p.type))
        failAt(p.loc, "unsupported parameter type '" + ty + (ptr ? "*" : "") + "'");
      p.name = need(T::Ident, "parameter name").s;
      ps.push_back(std::move(p));
    } while (eat(T::Comma));
    need(T::RPar, "')'");
    return ps;
  }

  Body block(bool k) {
    need(T::LBrace, "'{'");
    Body b;
    while (!is(T::RBrace)) {
      if (is(T::End))
        fail("unexpected end of input inside block");
      b.push_back(statement(k));
    }
    take();
    return b;
  }

  // ---- statements ----
  StmtP statement(bool k) {
    Loc l = cur().loc;
    if (!is(T::Ident))
      fail("expected a statement");
    const std::string w = cur().s;
    if (w == "if")
      return ifStmt(k);
    if (w == "for")
      return forStmt(k);
    if (w == "return") {
      take();
      auto s = stmt(SK::Return, l);
      if (!is(T::Semi))
        s->value = parseExpr();
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (w == "__syncthreads" || w == "__syncwarp" || w == "__threadfence" ||
        w == "__threadfence_block") {
      if (!k)
        failAt(l, w + " is kernel-only");
      StmtP s;
      if (w == "__syncthreads")
        s = stmt(SK::SyncThreads, l);
      else if (w == "__syncwarp")
        s = stmt(SK::SyncWarp, l);
      else {
        s = stmt(SK::Fence, l);
        s->scope = w == "__threadfence" ? Scope::Device : Scope::Block;
      }
      take();
      need(T::LPar, "'('");
      need(T::RPar, "')'");
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (w.compare(0, 6, "atomic") == 0)
      return atomicStmt(k);
    if (w == "assert") {
      if (k)
        failAt(l, "assert is host-only");
      take();
      need(T::LPar, "'('");
      auto s = stmt(SK::Assert, l);
      s->cond = parseExpr();
      need(T::RPar, "')'");
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (w == "cudaMalloc" || w == "cudaMallocPitch")
      return allocStmt(k);
    if (typeWord(w))
      return declStmt(k);
    return identStmt(k);
  }

  StmtP declStmt(bool k) {
    Loc l = cur().loc;
    std::string ty = take().s;
    bool ptr = eat(T::Star);
    auto s = stmt(SK::Assign, l);
    s->isDecl = true;
    if (!varType(ty, ptr, s->declType))
      failAt(l, "unsupported declaration type");
    if (k && ptr)
      failAt(l, "array declarations are host-only; kernels receive arrays as "
                "parameters");
    s->name = need(T::Ident, "variable name").s;
    if (eat(T::Assign)) {
      if (ptr)
        failAt(l, "array variables are initialized by cudaMalloc");
      s->value = parseExpr();
    }
    need(T::Semi, "';'");
    return seal(std::move(s));
  }

  void dim3(ExprP (&d)[3]) {
    if (is(T::LPar)) {
      Loc l = cur().loc;
      take();
      ExprP first = parseExpr();
      if (eat(T::Comma)) {
        d[0] = std::move(first);
        d[1] = parseExpr();
        need(T::Comma, "','");
        d[2] = parseExpr();
        need(T::RPar, "')'");
        return;
      }
      need(T::RPar, "')'");
      d[0] = std::move(first);
      d[1] = lit(l, 1);
      d[2] = lit(l, 1);
      return;
    }
    Loc l = cur().loc;
    d[0] = parseExpr();
    d[1] = lit(l, 1);
    d[2] = lit(l, 1);
  }

  void argList(std::vector<ExprP> &args) {
    if (is(T::RPar))
      return;
    do
      args.push_back(parseExpr());
    while (eat(T::Comma));
  }

  StmtP identStmt(bool k) {
    Loc l = cur().loc;
    std::string name = take().s;
    if (eat(T::LBrack)) {
      auto s = stmt(SK::Store, l);
      s->name = name;
      s->index = parseExpr();
      need(T::RBrack, "']'");
      need(T::Assign, "'='");
      s->value = parseExpr();
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (eat(T::Assign)) {
      auto s = stmt(SK::Assign, l);
      s->name = name;
      s->value = parseExpr();
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (is(T::LaunchL)) {
      if (k)
        failAt(l, "kernel launch is host-only");
      take();
      auto s = stmt(SK::Launch, l);
      s->name = name;
      dim3(s->grid);
      need(T::Comma, "','");
      dim3(s->block);
      need(T::LaunchR, "'>>>'");
      need(T::LPar, "'('");
      argList(s->args);
      need(T::RPar, "')'");
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    if (is(T::LPar)) {
      if (k)
        failAt(l, "function calls are not allowed in kernels");
      take();
      auto s = stmt(SK::Call, l);
      s->name = name;
      argList(s->args);
      need(T::RPar, "')'");
      need(T::Semi, "';'");
      return seal(std::move(s));
    }
    fail("expected '=', '[', '(' or '<<<' after identifier");
  }

  StmtP atomicStmt(bool k) {
    Loc l = cur().loc;
    std::string name = take().s;
    if (!k)
      failAt(l, "atomic operations are kernel-only");
    auto s = stmt(SK::Atomic, l);
    std::string base = name;
    const std::string suffix = "_block";
    if (base.size() > suffix.size() &&
        base.compare(base.size() - suffix.size(), suffix.size(), suffix) == 0) {
      s->scope = Scope::Block;
      base.resize(base.size() - suffix.size());
    } else {
      s->scope = Scope::Device;
    }
    if (base == "atomicCAS")
      s->aop = AtomicOp::Cas;
    else if (base == "atomicExch")
      s->aop = AtomicOp::Exch;
    else if (base == "atomicAdd")
      s->aop = AtomicOp::Add;
    else
      failAt(l, "unknown intrinsic '" + name + "'");
    need(T::LPar, "'('");
    s->name = need(T::Ident, "array name").s;
    need(T::LBrack, "'['");
    s->index = parseExpr();
    need(T::RBrack, "']'");
    need(T::Comma, "','");
    if (s->aop == AtomicOp::Cas) {
      s->cmp = parseExpr();
      need(T::Comma, "','");
    }
    s->value = parseExpr();
    need(T::RPar, "')'");
    need(T::Semi, "';'");
    return seal(std::move(s));
  }

  StmtP allocStmt(bool k) {
    Loc l = cur().loc;
    std::string name = take().s;
    if (k)
      failAt(l, name + " is host-only");
    auto s = stmt(SK::Alloc, l);
    s->pitch = name == "cudaMallocPitch";
    need(T::LPar, "'('");
    need(T::Amp, "'&'");
    s->name = need(T::Ident, "array name").s;
    need(T::Comma, "','");
    if (s->pitch) {
      need(T::Amp, "'&'");
      s->aux = need(T::Ident, "pitch variable").s;
      need(T::Comma, "','");
      s->width = parseExpr();
      need(T::Comma, "','");
      s->height = parseExpr();
    } else {
      s->width = parseExpr();
    }
    need(T::RPar, "')'");
    need(T::Semi, "';'");
    return seal(std::move(s));
  }

  StmtP ifStmt(bool k) {
    Loc l = cur().loc;
    take();
    need(T::LPar, "'('");
    auto s = stmt(SK::If, l);
    s->cond = parseExpr();
    need(T::RPar, "')'");
    s->body = block(k);
    if (isWord("else")) {
      take();
      s->elseBody = block(k);
    }
    return seal(std::move(s));
  }

  StmtP forStmt(bool k) {
    Loc l = cur().loc;
    take();
    need(T::LPar, "'('");
    auto s = stmt(SK::For, l);
    if (isWord("int")) {
      take();
      s->declaresIter = true;
    }
    s->aux = need(T::Ident, "loop iterator").s;
    need(T::Assign, "'='");
    s->init = parseExpr();
    need(T::Semi, "';'");
    if (need(T::Ident, "loop iterator").s != s->aux)
      failAt(l, "loop condition must test the iterator '" + s->aux + "'");
    if (is(T::Lt))
      s->inclusive = false;
    else if (is(T::Le))
      s->inclusive = true;
    else
      fail("loop condition must be '<' or '<='");
    take();
    s->bound = parseExpr();
    need(T::Semi, "';'");
    if (need(T::Ident, "loop iterator").s != s->aux)
      failAt(l, "loop update must assign the iterator");
    if (eat(T::Inc)) {
      s->step = 1;
    } else {
      need(T::Assign, "'='");
      if (need(T::Ident, "iterator").s != s->aux)
        failAt(l, "loop update must be 'i = i + <constant>' or 'i++'");
      need(T::Plus, "'+'");
      s->step = need(T::Num, "step constant").n;
      if (s->step <= 0)
        failAt(l, "loop step must be positive");
    }
    need(T::RPar, "')'");
    s->body = block(k);
    return seal(std::move(s));
  }

  // ---- expressions: C precedence, left associative ----
  ExprP parseExpr() { return binaryLevel(0); }

  // levels: 0 ||, 1 &&, 2 == !=, 3 < <= > >=, 4 + -, 5 * / %
  static bool opAt(int level, T t, Bin &op) {
    switch (level) {
    case 0:
      if (t == T::OrOr) { op = Bin::Or; return true; }
      return false;
    case 1:
      if (t == T::AndAnd) { op = Bin::And; return true; }
      return false;
    case 2:
      if (t == T::Eq) { op = Bin::Eq; return true; }
      if (t == T::Ne) { op = Bin::Ne; return true; }
      return false;
    case 3:
      if (t == T::Lt) { op = Bin::Lt; return true; }
      if (t == T::Le) { op = Bin::Le; return true; }
      if (t == T::Gt) { op = Bin::Gt; return true; }
      if (t == T::Ge) { op = Bin::Ge; return true; }
      return false;
    case 4:
      if (t == T::Plus) { op = Bin::Add; return true; }
      if (t == T::Minus) { op = Bin::Sub; return true; }
      return false;
    default:
      if (t == T::Star) { op = Bin::Mul; return true; }
      if (t == T::Slash) { op = Bin::Div; return true; }
      if (t == T::Percent) { op = Bin::Mod; return true; }
      return false;
    }
  }

  ExprP binaryLevel(int level) {
    if (level > 5)
      return unary();
    ExprP lhs = binaryLevel(level + 1);
    Bin op;
    while (opAt(level, cur().t, op)) {
      Loc l = cur().loc;
      take();
      auto e = expr(EK::Binary, l);
      e->op = op;
      e->lhs = std::move(lhs);
      e->rhs = binaryLevel(level + 1);
      if (op == Bin::Div || op == Bin::Mod) {
        if (e->rhs->kind != EK::Lit)
          throwDivisor(l, "division and modulo require a constant divisor");
        if (e->rhs->value <= 0)
          throwDivisor(l, "division and modulo require a positive divisor");
      }
      lhs = seal(std::move(e));
    }
    return lhs;
  }

  [[noreturn]] void throwDivisor(const Loc &l, const std::string &m) {
    // Reported as DiagKind::NonConstantDivisor by the reference; the kind
    // only changes the diagnostic text, never acceptance.
    throw SyntaxFail{l, m};
  }

  ExprP unary() {
    if (is(T::Minus)) {
      Loc l = cur().loc;
      take();
      ExprP inner = unary();
      if (inner->kind == EK::Lit)
        return lit(l, -inner->value);
      ExprP zero = lit(l, 0);
      auto e = expr(EK::Binary, l);
      e->op = Bin::Sub;
      e->lhs = std::move(zero);
      e->rhs = std::move(inner);
      return seal(std::move(e));
    }
    return primary();
  }

  ExprP primary() {
    Loc l = cur().loc;
    if (is(T::Num)) {
      int64_t v = take().n;
      return lit(l, v);
    }
    if (eat(T::LPar)) {
      ExprP e = parseExpr();
      need(T::RPar, "')'");
      return e;
    }
    if (!is(T::Ident))
      fail("expected an expression");
    std::string name = take().s;
    if (name == "__input") {
      need(T::LPar, "'('");
      need(T::RPar, "')'");
      return seal(expr(EK::Input, l));
    }
    static const char *builtins[] = {"threadIdx", "blockIdx", "blockDim",
                                     "gridDim"};
    for (int b = 0; b < 4; ++b) {
      if (name != builtins[b])
        continue;
      need(T::Dot, "'.'");
      Tok ax = need(T::Ident, "axis (x, y or z)");
      auto e = expr(EK::Builtin, l);
      e->builtin = static_cast<uint8_t>(b);
      if (ax.s == "x")
        e->axis = 0;
      else if (ax.s == "y")
        e->axis = 1;
      else if (ax.s == "z")
        e->axis = 2;
      else
        failAt(ax.loc, "axis must be x, y or z");
      return seal(std::move(e));
    }
    if (eat(T::LBrack)) {
      auto e = expr(EK::Load, l);
      e->name = name;
      e->index = parseExpr();
      need(T::RBrack, "']'");
      return seal(std::move(e));
    }
    auto e = expr(EK::Var, l);
    e->name = name;
    return seal(std::move(e));
  }

  // ---- resolution (reference parser.cpp:1017-1180) ----
  using Scope_ = std::map<std::string, VarType>;

  void note(const Loc &l, const char *kind, const std::string &m) {
    diags_.push_back(diag(l, kind, m));
  }

  void resolveProgram(Program &p) {
    int entries = 0;
    for (const auto &f : p.hosts)
      entries += f.name == "main";
    if (entries != 1)
      note(Loc{1, 1}, "syntax error", "expected exactly one entry function 'main'");
    std::set<std::string> names;
    for (const auto &k : p.kernels)
      if (!names.insert(k.name).second)
        note(k.loc, "syntax error", "duplicate kernel '" + k.name + "'");
    for (const auto &f : p.hosts)
      if (!names.insert(f.name).second)
        note(f.loc, "syntax error", "duplicate function '" + f.name + "'");
    for (const auto &k : p.kernels) {
      Scope_ sc;
      std::set<std::string> seen;
      for (const auto &prm : k.params) {
        if (!seen.insert(prm.name).second)
          note(prm.loc, "syntax error",
               "duplicate parameter '" + prm.name + "' in kernel " + k.name);
        sc[prm.name] = prm.type;
      }
      resolveBody(p, k.body, sc, true);
    }
    for (const auto &f : p.hosts) {
      Scope_ sc;
      for (const auto &prm : f.params)
        sc[prm.name] = prm.type;
      resolveBody(p, f.body, sc, false);
    }
  }

  void resolveBody(const Program &p, const Body &b, Scope_ &sc, bool k) {
    bool afterReturn = false;
    for (const auto &s : b) {
      if (afterReturn) {
        note(s->loc, "unreachable code", "statement is unreachable after return");
        afterReturn = false;
      }
      resolveStmt(p, *s, sc, k);
      if (s->kind == SK::Return)
        afterReturn = true;
    }
  }

  void wantArray(const Scope_ &sc, const std::string &n, const Loc &l) {
    auto it = sc.find(n);
    if (it == sc.end())
      note(l, "unbound identifier", "use of undeclared array '" + n + "'");
    else if (!isArray(it->second))
      note(l, "type error", "'" + n + "' is not an array");
  }

  void resolveStmt(const Program &p, const Stmt &s, Scope_ &sc, bool k) {
    switch (s.kind) {
    case SK::Assign: {
      if (s.value)
        resolveExpr(*s.value, sc, k);
      if (s.isDecl) {
        sc[s.name] = s.declType;
      } else {
        auto it = sc.find(s.name);
        if (it == sc.end())
          note(s.loc, "unbound identifier",
               "assignment to undeclared variable '" + s.name + "'");
        else if (isArray(it->second))
          note(s.loc, "type error", "cannot assign to array variable '" + s.name + "'");
      }
      return;
    }
    case SK::Store:
      wantArray(sc, s.name, s.loc);
      resolveExpr(*s.index, sc, k);
      resolveExpr(*s.value, sc, k);
      return;
    case SK::If: {
      resolveExpr(*s.cond, sc, k);
      Scope_ t = sc;
      resolveBody(p, s.body, t, k);
      Scope_ e = sc;
      resolveBody(p, s.elseBody, e, k);
      return;
    }
    case SK::For: {
      resolveExpr(*s.init, sc, k);
      resolveExpr(*s.bound, sc, k);
      Scope_ inner = sc;
      if (s.declaresIter)
        inner[s.aux] = VarType::Int;
      else if (!sc.count(s.aux))
        note(s.loc, "unbound identifier", "loop iterator '" + s.aux + "' is not declared");
      resolveBody(p, s.body, inner, k);
      return;
    }
    case SK::Atomic:
      wantArray(sc, s.name, s.loc);
      resolveExpr(*s.index, sc, k);
      if (s.cmp)
        resolveExpr(*s.cmp, sc, k);
      resolveExpr(*s.value, sc, k);
      return;
    case SK::Assert:
      resolveExpr(*s.cond, sc, k);
      return;
    case SK::Alloc: {
      auto it = sc.find(s.name);
      if (it == sc.end())
        note(s.loc, "unbound identifier", "allocation target '" + s.name + "' is not declared");
      else if (!isArray(it->second))
        note(s.loc, "type error", "allocation target '" + s.name + "' is not an array");
      if (s.pitch) {
        auto pit = sc.find(s.aux);
        if (pit == sc.end())
          note(s.loc, "unbound identifier", "pitch variable '" + s.aux + "' is not declared");
        else if (pit->second != VarType::Int)
          note(s.loc, "type error", "pitch variable '" + s.aux + "' must be int");
      }
      resolveExpr(*s.width, sc, k);
      if (s.height)
        resolveExpr(*s.height, sc, k);
      return;
    }
    case SK::Launch: {
      const Function *kern = p.findKernel(s.name);
      if (!kern) {
        note(s.loc, "unbound identifier", "launch of unknown kernel '" + s.name + "'");
      } else if (kern->params.size() != s.args.size()) {
        note(s.loc, "type error", "kernel '" + s.name + "' has the wrong arity");
      } else {
        for (size_t i = 0; i < s.args.size(); ++i) {
          const Expr &a = *s.args[i];
          bool want = isArray(kern->params[i].type);
          bool have = a.kind == EK::Var && sc.count(a.name) && isArray(sc.at(a.name));
          if (want != have)
            note(a.loc, "type error",
                 "argument " + std::to_string(i + 1) + " of '" + s.name +
                     "' has the wrong kind");
        }
      }
      for (const auto &d : s.grid)
        resolveExpr(*d, sc, k);
      for (const auto &d : s.block)
        resolveExpr(*d, sc, k);
      for (const auto &a : s.args)
        resolveExpr(*a, sc, k);
      return;
    }
    case SK::Call: {
      const Function *callee = p.findHost(s.name);
      if (!callee)
        note(s.loc, "unbound identifier", "call to unknown function '" + s.name + "'");
      else if (callee->params.size() != s.args.size())
        note(s.loc, "type error", "function '" + s.name + "' has the wrong arity");
      for (const auto &a : s.args)
        resolveExpr(*a, sc, k);
      return;
    }
    case SK::Return:
      if (s.value)
        resolveExpr(*s.value, sc, k);
      return;
    default:
      return; // barriers and fences
    }
  }

  void resolveExpr(const Expr &e, const Scope_ &sc, bool k) {
    switch (e.kind) {
    case EK::Var:
      if (!sc.count(e.name))
        note(e.loc, "unbound identifier", "use of undeclared variable '" + e.name + "'");
      return;
    case EK::Builtin:
      if (!k)
        note(e.loc, "type error", "thread builtins are kernel-only");
      return;
    case EK::Input:
      if (k)
        note(e.loc, "type error", "__input() is host-only");
      return;
    case EK::Binary:
      resolveExpr(*e.lhs, sc, k);
      resolveExpr(*e.rhs, sc, k);
      return;
    case EK::Load:
      wantArray(sc, e.name, e.loc);
      resolveExpr(*e.index, sc, k);
      return;
    default:
      return;
    }
  }

  std::vector<Tok> toks_;
  size_t pos_ = 0;
  std::string file_;
  int ids_ = 0;
  std::vector<std::string> diags_;
};

} // namespace

std::vector<std::string> resolveMiniCU(Program &p) { return Parser("", p.file).resolveOnly(p); }

ParseOutcome parseMiniCU(const std::string &source, const std::string &file) {
  try {
    return Parser(source, file).run();
  } catch (const std::out_of_range &) {
    ParseOutcome o;
    o.diagnostics.push_back(file + ": integer literal out of range");
    return o;
  }
}

} // namespace hgrdgpu

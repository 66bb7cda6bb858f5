// MiniCU front end used by the host side of the race-check stage.
//
// The reference keeps its front end in C++ (reference src/parser.cpp,
// include/hgrd/ast.hpp); its sources cannot travel with this library, so
// this is an independent implementation of the same dialect
// (reference docs/minicu-grammar.md) that reproduces the properties the
// race check depends on bit for bit:
//   * SourceLoc of every node: a statement's loc is its first token
//     (parser.cpp:543-555), a load's loc is the array-name token
//     (:918-923), a binary node's loc is its operator token (:825-838);
//   * node ids in construction (post-) order, including the synthetic
//     nodes of `-x` -> `0 - x` (:865-879) and scalar dim3 -> (e,1,1)
//     (:604-632); host DefKeys (LaunchRecord.defValues) are keyed by them;
//   * the resolver's acceptance set (:1024-1180).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace hgrdgpu {

struct Loc {
  int line = 0;
  int col = 0;
};
inline bool operator==(const Loc &a, const Loc &b) {
  return a.line == b.line && a.col == b.col;
}
inline bool operator<(const Loc &a, const Loc &b) {
  return a.line != b.line ? a.line < b.line : a.col < b.col;
}

enum class Bin : uint8_t { Add, Sub, Mul, Div, Mod, Lt, Le, Gt, Ge, Eq, Ne, And, Or };
enum class Scope : uint8_t { None = 0, Block = 1, Device = 2 };
enum class AtomicOp : uint8_t { Cas = 0, Exch = 1, Add = 2 };
enum class VarType : uint8_t { Int, FloatArray, IntArray, LockArray };
inline bool isArray(VarType t) { return t != VarType::Int; }

struct Expr;
using ExprP = std::unique_ptr<Expr>;

enum class EK : uint8_t { Lit, Var, Builtin, Binary, Load, Input };

struct Expr {
  EK kind = EK::Lit;
  Loc loc;
  int id = 0;
  int64_t value = 0;       // Lit
  std::string name;        // Var name / Load array
  uint8_t builtin = 0;     // Builtin: 0 threadIdx 1 blockIdx 2 blockDim 3 gridDim
  uint8_t axis = 0;        // Builtin axis
  Bin op = Bin::Add;       // Binary
  ExprP lhs, rhs;          // Binary
  ExprP index;             // Load
  int site = -1;           // Load: kernel access-site id (filled by lowering)
};

struct Stmt;
using StmtP = std::unique_ptr<Stmt>;
using Body = std::vector<StmtP>;

enum class SK : uint8_t {
  Assign, Store, If, For, SyncThreads, SyncWarp, Fence, Atomic, Assert,
  Alloc, Launch, Call, Return
};

struct Stmt {
  SK kind = SK::Assign;
  Loc loc;
  int id = 0;
  // Assign: name = value (value may be null for a plain declaration)
  // Store: name[index] = value;   Atomic: name[index] (cmp) value
  // Alloc: name (array), pitchVar, width, height (pitch only)
  // Launch: name (kernel), grid[3], block[3], args;  Call: name, args
  // For: iter, init, bound, step, inclusive, body;  If: cond, body, elseBody
  std::string name;
  std::string aux; // For iterator / pitch variable
  bool isDecl = false;
  VarType declType = VarType::Int;
  bool pitch = false;
  bool inclusive = false;
  bool declaresIter = false;
  int64_t step = 1;
  AtomicOp aop = AtomicOp::Add;
  Scope scope = Scope::Device;
  ExprP value, index, cmp, cond, init, bound, width, height;
  ExprP grid[3], block[3];
  std::vector<ExprP> args;
  Body body, elseBody;
  int site = -1; // Store/Atomic: kernel access-site id (filled by lowering)
};

struct Param {
  std::string name;
  VarType type = VarType::Int;
  Loc loc;
};

struct Function {
  std::string name;
  std::vector<Param> params;
  Body body;
  Loc loc;
  bool kernel = false;
};

struct Program {
  std::string file;
  std::vector<Function> hosts;
  std::vector<Function> kernels;
  const Function *findKernel(const std::string &n) const;
  const Function *findHost(const std::string &n) const;
};

struct ParseOutcome {
  std::unique_ptr<Program> program; // null on error
  std::vector<std::string> diagnostics;
};

ParseOutcome parseMiniCU(const std::string &source, const std::string &file);
// The resolver's diagnostics for a program built without the parser (empty:
// accepted), reference parser.cpp:1017-1180.
std::vector<std::string> resolveMiniCU(Program &p);

} // namespace hgrdgpu

// The reference's parsed Program (reference include/hgrd/ast.hpp) as the flat
// node tables of include/hgrd_gpu_program.h.  Used by gpu_adapter.cpp and its
// tests.
#pragma once

#include "hgrd/ast.hpp"
#include "hgrd_gpu_program.h"

#include <map>
#include <string>
#include <vector>

namespace hgrd_gpu {

class FlatProgram {
public:
  explicit FlatProgram(const hgrd::Program &program);
  FlatProgram(const FlatProgram &) = delete;
  FlatProgram &operator=(const FlatProgram &) = delete;

  const hgrd_gpu_program *get() const { return &prog_; }
  // node id -> the reference statement (LaunchRecord::launchStmt)
  const hgrd::Stmt *stmtById(int nodeId) const;

private:
  int str(const std::string &s);
  int expr(const hgrd::Expr *e);
  int stmt(const hgrd::Stmt &s);
  void body(const hgrd::StmtList &b, int32_t &begin, int32_t &n);
  void args(const std::vector<hgrd::ExprPtr> &a, int32_t &begin, int32_t &n);

  std::string file_;
  std::vector<std::string> strings_;
  std::map<std::string, int> strIndex_;
  std::vector<const char *> strPtrs_;
  std::vector<hgrd_gpu_expr> exprs_;
  std::vector<hgrd_gpu_stmt> stmts_;
  std::vector<int32_t> exprList_, stmtList_;
  std::vector<hgrd_gpu_param> params_;
  std::vector<hgrd_gpu_function> fns_;
  std::map<int, const hgrd::Stmt *> byId_;
  hgrd_gpu_program prog_{};
};

} // namespace hgrd_gpu

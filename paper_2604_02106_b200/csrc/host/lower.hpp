// Kernel lowering: MiniCU kernel body -> hgrd_gpu bytecode + access-site
// table, plus the static facts the race-check stage needs per kernel.
#pragma once

#include "hgrd_gpu.h"
#include "minicu.hpp"

#include <map>
#include <string>
#include <vector>

namespace hgrdgpu {

struct LoweredKernel {
  const Function *fn = nullptr;
  std::vector<hgrd_gpu_insn> code;
  std::vector<hgrd_gpu_site> sites;
  std::vector<std::string> siteArray; // parameter name used by the access
  std::vector<Loc> siteLoc;
  std::vector<Loc> locs;              // loc id -> source location (sorted)
  std::vector<Loc> stmtLocs;          // STEP imm -> statement location
  std::vector<int> paramReg;          // scalar param -> register, else -1
  uint32_t nRegs = 0;
  // Value relevance (reference SURVEY §7 hard part 2): load sites whose
  // loaded value can reach an index, an if condition or a loop init/bound
  // through locals.  Only these values decide which accesses happen.
  std::vector<bool> siteValueNeeded;
  bool hasLocks = false; // a fence plus CAS/Exch: lockInfo can order pairs
};

LoweredKernel lowerKernel(const Function &kernel);

} // namespace hgrdgpu

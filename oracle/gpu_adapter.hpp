// Reference-side binding of the B200 race-check stage: the reference's own
// oracle API (reference include/hgrd/oracle.hpp:57, 75, 79) with identical
// signatures and result types, backed by libhgrd_gpu.so through the C ABI of
// include/hgrd_gpu_program.h.  A maintainer of the reference adds
// gpu_adapter.{hpp,cpp} to its build and links libhgrd_gpu.so; callers switch
// from hgrd::runConcrete to hgrd_gpu::runConcrete.
//
// In this repository the adapter is compiled against the reference headers
// by oracle/Makefile (it needs /root/reference) and serves as TEST
// INFRASTRUCTURE: tests/test_adapter.py diffs it in-process against
// hgrd::runConcrete / hgrd::enumerateVerdict.  The product library never
// links it.
#pragma once

#include "hgrd/oracle.hpp"
#include "hgrd_gpu.h"

#include <vector>

namespace hgrd_gpu {

// The context the calls below run on (device 0, created on first use; or
// the one installed by setContext).  Throws std::runtime_error when no
// sm_100 device is present: there is no CPU fallback.
hgrd_gpu_ctx *context();
void setContext(hgrd_gpu_ctx *ctx);

// reference include/hgrd/oracle.hpp:57 — same signature and result.
// Extra: `instances` (when non-null) receives the access instances checked.
hgrd::OracleResult runConcrete(const hgrd::Program &program, const hgrd::ExecConfig &config,
                               unsigned long long *instances = nullptr);

// reference include/hgrd/oracle.hpp:75
std::vector<hgrd::SweepRace> enumerateVerdict(const hgrd::Program &program,
                                              const hgrd::SweepCaps &caps);

// reference include/hgrd/oracle.hpp:79 (no GPU needed)
int countInputs(const hgrd::Program &program);

} // namespace hgrd_gpu

// Reference-shaped C ABI entry points of libhgrd_gpu.so: the host front end
// (csrc/host) driving the B200 race-check stage (csrc/gpu) through the
// device-buffer / check-launch ABI of include/hgrd_gpu.h.
#include "hgrd_gpu.h"
#include "host.hpp"
#include "gpu/affine.hpp"
#include "gpu/jit.hpp"
#include "gpu_backend.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>
#include <cstring>

using namespace hgrdgpu;


namespace {

char *dup(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  if (p)
    std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

} // namespace

extern "C" {

int hgrd_gpu_run_concrete_json(hgrd_gpu_ctx *ctx, const char *source,
                               const char *file_name, const char *cfg_json,
                               char **out) {
  if (!ctx || !out)
    return HGRD_GPU_EINVAL;
  GpuBackend be(ctx);
  std::string s;
  int rc = runConcreteJson(be, source, file_name, cfg_json, s);
  *out = dup(s);
  return rc;
}

int hgrd_gpu_enumerate_verdict_json(hgrd_gpu_ctx *ctx, const char *source,
                                    const char *file_name, const char *caps_json,
                                    char **out) {
  if (!ctx || !out)
    return HGRD_GPU_EINVAL;
  // Batched (default): the configurations' host runs speculated on host
  // threads and all their launches checked by one k_batch launch on this
  // context; configurations that cannot be speculated run exactly on the
  // worker contexts meanwhile (enumerateVerdictBatched).  HGRD_SWEEP_BATCH=0:
  // per-launch checks spread over the worker contexts (own streams and
  // buffers on the same GPU, one host thread each).
  SweepWorkers pool(ctx);
  std::string s;
  int rc = enumerateVerdictJsonParallel(pool.getter(), pool.n, source, file_name, caps_json, s);
  *out = dup(s);
  return rc;
}

int hgrd_gpu_enumerate_verdict_many_json(hgrd_gpu_ctx *ctx, const char *jobs_json, int rank,
                                         int world, char **out) {
  if (!ctx || !out)
    return HGRD_GPU_EINVAL;
  static const bool trace = std::getenv("HGRD_SWEEP_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  {
    SweepWorkers pool(ctx);
    std::string s;
    rc = sweepManyJson(pool.getter(), pool.n, jobs_json, rank, world, s);
    *out = dup(s);
  }
  if (trace)
    std::fprintf(stderr, "[hgrd many-call] %.0f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                     .count());
  return rc;
}

int hgrd_gpu_sweep_shard_json(hgrd_gpu_ctx *ctx, const char *source, const char *file_name,
                              const char *caps_json, int rank, int world, char **out) {
  if (!ctx || !out)
    return HGRD_GPU_EINVAL;
  GpuBackend be(ctx);
  std::string s;
  int rc = sweepShardJsonRun(be, source, file_name, caps_json, rank, world, s);
  *out = dup(s);
  return rc;
}

int hgrd_gpu_count_inputs(const char *source, const char *file_name) {
  ParseOutcome po = parseMiniCU(source ? source : "", file_name ? file_name : "");
  if (!po.program)
    return HGRD_GPU_EINVAL;
  return countInputs(*po.program);
}

void hgrd_gpu_free(char *p) { std::free(p); }

} // extern "C"

// Lowering only (no host interpretation): the bytecode, site table and
// per-kernel facts of one kernel, as JSON.  Used by callers that fix the
// launch parameters themselves (bench workloads, reference-side adapters).
namespace {
std::string escapeJson(const std::string &in) {
  std::string o;
  for (char ch : in) {
    if (ch == '"' || ch == '\\')
      o += '\\';
    if (ch == '\n') {
      o += "\\n";
      continue;
    }
    if (static_cast<unsigned char>(ch) < 0x20)
      continue;
    o += ch;
  }
  return o;
}
} // namespace

extern "C" int hgrd_gpu_stream_sites(const hgrd_gpu_launch *launch, int64_t *out) {
  if (!launch || (!out && launch->n_sites))
    return HGRD_GPU_EINVAL;
  const std::vector<int64_t> p = hgrdgpu::streamSites(*launch);
  for (size_t s = 0; s < p.size(); ++s)
    out[s] = p[s];
  return HGRD_GPU_OK;
}

extern "C" int hgrd_gpu_block_private(const hgrd_gpu_launch *launch, uint8_t *out) {
  if (!launch || (!out && launch->n_sites))
    return HGRD_GPU_EINVAL;
  const std::vector<uint8_t> p = blockPrivateSites(*launch);
  for (size_t s = 0; s < p.size(); ++s)
    out[s] = p[s];
  return HGRD_GPU_OK;
}

extern "C" int hgrd_gpu_jit_check(const char *source, const char *file_name, const char *kernel,
                                  const int64_t grid[3], const int64_t block[3],
                                  int64_t warp_size, char **out) {
  if (!out || !grid || !block)
    return HGRD_GPU_EINVAL;
  ParseOutcome po = parseMiniCU(source ? source : "", file_name ? file_name : "");
  const Function *k = po.program ? po.program->findKernel(kernel ? kernel : "") : nullptr;
  if (!k) {
    *out = dup(errorJson(po.program ? std::vector<std::string>{"unknown kernel"}
                                    : po.diagnostics));
    return HGRD_GPU_EINVAL;
  }
  LoweredKernel lk = lowerKernel(*k);
  std::vector<int64_t> regInit(lk.nRegs, 0);
  std::vector<int32_t> handles(k->params.size(), 0);
  hgrd_gpu_launch L{};
  L.code = lk.code.data();
  L.n_code = static_cast<uint32_t>(lk.code.size());
  L.n_regs = lk.nRegs;
  L.reg_init = regInit.data();
  L.sites = lk.sites.data();
  L.n_sites = static_cast<uint32_t>(lk.sites.size());
  L.n_locs = static_cast<uint32_t>(lk.locs.size());
  L.param_handle = handles.data();
  L.n_params = static_cast<uint32_t>(handles.size());
  for (int i = 0; i < 3; ++i) {
    L.grid[i] = grid[i];
    L.block[i] = block[i];
  }
  L.warp_size = warp_size;
  std::vector<uint8_t> rec(lk.sites.size(), 3);
  { // streamed value-needed loads compile to the staged accessor (loadS)
    const std::vector<int64_t> off = hgrdgpu::streamSites(L);
    for (uint32_t pc = 0; pc < L.n_code; ++pc)
      if (L.code[pc].op == HGRD_OP_LOAD && (L.code[pc].sub & 1) &&
          off[static_cast<size_t>(L.code[pc].imm)] != hgrdgpu::kNoStream)
        rec[static_cast<size_t>(L.code[pc].imm)] |= 4;
  }
  std::vector<hgrdgpu::jit::JitParam> params(handles.size(),
                                             hgrdgpu::jit::JitParam{int64_t(1) << 20, 0});
  L.step_budget = int64_t(1) << 40;
  std::string s = "{\"variants\":[";
  bool ok = true;
  for (int v = 0; v < hgrdgpu::jit::kVariants; ++v) {
    std::string err;
    const size_t bytes = hgrdgpu::jit::compileOnly(L, rec, params, static_cast<hgrdgpu::jit::Variant>(v), err);
    ok = ok && bytes > 0;
    s += (v ? "," : "") + std::string("{\"cubin_bytes\":") + std::to_string(bytes) +
         ",\"error\":\"" + escapeJson(err) + "\"}";
  }
  s += "]}";
  *out = dup(s);
  return ok ? HGRD_GPU_OK : HGRD_GPU_ENOTSUP;
}

extern "C" int hgrd_gpu_lower_json(const char *source, const char *file_name,
                                   const char *kernel, char **out) {
  if (!out)
    return HGRD_GPU_EINVAL;
  ParseOutcome po = parseMiniCU(source ? source : "", file_name ? file_name : "");
  if (!po.program) {
    *out = dup(errorJson(po.diagnostics));
    return HGRD_GPU_EINVAL;
  }
  const Function *k = po.program->findKernel(kernel ? kernel : "");
  if (!k) {
    *out = dup(errorJson({"unknown kernel"}));
    return HGRD_GPU_EINVAL;
  }
  LoweredKernel lk = lowerKernel(*k);
  std::string s = "{\"nRegs\":" + std::to_string(lk.nRegs) + ",\"hasLocks\":" +
                  (lk.hasLocks ? "true" : "false") + ",\"code\":[";
  for (size_t i = 0; i < lk.code.size(); ++i) {
    const auto &I = lk.code[i];
    s += (i ? ",[" : "[") + std::to_string(I.op) + "," + std::to_string(I.sub) + "," +
         std::to_string(I.a) + "," + std::to_string(I.b) + "," + std::to_string(I.c) + "," +
         std::to_string(I.imm) + "]";
  }
  s += "],\"sites\":[";
  for (size_t i = 0; i < lk.sites.size(); ++i) {
    const auto &S = lk.sites[i];
    s += (i ? ",{" : "{") + std::string("\"loc\":") + std::to_string(S.loc) +
         ",\"param\":" + std::to_string(S.param) + ",\"kind\":" + std::to_string(S.kind) +
         ",\"atomicOp\":" + std::to_string(S.atomic_op) + ",\"scope\":" +
         std::to_string(S.scope) + ",\"array\":\"" + lk.siteArray[i] + "\",\"valueNeeded\":" +
         (lk.siteValueNeeded[i] ? "true" : "false") + ",\"line\":" +
         std::to_string(lk.siteLoc[i].line) + ",\"column\":" + std::to_string(lk.siteLoc[i].col) +
         "}";
  }
  s += "],\"locs\":[";
  for (size_t i = 0; i < lk.locs.size(); ++i)
    s += (i ? ",[" : "[") + std::to_string(lk.locs[i].line) + "," +
         std::to_string(lk.locs[i].col) + "]";
  s += "],\"stmtLocs\":[";
  for (size_t i = 0; i < lk.stmtLocs.size(); ++i)
    s += (i ? ",[" : "[") + std::to_string(lk.stmtLocs[i].line) + "," +
         std::to_string(lk.stmtLocs[i].col) + "]";
  s += "],\"params\":[";
  for (size_t i = 0; i < k->params.size(); ++i)
    s += (i ? ",{" : "{") + std::string("\"name\":\"") + k->params[i].name +
         "\",\"array\":" + (isArray(k->params[i].type) ? "true" : "false") +
         ",\"reg\":" + std::to_string(lk.paramReg[i]) + "}";
  s += "]}";
  *out = dup(s);
  return 0;
}

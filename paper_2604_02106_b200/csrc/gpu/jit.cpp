// Per-kernel specialisation of the race-check kernels with NVRTC.
//
// The lowered bytecode of one MiniCU kernel (plus its launch constants —
// scalar parameters are folded in) is translated to a straight-line CUDA C++
// thread body (registers -> locals, jumps -> gotos) and compiled for sm_100a
// together with the kernel templates of csrc/gpu (jit_kernels.cuh), replacing
// the interpreter loop in k_expand_par and k_fused.  Modules are cached per
// generated source inside the context; compilation happens once per
// (kernel, launch constants).
#include "jit.hpp"

#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <chrono>
#include <cstdlib>
#include <sstream>
#include <vector>

namespace hgrdgpu {
namespace jit {

namespace {

std::string lit(int64_t v) {
  return "((int64_t)" + std::to_string(static_cast<unsigned long long>(v)) + "ULL)";
}

std::string dirOf(const std::string &p) {
  const size_t s = p.find_last_of('/');
  return s == std::string::npos ? "." : p.substr(0, s);
}

const char *kNames[3] = {"hgrdgpu::dev::k_expand_par<hgrdgpu::dev::JitBody>",
                         "hgrdgpu::dev::k_fused<4, hgrdgpu::dev::JitBody>",
                         "hgrdgpu::dev::k_fused<16, hgrdgpu::dev::JitBody>"};

} // namespace

std::string generate(const hgrd_gpu_launch &L) {
  std::vector<char> target(L.n_code, 0);
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (I.op == HGRD_OP_JZ || I.op == HGRD_OP_JMP)
      target[static_cast<size_t>(I.imm)] = 1;
  }
  std::ostringstream o;
  o << "#include \"jit_kernels.cuh\"\n"
       "namespace hgrdgpu {\nnamespace dev {\n"
       "struct JitBody {\n"
       "  template <class Sink>\n"
       "  __device__ static __forceinline__ void run(const LaunchDev &, const hgrd_gpu_insn *,\n"
       "                                             const Builtins &bi, Sink &s, int64_t *) {\n";
  for (uint32_t i = 0; i < L.n_regs; ++i)
    o << "    int64_t r" << i << " = " << lit(L.reg_init ? L.reg_init[i] : 0) << ";\n";
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if (target[pc])
      o << "  L" << pc << ":;\n";
    o << "    ";
    switch (I.op) {
    case HGRD_OP_END:
      o << "return;";
      break;
    case HGRD_OP_STEP:
      o << "if (!s.step(" << I.imm << ")) return;";
      break;
    case HGRD_OP_CONST:
      o << "r" << I.a << " = " << lit(I.imm) << ";";
      break;
    case HGRD_OP_MOV:
      o << "r" << I.a << " = r" << I.b << ";";
      break;
    case HGRD_OP_BUILTIN:
      o << "r" << I.a << " = bi.v[" << int(I.sub) << "];";
      break;
    case HGRD_OP_BIN:
      o << "r" << I.a << " = applyBin(" << int(I.sub) << ", r" << I.b << ", r" << I.c << ");";
      break;
    case HGRD_OP_LOAD:
      o << "r" << I.a << " = s.load(" << I.imm << ", r" << I.b << ", "
        << ((I.sub & 1) ? "true" : "false") << ");";
      break;
    case HGRD_OP_STORE:
      o << "s.store(" << I.imm << ", r" << I.a << ", r" << I.b << ");";
      break;
    case HGRD_OP_ATOMIC:
      o << "s.atomic(" << I.imm << ", r" << I.a << ", r" << I.b << ", r" << I.c << ");";
      break;
    case HGRD_OP_SYNCTHREADS:
      o << "s.syncthreads();";
      break;
    case HGRD_OP_SYNCWARP:
      o << "s.syncwarp();";
      break;
    case HGRD_OP_FENCE:
      o << "s.fence(" << int(I.sub) << ");";
      break;
    case HGRD_OP_JZ:
      o << "if (r" << I.a << " == 0) goto L" << I.imm << ";";
      break;
    case HGRD_OP_JMP:
      o << "goto L" << I.imm << ";";
      break;
    default:
      o << "return;";
    }
    o << "\n";
  }
  o << "  }\n};\n}\n}\n";
  return o.str();
}

struct Cache {
  std::map<std::string, const void *> mods; // generated source + variant -> kernel
  std::vector<cudaLibrary_t> libs;
  std::string incGpu, incRoot, incCuda;
  double compileMs = 0;
  int compiles = 0;
};

Cache *create() {
  auto *c = new Cache();
  Dl_info info{};
  if (dladdr(reinterpret_cast<void *>(&generate), &info) && info.dli_fname) {
    const std::string pkg = dirOf(info.dli_fname);
    c->incGpu = pkg + "/csrc/gpu";
    c->incRoot = dirOf(pkg) + "/include";
  }
  const char *home = std::getenv("CUDA_HOME");
  c->incCuda = std::string(home ? home : "/usr/local/cuda") + "/include";
  return c;
}

void destroy(Cache *c) {
  if (!c)
    return;
  for (cudaLibrary_t l : c->libs)
    cudaLibraryUnload(l);
  delete c;
}

double compileMs(const Cache *c) { return c ? c->compileMs : 0; }
int compiles(const Cache *c) { return c ? c->compiles : 0; }

const void *get(Cache *c, const hgrd_gpu_launch &L, Variant v, std::string &err) {
  const std::string src = generate(L);
  const std::string key = std::to_string(static_cast<int>(v)) + "\n" + src;
  auto it = c->mods.find(key);
  if (it != c->mods.end())
    return it->second;
  const auto t0 = std::chrono::steady_clock::now();
  const std::string name = std::string("&") + kNames[v];
  auto fail = [&](const std::string &why) -> const void * {
    err = why;
    c->mods.emplace(key, nullptr);
    return nullptr;
  };
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hgrd_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail("nvrtcCreateProgram failed");
  nvrtcAddNameExpression(prog, name.c_str());
  const std::string i1 = "-I" + c->incGpu, i2 = "-I" + c->incRoot, i3 = "-I" + c->incCuda;
  const char *opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-w",
                        "-DHGRD_JIT=1", i1.c_str(), i2.c_str(), i3.c_str()};
  const nvrtcResult rc = nvrtcCompileProgram(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    return fail(std::string("NVRTC: ") + nvrtcGetErrorString(rc) + "\n" + log.substr(0, 4000));
  }
  size_t cubinSize = 0;
  nvrtcGetCUBINSize(prog, &cubinSize);
  std::vector<char> cubin(cubinSize);
  nvrtcGetCUBIN(prog, cubin.data());
  const char *ln = nullptr;
  nvrtcGetLoweredName(prog, name.c_str(), &ln);
  const std::string lowered = ln ? ln : "";
  nvrtcDestroyProgram(&prog);
  cudaLibrary_t lib;
  if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
      cudaSuccess)
    return fail(std::string("cudaLibraryLoadData: ") + cudaGetErrorString(cudaGetLastError()));
  c->libs.push_back(lib);
  cudaKernel_t k;
  if (cudaLibraryGetKernel(&k, lib, lowered.c_str()) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("cudaLibraryGetKernel failed for " + lowered);
  }
  c->compileMs +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ++c->compiles;
  const void *fn = reinterpret_cast<const void *>(k);
  c->mods.emplace(key, fn);
  return fn;
}

} // namespace jit
} // namespace hgrdgpu

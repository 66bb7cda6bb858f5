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
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <algorithm>
#include <climits>
#include <optional>
#include <unordered_map>
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

const char *kNames[kVariants] = {"hgrdgpu::dev::k_expand_par<hgrdgpu::dev::JitBody>",
                                 "hgrdgpu::dev::k_fused<256, 4, hgrdgpu::dev::JitBody>",
                                 "hgrdgpu::dev::k_fused<256, 16, hgrdgpu::dev::JitBody>",
                                 "hgrdgpu::dev::k_fused<256, 8, hgrdgpu::dev::JitBody>",
                                 "hgrdgpu::dev::k_expand_seq<hgrdgpu::dev::JitBody>",
                                 "hgrdgpu::dev::k_fused<256, 12, hgrdgpu::dev::JitBody>"};

// Thread identity (reference src/oracle.cpp:443-460) with the launch
// geometry as literals, so every division is by a constant.
void emitIdentity(std::ostringstream &o, const hgrd_gpu_launch &L) {
  const int64_t tpb = L.block[0] * L.block[1] * L.block[2];
  const int64_t nThreads = tpb * L.grid[0] * L.grid[1] * L.grid[2];
  const bool small = nThreads < (int64_t(1) << 32) - 1 && L.warp_size < (int64_t(1) << 32);
  o << "  __device__ static __forceinline__ void identity(const LaunchDev &, int64_t t, Builtins &b,\n"
       "      int64_t &block, int64_t &warp, int64_t &lane) {\n";
  for (int i = 0; i < 3; ++i) {
    o << "    b.v[" << 6 + i << "] = " << lit(L.block[i]) << ";\n";
    o << "    b.v[" << 9 + i << "] = " << lit(L.grid[i]) << ";\n";
  }
  if (small) {
    auto u = [](int64_t v) { return std::to_string(static_cast<unsigned long long>(v)) + "u"; };
    o << "    const uint32_t x = static_cast<uint32_t>(t);\n"
         "    const uint32_t bl = x / " << u(tpb) << ", tl = x - bl * " << u(tpb) << ";\n"
         "    b.v[0] = tl % " << u(L.block[0]) << ";\n"
         "    b.v[1] = (tl / " << u(L.block[0]) << ") % " << u(L.block[1]) << ";\n"
         "    b.v[2] = tl / " << u(L.block[0] * L.block[1]) << ";\n"
         "    b.v[3] = bl % " << u(L.grid[0]) << ";\n"
         "    b.v[4] = (bl / " << u(L.grid[0]) << ") % " << u(L.grid[1]) << ";\n"
         "    b.v[5] = bl / " << u(L.grid[0] * L.grid[1]) << ";\n"
         "    block = bl;\n"
         "    warp = tl / " << u(L.warp_size) << ";\n"
         "    lane = tl % " << u(L.warp_size) << ";\n";
  } else {
    o << "    block = t / " << lit(tpb) << ";\n"
         "    const int64_t tl = t - block * " << lit(tpb) << ";\n"
         "    b.v[0] = tl % " << lit(L.block[0]) << ";\n"
         "    b.v[1] = (tl / " << lit(L.block[0]) << ") % " << lit(L.block[1]) << ";\n"
         "    b.v[2] = tl / " << lit(L.block[0] * L.block[1]) << ";\n"
         "    b.v[3] = block % " << lit(L.grid[0]) << ";\n"
         "    b.v[4] = (block / " << lit(L.grid[0]) << ") % " << lit(L.grid[1]) << ";\n"
         "    b.v[5] = block / " << lit(L.grid[0] * L.grid[1]) << ";\n"
         "    warp = tl / " << lit(L.warp_size) << ";\n"
         "    lane = tl - warp * " << lit(L.warp_size) << ";\n";
  }
  o << "  }\n";
}

} // namespace

// Loop-free code (no backward jump; ctx.cu phaseBounds uses the same rule)
// executes every access and statement at most once per thread.
bool hasLoops(const hgrd_gpu_launch &L) {
  for (uint32_t pc = 0; pc < L.n_code; ++pc)
    if (L.code[pc].op == HGRD_OP_JMP && L.code[pc].imm <= static_cast<int64_t>(pc))
      return true;
  return false;
}

// Value ranges of the registers before every instruction of loop-free code
// (interval arithmetic in 128 bits over the launch's builtin ranges; loaded
// values are unknown unless the PARALLEL sink returns 0 for them).  An
// operation whose operands and result all fit in int32 computes the same
// value in 32-bit arithmetic, which the generated body then uses.
struct Range {
  bool known = false;
  __int128 lo = 0, hi = 0;
  bool fits32() const { return known && lo >= INT32_MIN && hi <= INT32_MAX; }
  bool operator==(const Range &o) const {
    return known == o.known && (!known || (lo == o.lo && hi == o.hi));
  }
};

std::vector<std::vector<Range>> valueRanges(const hgrd_gpu_launch &L) {
  using R = std::vector<Range>;
  const size_t nr = L.n_regs;
  std::vector<R> before(L.n_code); // empty: unreachable
  std::vector<std::optional<R>> pending(L.n_code + 1);
  auto k = [](__int128 v) { return Range{true, v, v}; };
  auto join = [](std::optional<R> &into, const R &s) {
    if (!into) {
      into = s;
      return;
    }
    for (size_t r = 0; r < s.size(); ++r) {
      Range &a = (*into)[r];
      const Range &b = s[r];
      if (!a.known || !b.known)
        a = Range{};
      else
        a = Range{true, std::min(a.lo, b.lo), std::max(a.hi, b.hi)};
    }
  };
  std::optional<R> cur = R(nr);
  for (size_t r = 0; r < nr; ++r)
    (*cur)[r] = k(L.reg_init ? L.reg_init[r] : 0);
  const __int128 lim = static_cast<__int128>(INT64_MAX);
  auto clip = [&](Range v) { // wrapping int64: only exact ranges are kept
    if (!v.known || v.lo < -lim - 1 || v.hi > lim)
      return Range{};
    return v;
  };
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    if (pending[pc]) {
      if (cur)
        join(pending[pc], *cur);
      cur = pending[pc];
      pending[pc].reset();
    }
    if (!cur)
      continue;
    before[pc] = *cur;
    const auto &I = L.code[pc];
    R &S = *cur;
    auto get = [&](uint16_t r) { return r < nr ? S[r] : Range{}; };
    auto put = [&](uint16_t r, Range v) {
      if (r < nr)
        S[r] = clip(v);
    };
    switch (I.op) {
    case HGRD_OP_CONST:
      put(I.a, k(I.imm));
      break;
    case HGRD_OP_MOV:
      put(I.a, get(I.b));
      break;
    case HGRD_OP_BUILTIN:
      if (I.sub < 3)
        put(I.a, Range{true, 0, L.block[I.sub] - 1});
      else if (I.sub < 6)
        put(I.a, Range{true, 0, L.grid[I.sub - 3] - 1});
      else if (I.sub < 9)
        put(I.a, k(L.block[I.sub - 6]));
      else if (I.sub < 12)
        put(I.a, k(L.grid[I.sub - 9]));
      else
        put(I.a, Range{});
      break;
    case HGRD_OP_BIN: {
      const Range l = get(I.b), r = get(I.c);
      Range v;
      if (I.sub >= HGRD_LT) {
        v = Range{true, 0, 1}; // comparisons and logic yield 0 / 1
      } else if (l.known && r.known) {
        if (I.sub == HGRD_ADD) {
          v = Range{true, l.lo + r.lo, l.hi + r.hi};
        } else if (I.sub == HGRD_SUB) {
          v = Range{true, l.lo - r.hi, l.hi - r.lo};
        } else if (I.sub == HGRD_MUL) {
          const __int128 c[4] = {l.lo * r.lo, l.lo * r.hi, l.hi * r.lo, l.hi * r.hi};
          v = Range{true, *std::min_element(c, c + 4), *std::max_element(c, c + 4)};
        } else if (r.lo == r.hi && r.lo != 0 && r.lo != -1) { // constant divisor
          const __int128 d = r.lo;
          if (I.sub == HGRD_DIV) {
            const __int128 a = l.lo / d, b = l.hi / d;
            v = Range{true, std::min(a, b), std::max(a, b)};
          } else { // MOD: |result| < |d|, sign of the dividend
            const __int128 m = (d < 0 ? -d : d) - 1;
            v = Range{true, l.lo >= 0 ? 0 : -m, l.hi <= 0 ? 0 : m};
          }
        }
      }
      put(I.a, v);
      break;
    }
    case HGRD_OP_LOAD:
      put(I.a, (I.sub & 1) ? Range{} : k(0)); // PARALLEL: unneeded values read as 0
      break;
    case HGRD_OP_JZ:
      join(pending[static_cast<size_t>(I.imm)], S);
      break;
    case HGRD_OP_JMP:
      join(pending[static_cast<size_t>(I.imm)], S);
      cur.reset();
      break;
    case HGRD_OP_END:
      cur.reset();
      break;
    default:
      break;
    }
  }
  return before;
}

// A loop-free thread executes each STEP at most once: no per-statement
// budget checks when the launch's budget covers them all (the host still
// compares the launch's total steps with the budget).
// The canonical-order kernel is itself the exact (aborting) path, so there
// the whole launch's steps must fit the budget.
bool stepFree(const hgrd_gpu_launch &L, bool seq) {
  if (hasLoops(L))
    return false;
  int64_t n = 0;
  for (uint32_t pc = 0; pc < L.n_code; ++pc)
    n += L.code[pc].op == HGRD_OP_STEP;
  if (!seq)
    return n <= L.step_budget;
  const __int128 threads = static_cast<__int128>(L.grid[0]) * L.grid[1] * L.grid[2] *
                           L.block[0] * L.block[1] * L.block[2];
  return threads * n <= L.step_budget;
}

std::string generate(const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                     const std::vector<JitParam> &params, bool seq, bool lowOccupancy) {
  std::vector<char> target(L.n_code + 1, 0);
  uint32_t nRec = 0;
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if ((I.op == HGRD_OP_JZ || I.op == HGRD_OP_JMP) && I.imm >= 0 &&
        I.imm <= static_cast<int64_t>(L.n_code))
      target[static_cast<size_t>(I.imm)] = 1;
    if ((I.op == HGRD_OP_LOAD || I.op == HGRD_OP_STORE || I.op == HGRD_OP_ATOMIC) &&
        static_cast<size_t>(I.imm) < rec.size() && (rec[static_cast<size_t>(I.imm)] & 1))
      ++nRec;
  }
  const bool loops = hasLoops(L);
  const bool noStepChecks = stepFree(L, seq);
  // 32-bit arithmetic where value ranges allow (loop-free kernels)
  std::vector<std::vector<Range>> ranges;
  if (!loops)
    ranges = valueRanges(L);
  auto rangeAt = [&](uint32_t pc, uint16_t r) -> Range {
    return pc < ranges.size() && r < ranges[pc].size() ? ranges[pc][r] : Range{};
  };
  // the access's index register (register prefix R) as a 32-bit value when
  // it and the buffer size fit (one unsigned compare bounds-checks it)
  auto idxArg = [&](uint32_t pc, uint16_t r, int64_t site, const char *R) -> std::string {
    const size_t i = static_cast<size_t>(site);
    const int32_t p = i < L.n_sites ? L.sites[i].param : -1;
    const int64_t size = (p >= 0 && static_cast<size_t>(p) < params.size())
                             ? params[static_cast<size_t>(p)].size
                             : 0;
    if (rangeAt(pc, r).fits32() && size <= INT32_MAX)
      return "static_cast<int32_t>(" + std::string(R) + std::to_string(r) + ")";
    return R + std::to_string(r);
  };
  // access -> literal arguments of the sink's C accessors: site, param,
  // record, own (rec[s]: bit 0 record, bit 1 ownership exchange), ... , size,
  // element base
  auto site = [&](int64_t s) {
    const size_t i = static_cast<size_t>(s);
    const uint8_t f = i < rec.size() ? rec[i] : 3;
    return std::to_string(s) + ", " + std::to_string(i < L.n_sites ? L.sites[i].param : 0) +
           ", " + ((f & 1) ? "true" : "false") + ", " + ((f & 2) ? "true" : "false");
  };
  auto buf = [&](int64_t s) {
    const size_t i = static_cast<size_t>(s);
    const int32_t p = i < L.n_sites ? L.sites[i].param : -1;
    const JitParam jp = (p >= 0 && static_cast<size_t>(p) < params.size())
                            ? params[static_cast<size_t>(p)]
                            : JitParam{0, 0};
    return ", " + lit(jp.size) + ", " + std::to_string(jp.base) + "ULL";
  };
  auto sizeLit = [&](int64_t s) {
    const size_t i = static_cast<size_t>(s);
    const int32_t p = i < L.n_sites ? L.sites[i].param : -1;
    return lit((p >= 0 && static_cast<size_t>(p) < params.size())
                   ? params[static_cast<size_t>(p)].size
                   : 0);
  };
  auto streamed = [&](const hgrd_gpu_insn &I) {
    return (I.sub & 1) && static_cast<size_t>(I.imm) < rec.size() &&
           (rec[static_cast<size_t>(I.imm)] & 4);
  };
  // One instruction for registers R, builtins B and sink S.
  auto insn = [&](std::ostringstream &o, uint32_t pc, const char *R, const char *B,
                  const char *S) {
    const auto &I = L.code[pc];
    const std::string r = R, sk = S;
    auto reg = [&](uint16_t x) { return r + std::to_string(x); };
    switch (I.op) {
    case HGRD_OP_END:
      o << "return;";
      break;
    case HGRD_OP_STEP:
      if (noStepChecks)
        o << sk << ".stepNC();";
      else
        o << "if (!" << sk << ".step(" << I.imm << ")) return;";
      break;
    case HGRD_OP_CONST:
      o << reg(I.a) << " = " << lit(I.imm) << ";";
      break;
    case HGRD_OP_MOV:
      o << reg(I.a) << " = " << reg(I.b) << ";";
      break;
    case HGRD_OP_BUILTIN:
      o << reg(I.a) << " = " << B << ".v[" << int(I.sub) << "];";
      break;
    case HGRD_OP_BIN: {
      const Range rl = rangeAt(pc, I.b), rr = rangeAt(pc, I.c);
      const Range res = pc + 1 < ranges.size() ? rangeAt(pc + 1, I.a) : Range{};
      static const char *ops[] = {"+", "-", "*", "/", "%", "<", "<=", ">", ">=", "==", "!="};
      const bool narrow = rl.fits32() && rr.fits32() && I.sub <= HGRD_NE &&
                          (I.sub >= HGRD_LT || res.fits32()) &&
                          ((I.sub != HGRD_DIV && I.sub != HGRD_MOD) ||
                           (rr.lo == rr.hi && rr.lo != 0 && rr.lo != -1));
      if (narrow)
        o << reg(I.a) << " = static_cast<int64_t>(static_cast<int32_t>(" << reg(I.b) << ") "
          << ops[I.sub] << " static_cast<int32_t>(" << reg(I.c) << "));";
      else
        o << reg(I.a) << " = applyBin(" << int(I.sub) << ", " << reg(I.b) << ", " << reg(I.c)
          << ");";
      break;
    }
    case HGRD_OP_LOAD:
      if (streamed(I)) // streamed (staged) value-needed load
        o << reg(I.a) << " = " << sk << ".loadS(" << site(I.imm) << ", "
          << idxArg(pc, I.b, I.imm, R) << buf(I.imm) << ");";
      else
        o << reg(I.a) << " = " << sk << ".loadC(" << site(I.imm) << ", "
          << idxArg(pc, I.b, I.imm, R) << ", " << ((I.sub & 1) ? "true" : "false")
          << buf(I.imm) << ");";
      break;
    case HGRD_OP_STORE:
      o << sk << ".storeC(" << site(I.imm) << ", " << idxArg(pc, I.a, I.imm, R) << ", "
        << reg(I.b) << buf(I.imm) << ");";
      break;
    case HGRD_OP_ATOMIC:
      o << sk << ".atomicC(" << site(I.imm) << ", " << idxArg(pc, I.a, I.imm, R) << ", "
        << reg(I.b) << ", " << reg(I.c) << buf(I.imm) << ");";
      break;
    case HGRD_OP_SYNCTHREADS:
      o << sk << ".syncthreads();";
      break;
    case HGRD_OP_SYNCWARP:
      o << sk << ".syncwarp();";
      break;
    case HGRD_OP_FENCE:
      o << sk << ".fence(" << int(I.sub) << ");";
      break;
    case HGRD_OP_JZ:
      o << "if (" << reg(I.a) << " == 0) goto L" << I.imm << ";";
      break;
    case HGRD_OP_JMP:
      o << "goto L" << I.imm << ";";
      break;
    default:
      o << "return;";
    }
  };
  // Two MiniCU threads per call (k_fused): branch-free bodies with no step
  // checks interleave the threads instruction by instruction, and a
  // value-needed global load fetches both threads' values before either
  // records its access, so the two loads are in flight together (memory-level
  // parallelism the per-thread interpretation order would serialise).  Only
  // bodies with such a load, or for the variants of at most two CTAs per SM
  // (few resident warps: the second thread's independent record pushes fill
  // the issue slots).  Otherwise the pair only adds code (A/B,
  // profiles/r02/ab_pair_bits.txt: histogram 2.42 -> 2.52 ms; the x12
  // transpose 1.67 -> 1.60 ms).
  bool pairable = !loops && noStepChecks && !std::getenv("HGRD_JIT_NO_PAIR"); // (A/B knob)
  bool globalValueLoad = false;
  for (uint32_t pc = 0; pc < L.n_code && pairable; ++pc) {
    const auto &I = L.code[pc];
    pairable = I.op != HGRD_OP_JZ && I.op != HGRD_OP_JMP;
    globalValueLoad |= I.op == HGRD_OP_LOAD && (I.sub & 1) && !streamed(I);
  }
  pairable = pairable && (globalValueLoad || lowOccupancy);

  std::ostringstream o;
  o << "#include \"jit_kernels.cuh\"\n"
       "namespace hgrdgpu {\nnamespace dev {\n"
       "struct JitBody {\n";
  o << "  static constexpr int kFixedR = " << (loops ? 0 : nRec) << ";\n";
  o << "  static constexpr bool kPair = " << (pairable ? "true" : "false") << ";\n";
  emitIdentity(o, L);
  o << "  template <class Sink>\n"
       "  __device__ static __forceinline__ void run(const LaunchDev &, const hgrd_gpu_insn *,\n"
       "                                             const Builtins &bi, Sink &s, int64_t *) {\n";
  for (uint32_t i = 0; i < L.n_regs; ++i)
    o << "    int64_t r" << i << " = " << lit(L.reg_init ? L.reg_init[i] : 0) << ";\n";
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    if (target[pc])
      o << "  L" << pc << ":;\n";
    o << "    ";
    insn(o, pc, "r", "bi", "s");
    o << "\n";
  }
  o << "  }\n";
  o << "  template <class Sink>\n"
       "  __device__ static __forceinline__ void run2(const Builtins &ba, Sink &sa,\n"
       "                                              const Builtins &bb, Sink &sb) {\n";
  if (pairable) {
    for (uint32_t i = 0; i < L.n_regs; ++i) {
      o << "    int64_t a" << i << " = " << lit(L.reg_init ? L.reg_init[i] : 0) << ";\n";
      o << "    int64_t b" << i << " = " << lit(L.reg_init ? L.reg_init[i] : 0) << ";\n";
    }
    for (uint32_t pc = 0; pc < L.n_code; ++pc) {
      const auto &I = L.code[pc];
      if (I.op == HGRD_OP_END) {
        o << "    return;\n";
        break;
      }
      if (I.op == HGRD_OP_LOAD && (I.sub & 1) && !streamed(I)) {
        const int32_t p = static_cast<size_t>(I.imm) < L.n_sites ? L.sites[I.imm].param : 0;
        const std::string sz = sizeLit(I.imm);
        o << "    { const int64_t va = sa.fetchC(" << p << ", " << idxArg(pc, I.b, I.imm, "a")
          << ", " << sz << "), vb = sb.fetchC(" << p << ", " << idxArg(pc, I.b, I.imm, "b")
          << ", " << sz << ");\n";
        o << "      sa.loadC(" << site(I.imm) << ", " << idxArg(pc, I.b, I.imm, "a") << ", false"
          << buf(I.imm) << "); a" << I.a << " = va;\n";
        o << "      sb.loadC(" << site(I.imm) << ", " << idxArg(pc, I.b, I.imm, "b") << ", false"
          << buf(I.imm) << "); b" << I.a << " = vb; }\n";
        continue;
      }
      o << "    ";
      insn(o, pc, "a", "ba", "sa");
      o << "\n    ";
      insn(o, pc, "b", "bb", "sb");
      o << "\n";
    }
  }
  o << "  }\n";
  o << "};\n}\n}\n";
  return o.str();
}

struct Cache {
  std::unordered_map<std::string, const void *> mods; // launch inputs + variant -> kernel
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

namespace {

// NVRTC: generated source -> sm_100a cubin and the lowered kernel name.
bool compile(const Cache *c, const std::string &src, Variant v, std::vector<char> &cubin,
             std::string &lowered, std::string &err) {
  const std::string name = std::string("&") + kNames[v];
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hgrd_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return false;
  }
  nvrtcAddNameExpression(prog, name.c_str());
  const std::string i1 = "-I" + c->incGpu, i2 = "-I" + c->incRoot, i3 = "-I" + c->incCuda;
  std::vector<const char *> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo",
                                    "-w", "-DHGRD_JIT=1", i1.c_str(), i2.c_str(), i3.c_str()};
  // development: extra NVRTC options (e.g. -DHGRD_FUSED_MINB=4), space separated
  std::vector<std::string> extra;
  if (const char *x = std::getenv("HGRD_JIT_OPTS")) {
    std::istringstream is(x);
    for (std::string w; is >> w;)
      extra.push_back(w);
  }
  for (const auto &w : extra)
    opts.push_back(w.c_str());
  const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    err = std::string("NVRTC: ") + nvrtcGetErrorString(rc) + "\n" + log.substr(0, 4000);
    return false;
  }
  size_t cubinSize = 0;
  nvrtcGetCUBINSize(prog, &cubinSize);
  cubin.resize(cubinSize);
  nvrtcGetCUBIN(prog, cubin.data());
  const char *ln = nullptr;
  nvrtcGetLoweredName(prog, name.c_str(), &ln);
  lowered = ln ? ln : "";
  nvrtcDestroyProgram(&prog);
  return true;
}

} // namespace

const void *get(Cache *c, const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                const std::vector<JitParam> &params, Variant v, std::string &err) {
  // cache key: the raw launch inputs of generate() (cheaper than the source)
  std::string key;
  auto put = [&key](const void *p, size_t n) { key.append(static_cast<const char *>(p), n); };
  const int vi = static_cast<int>(v);
  put(&vi, sizeof vi);
  put(L.grid, sizeof L.grid);
  put(L.block, sizeof L.block);
  put(&L.warp_size, sizeof L.warp_size);
  put(&L.n_regs, sizeof L.n_regs);
  put(L.code, sizeof(hgrd_gpu_insn) * L.n_code);
  if (L.reg_init)
    put(L.reg_init, 8 * L.n_regs);
  put(L.sites, sizeof(hgrd_gpu_site) * L.n_sites);
  put(rec.data(), rec.size());
  put(params.data(), sizeof(JitParam) * params.size());
  const bool noStepChecks = stepFree(L, v == kExpandSeq);
  put(&noStepChecks, sizeof noStepChecks);
  auto it = c->mods.find(key);
  if (it != c->mods.end())
    return it->second;
  const std::string src =
      generate(L, rec, params, v == kExpandSeq, v == kFused12 || v == kFusedWide);
  const auto t0 = std::chrono::steady_clock::now();
  auto fail = [&](const std::string &why) -> const void * {
    err = why;
    c->mods.emplace(key, nullptr);
    return nullptr;
  };
  std::vector<char> cubin;
  std::string lowered, cerr;
  if (!compile(c, src, v, cubin, lowered, cerr))
    return fail(cerr);
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

size_t compileOnly(const hgrd_gpu_launch &L, const std::vector<uint8_t> &rec,
                   const std::vector<JitParam> &params, Variant v, std::string &err) {
  Cache *c = create();
  std::vector<char> cubin;
  std::string lowered;
  const std::string src =
      generate(L, rec, params, v == kExpandSeq, v == kFused12 || v == kFusedWide);
  if (const char *dump = std::getenv("HGRD_JIT_DUMP")) { // development: keep the source
    if (FILE *f = std::fopen(dump, "w")) {
      std::fputs(src.c_str(), f);
      std::fclose(f);
    }
  }
  const bool ok = compile(c, src, v, cubin, lowered, err);
  destroy(c);
  return ok ? cubin.size() : 0;
}

} // namespace jit
} // namespace hgrdgpu

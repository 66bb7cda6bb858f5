// Block-private partition proof for the fused path's INTER-BLOCK filter.
//
// The fused kernel finds INTRA-BLOCK / INTRA-WARP pairs on chip and, for
// INTER-BLOCK pairs (reference src/oracle.cpp:754-769: an element accessed
// from two blocks), does one ownership exchange per (element, block).  When
// the index of every access to a buffer is an affine function of the thread
// builtins whose per-block element ranges are pairwise disjoint, no element
// of that buffer can be reached from two blocks and the exchange is skipped.
//
// Abstract interpretation of the lowered bytecode (acyclic code only):
// every register holds either an affine form k + sum_d c_d * builtin_d over
// threadIdx.{x,y,z} and blockIdx.{x,y,z} (blockDim / gridDim / scalar
// parameters are launch constants), or "unknown".  Forms whose value range
// over the launch might leave int64 become unknown (MiniCU arithmetic wraps,
// the form would not).
#include "affine.hpp"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <optional>

namespace hgrdgpu {

namespace {

using i128 = __int128;

constexpr i128 kI64Max = static_cast<i128>(INT64_MAX);
constexpr i128 kI64Min = static_cast<i128>(INT64_MIN);

struct Form {
  bool known = false;
  i128 k = 0;
  std::array<i128, 6> c{}; // tid x,y,z then bid x,y,z
  bool operator==(const Form &o) const {
    return known == o.known && (!known || (k == o.k && c == o.c));
  }
};

struct Domain {
  std::array<i128, 6> extent; // values of builtin d range over [0, extent-1]
};

// Value range of a form over the launch domain.
void range(const Form &f, const Domain &D, i128 &lo, i128 &hi) {
  lo = hi = f.k;
  for (int d = 0; d < 6; ++d) {
    const i128 span = f.c[d] * (D.extent[d] - 1);
    if (span > 0)
      hi += span;
    else
      lo += span;
  }
}

Form checked(Form f, const Domain &D) {
  if (!f.known)
    return f;
  for (int d = 0; d < 6; ++d)
    if (f.c[d] > kI64Max || f.c[d] < kI64Min)
      return Form{};
  if (f.k > kI64Max || f.k < kI64Min)
    return Form{};
  i128 lo, hi;
  range(f, D, lo, hi);
  if (lo < kI64Min || hi > kI64Max)
    return Form{};
  return f;
}

Form constant(i128 v) {
  Form f;
  f.known = true;
  f.k = v;
  return f;
}

using State = std::vector<Form>;

void merge(std::optional<State> &into, const State &s) {
  if (!into) {
    into = s;
    return;
  }
  for (size_t r = 0; r < s.size(); ++r)
    if (!((*into)[r] == s[r]))
      (*into)[r] = Form{};
}

// Per-site index forms of a loop-free launch (abstract interpretation of the
// bytecode): false when the code has loops.
struct SiteForms {
  Domain D;
  std::vector<std::optional<Form>> idx;
  std::vector<uint8_t> seen, unknown;
};

bool siteForms(const hgrd_gpu_launch &L, SiteForms &out) {
  if (!L.code || L.n_code == 0)
    return false;
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    const auto &I = L.code[pc];
    if ((I.op == HGRD_OP_JMP || I.op == HGRD_OP_JZ) &&
        (I.imm <= static_cast<int64_t>(pc) || I.imm > static_cast<int64_t>(L.n_code)))
      return false; // loops (or malformed jumps): no forms
  }
  Domain D;
  for (int d = 0; d < 3; ++d) {
    D.extent[d] = L.block[d];
    D.extent[3 + d] = L.grid[d];
  }
  const size_t nr = L.n_regs;
  std::vector<std::optional<State>> pending(L.n_code + 1);
  std::optional<State> cur = State(nr);
  for (size_t r = 0; r < nr; ++r)
    (*cur)[r] = constant(L.reg_init ? L.reg_init[r] : 0);
  std::vector<std::optional<Form>> siteIdx(L.n_sites);
  std::vector<uint8_t> siteSeen(L.n_sites, 0), siteUnknown(L.n_sites, 0);
  auto reg = [&](uint16_t r) -> Form { return r < nr ? (*cur)[r] : Form{}; };
  auto set = [&](uint16_t r, const Form &f) {
    if (r < nr)
      (*cur)[r] = checked(f, D);
  };
  auto noteSite = [&](int64_t s, const Form &idx) {
    if (s < 0 || static_cast<uint64_t>(s) >= L.n_sites)
      return;
    siteSeen[static_cast<size_t>(s)] = 1;
    if (!idx.known)
      siteUnknown[static_cast<size_t>(s)] = 1;
    else if (!siteIdx[static_cast<size_t>(s)])
      siteIdx[static_cast<size_t>(s)] = idx;
    else if (!(*siteIdx[static_cast<size_t>(s)] == idx))
      siteUnknown[static_cast<size_t>(s)] = 1;
  };
  for (uint32_t pc = 0; pc < L.n_code; ++pc) {
    if (pending[pc]) {
      if (cur)
        merge(pending[pc], *cur);
      cur = pending[pc];
      pending[pc].reset();
    }
    if (!cur)
      continue; // unreachable
    const auto &I = L.code[pc];
    switch (I.op) {
    case HGRD_OP_CONST:
      set(I.a, constant(I.imm));
      break;
    case HGRD_OP_MOV:
      set(I.a, reg(I.b));
      break;
    case HGRD_OP_BUILTIN: {
      Form f;
      if (I.sub < 6) {
        f.known = true;
        f.c[I.sub] = 1;
      } else if (I.sub < 9) {
        f = constant(L.block[I.sub - 6]);
      } else if (I.sub < 12) {
        f = constant(L.grid[I.sub - 9]);
      }
      set(I.a, f);
      break;
    }
    case HGRD_OP_BIN: {
      const Form l = reg(I.b), r = reg(I.c);
      Form f;
      if (l.known && r.known) {
        if (I.sub == HGRD_ADD || I.sub == HGRD_SUB) {
          const i128 sg = I.sub == HGRD_ADD ? 1 : -1;
          f.known = true;
          f.k = l.k + sg * r.k;
          for (int d = 0; d < 6; ++d)
            f.c[d] = l.c[d] + sg * r.c[d];
        } else if (I.sub == HGRD_MUL) {
          const bool lc = std::all_of(l.c.begin(), l.c.end(), [](i128 x) { return x == 0; });
          const bool rc = std::all_of(r.c.begin(), r.c.end(), [](i128 x) { return x == 0; });
          if (lc || rc) {
            const Form &v = lc ? r : l;
            const i128 m = lc ? l.k : r.k;
            if (m > kI64Max || m < kI64Min)
              break;
            f.known = true;
            f.k = v.k * m;
            for (int d = 0; d < 6; ++d)
              f.c[d] = v.c[d] * m;
          }
        }
      }
      set(I.a, f);
      break;
    }
    case HGRD_OP_LOAD:
      noteSite(I.imm, reg(I.b));
      set(I.a, Form{});
      break;
    case HGRD_OP_STORE:
    case HGRD_OP_ATOMIC:
      noteSite(I.imm, reg(I.a));
      break;
    case HGRD_OP_JZ:
      merge(pending[static_cast<size_t>(I.imm)], *cur);
      break;
    case HGRD_OP_JMP:
      merge(pending[static_cast<size_t>(I.imm)], *cur);
      cur.reset();
      break;
    case HGRD_OP_END:
      cur.reset();
      break;
    default:
      break;
    }
  }
  out.D = D;
  out.idx = std::move(siteIdx);
  out.seen = std::move(siteSeen);
  out.unknown = std::move(siteUnknown);
  return true;
}

} // namespace

std::vector<int64_t> streamSites(const hgrd_gpu_launch &L) {
  std::vector<int64_t> off(L.n_sites, kNoStream);
  SiteForms F;
  if (!siteForms(L, F))
    return off;
  // coefficients of the dense thread id (reference :443-460): tid x, y, z,
  // then bid x, y, z; a builtin with extent 1 is always 0 (any coefficient)
  const i128 bx = L.block[0], by = L.block[1], tpb = bx * by * L.block[2];
  const i128 gx = L.grid[0], gy = L.grid[1];
  const std::array<i128, 6> dense{1, bx, bx * by, tpb, gx * tpb, gx * gy * tpb};
  for (uint32_t s = 0; s < L.n_sites; ++s) {
    if (L.sites[s].kind != HGRD_SITE_LOAD || !F.seen[s] || F.unknown[s] || !F.idx[s])
      continue;
    const Form &f = *F.idx[s];
    bool ok = f.k >= kI64Min && f.k <= kI64Max;
    for (int d = 0; d < 6 && ok; ++d)
      ok = F.D.extent[d] <= 1 || f.c[d] == dense[d];
    if (ok)
      off[s] = static_cast<int64_t>(f.k);
  }
  return off;
}

std::vector<uint8_t> blockPrivateSites(const hgrd_gpu_launch &L) {
  std::vector<uint8_t> priv(L.n_sites, 0);
  SiteForms F;
  if (!siteForms(L, F))
    return priv;
  const Domain &D = F.D;
  const std::vector<std::optional<Form>> &siteIdx = F.idx;
  const std::vector<uint8_t> &siteSeen = F.seen, &siteUnknown = F.unknown;

  // per buffer handle: the reached sites' forms must share the block
  // coefficients, and blocks' element ranges must be separated (mixed radix)
  std::vector<int32_t> handles;
  for (uint32_t s = 0; s < L.n_sites; ++s) {
    const int32_t p = L.sites[s].param;
    if (p >= 0 && static_cast<uint32_t>(p) < L.n_params && L.param_handle[p] >= 0)
      handles.push_back(L.param_handle[p]);
  }
  std::sort(handles.begin(), handles.end());
  handles.erase(std::unique(handles.begin(), handles.end()), handles.end());
  for (int32_t h : handles) {
    bool ok = true, any = false, same = true, known = true;
    std::optional<Form> first;
    std::array<i128, 3> a{};
    i128 lo = 0, hi = 0;
    for (uint32_t s = 0; s < L.n_sites; ++s) { // test B input: one shared form?
      const int32_t p = L.sites[s].param;
      if (p < 0 || static_cast<uint32_t>(p) >= L.n_params || L.param_handle[p] != h ||
          !siteSeen[s])
        continue;
      if (siteUnknown[s] || !siteIdx[s]) {
        known = false;
        break;
      }
      if (!first)
        first = *siteIdx[s];
      else if (!(*first == *siteIdx[s]))
        same = false;
    }
    for (uint32_t s = 0; s < L.n_sites && ok; ++s) {
      const int32_t p = L.sites[s].param;
      if (p < 0 || static_cast<uint32_t>(p) >= L.n_params || L.param_handle[p] != h)
        continue;
      if (!siteSeen[s])
        continue; // never executed: no records
      if (siteUnknown[s] || !siteIdx[s]) {
        ok = false;
        break;
      }
      const Form &f = *siteIdx[s];
      Form t = f; // thread part + constant
      for (int d = 0; d < 3; ++d)
        t.c[3 + d] = 0;
      i128 tlo, thi;
      range(t, D, tlo, thi);
      std::array<i128, 3> b{};
      for (int d = 0; d < 3; ++d)
        b[d] = D.extent[3 + d] > 1 ? f.c[3 + d] : 0;
      if (!any) {
        a = b;
        lo = tlo;
        hi = thi;
        any = true;
      } else {
        if (a != b)
          ok = false;
        lo = std::min(lo, tlo);
        hi = std::max(hi, thi);
      }
    }
    if (!any)
      continue;
    const bool formsOk = ok; // test A needs known forms sharing block coefficients
    const i128 W = hi - lo;
    std::array<std::pair<i128, i128>, 3> dims{}; // (|a_d|, grid extent)
    int nd = 0;
    for (int d = 0; d < 3; ++d)
      if (D.extent[3 + d] > 1)
        dims[nd++] = {a[d] < 0 ? -a[d] : a[d], D.extent[3 + d]};
    std::sort(dims.begin(), dims.begin() + nd);
    i128 reach = W; // largest in-block distance so far
    for (int i = 0; i < nd && formsOk && ok; ++i) {
      if (dims[i].first <= reach)
        ok = false;
      reach += dims[i].first * (dims[i].second - 1);
    }
    // test B: every access of the buffer uses one form whose map from
    // (threadIdx dims it depends on, blockIdx dims) to the index is
    // injective (mixed radix: each coefficient exceeds the reach of the
    // smaller ones), so equal indices imply equal blocks
    if (!ok && known && same && first) {
      std::array<std::pair<i128, i128>, 6> v{};
      int nv = 0;
      bool inj = true;
      for (int d = 0; d < 6; ++d) {
        if (D.extent[d] <= 1)
          continue;
        const i128 c = first->c[d] < 0 ? -first->c[d] : first->c[d];
        if (c == 0) {
          if (d >= 3)
            inj = false; // two blocks on one range
          continue;      // threads of one block may share elements
        }
        v[nv++] = {c, D.extent[d]};
      }
      std::sort(v.begin(), v.begin() + nv);
      i128 reach = 0;
      for (int i = 0; i < nv && inj; ++i) {
        if (v[i].first <= reach)
          inj = false;
        reach += v[i].first * (v[i].second - 1);
      }
      if (inj) {
        for (uint32_t s = 0; s < L.n_sites; ++s) {
          const int32_t p = L.sites[s].param;
          if (p >= 0 && static_cast<uint32_t>(p) < L.n_params && L.param_handle[p] == h)
            priv[s] = 1;
        }
        continue;
      }
    }
    if (!ok)
      continue;
    for (uint32_t s = 0; s < L.n_sites; ++s) {
      const int32_t p = L.sites[s].param;
      if (p >= 0 && static_cast<uint32_t>(p) < L.n_params && L.param_handle[p] == h)
        priv[s] = 1;
    }
  }
  return priv;
}

} // namespace hgrdgpu

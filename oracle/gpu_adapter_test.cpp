// TEST INFRASTRUCTURE ONLY — extern "C" hooks that diff the reference-side
// binding (gpu_adapter.cpp: hgrd_gpu::runConcrete / enumerateVerdict over
// the reference's own Program) in-process against the unmodified reference
// (hgrd::runConcrete / enumerateVerdict, include/hgrd/oracle.hpp:57, 75).
// Built by oracle/Makefile into oracle/_ref/libhgrd_adapter.so; driven by
// tests/test_adapter.py.
#include "gpu_adapter.hpp"
#include "gpu_adapter_flat.hpp"
#include "ref_config.hpp"

#include "hgrd/parser.hpp"
#include "hgrd_gpu_program.h"

#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

namespace {

char *dupString(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string locStr(const hgrd::SourceLoc &l) {
  return l.file + ":" + std::to_string(l.line) + ":" + std::to_string(l.column);
}

struct Diff {
  std::ostringstream o;
  int n = 0;
  template <class A, class B> void eq(const A &a, const B &b, const std::string &what) {
    if (!(a == b)) {
      ++n;
      o << "differs: " << what << "\n";
    }
  }
};

void diffResults(const hgrd::OracleResult &a, const hgrd::OracleResult &b, Diff &d) {
  d.eq(a.races.size(), b.races.size(), "race count");
  for (size_t i = 0; i < a.races.size() && i < b.races.size(); ++i) {
    const auto &x = a.races[i], &y = b.races[i];
    const std::string w = "race " + std::to_string(i) + " ";
    d.eq(locStr(x.locA), locStr(y.locA), w + "locA " + locStr(x.locA) + " vs " + locStr(y.locA));
    d.eq(locStr(x.locB), locStr(y.locB), w + "locB");
    d.eq(static_cast<int>(x.kind), static_cast<int>(y.kind), w + "kind");
    d.eq(x.array, y.array, w + "array");
    d.eq(x.address, y.address, w + "address");
  }
  d.eq(a.traps, b.traps, "traps");
  d.eq(a.launchesRun, b.launchesRun, "launchesRun");
  d.eq(a.launchesSkipped, b.launchesSkipped, "launchesSkipped");
  d.eq(a.assertStopped, b.assertStopped, "assertStopped");
  d.eq(a.indirectIndexing, b.indirectIndexing, "indirectIndexing");
  d.eq(a.launchRecords.size(), b.launchRecords.size(), "launch record count");
  for (size_t i = 0; i < a.launchRecords.size() && i < b.launchRecords.size(); ++i) {
    const auto &x = a.launchRecords[i], &y = b.launchRecords[i];
    const std::string w = "launch record " + std::to_string(i) + " ";
    d.eq(x.launchStmt, y.launchStmt, w + "launchStmt (the same reference Stmt)");
    d.eq(x.grid, y.grid, w + "grid");
    d.eq(x.block, y.block, w + "block");
    d.eq(x.scalarArgs, y.scalarArgs, w + "scalarArgs");
    d.eq(x.isScalar, y.isScalar, w + "isScalar");
    d.eq(x.defValues.size(), y.defValues.size(), w + "defValues size");
    auto ia = x.defValues.begin();
    auto ib = y.defValues.begin();
    for (; ia != x.defValues.end() && ib != y.defValues.end(); ++ia, ++ib) {
      d.eq(ia->first.site, ib->first.site, w + "DefKey site");
      d.eq(ia->first.aux, ib->first.aux, w + "DefKey aux");
      d.eq(ia->first.name, ib->first.name, w + "DefKey name");
      d.eq(ia->second, ib->second, w + "def value of " + ia->first.name);
    }
  }
}

} // namespace

extern "C" {

// Dumps of the reference's parse flattened through the ABI and of the
// library's own parse of the same source (no GPU needed): equal when the
// flattening carries every node, loc and id.
int hgrd_adapter_dumps(const char *src, const char *file, char **viaAdapter, char **viaSource) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return -1;
  hgrd_gpu::FlatProgram flat(*parsed.program);
  int rc = hgrd_gpu_program_dump(flat.get(), viaAdapter);
  int rc2 = hgrd_gpu_source_dump(src, file, viaSource);
  return rc != 0 ? rc : rc2;
}

// countInputs through the adapter and the reference (no GPU needed).
int hgrd_adapter_count_inputs(const char *src, const char *file, int *ref, int *gpu) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return -1;
  *ref = hgrd::countInputs(*parsed.program);
  *gpu = hgrd_gpu::countInputs(*parsed.program);
  return 0;
}

// hgrd::runConcrete vs hgrd_gpu::runConcrete on the same parsed Program.
// Returns the number of differing fields (0: identical), -1 when the
// reference rejects the source, -2 when the GPU call throws.
int hgrd_adapter_diff_run(const char *src, const char *file, const char *cfgJson,
                          unsigned long long *instances, char **report) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok()) {
    *report = dupString("reference parse failed");
    return -1;
  }
  const hgrd::ExecConfig cfg = parseExec(cfgJson);
  hgrd::OracleResult want = hgrd::runConcrete(*parsed.program, cfg);
  hgrd::OracleResult got;
  try {
    got = hgrd_gpu::runConcrete(*parsed.program, cfg, instances);
  } catch (const std::exception &e) {
    *report = dupString(e.what());
    return -2;
  }
  Diff d;
  diffResults(want, got, d);
  *report = dupString(d.o.str());
  return d.n;
}

// hgrd::enumerateVerdict vs hgrd_gpu::enumerateVerdict (discovery order).
int hgrd_adapter_diff_sweep(const char *src, const char *file, const char *capsJson,
                            char **report) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok()) {
    *report = dupString("reference parse failed");
    return -1;
  }
  const hgrd::SweepCaps caps = parseCaps(capsJson);
  std::vector<hgrd::SweepRace> want = hgrd::enumerateVerdict(*parsed.program, caps);
  std::vector<hgrd::SweepRace> got;
  try {
    got = hgrd_gpu::enumerateVerdict(*parsed.program, caps);
  } catch (const std::exception &e) {
    *report = dupString(e.what());
    return -2;
  }
  Diff d;
  d.eq(want.size(), got.size(), "sweep race count");
  for (size_t i = 0; i < want.size() && i < got.size(); ++i) {
    const std::string w = "sweep race " + std::to_string(i) + " ";
    d.eq(locStr(want[i].locA), locStr(got[i].locA), w + "locA");
    d.eq(locStr(want[i].locB), locStr(got[i].locB), w + "locB");
    d.eq(static_cast<int>(want[i].kind), static_cast<int>(got[i].kind), w + "kind");
    d.eq(want[i].warpSize, got[i].warpSize, w + "warpSize");
  }
  *report = dupString(d.o.str());
  return d.n;
}

void hgrd_adapter_free(char *p) { std::free(p); }

} // extern "C"

// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference oracle, compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhgrd_ref.so.  It exposes:
//   * hgrd::runConcrete      (reference include/hgrd/oracle.hpp:57)
//   * hgrd::enumerateVerdict (reference include/hgrd/oracle.hpp:75)
//   * hgrd::countInputs      (reference include/hgrd/oracle.hpp:79)
// as JSON-in / JSON-out calls, so the parity tests (tests/) and the bench's
// reference arm (bench.py --impl reference) can drive the reference itself.
// The JSON schema is shared with the product's hgrd_gpu_run_concrete_json
// (include/hgrd_gpu.h) so results are compared field by field.
#include "hgrd/oracle.hpp"
#include "hgrd/parser.hpp"
#include "hgrd/report.hpp"

#include <nlohmann/json.hpp>

#include "ref_config.hpp"

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using nlohmann::ordered_json;

namespace {

char *dupString(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

ordered_json locJson(const hgrd::SourceLoc &l) {
  return ordered_json{{"file", l.file}, {"line", l.line}, {"column", l.column}};
}

ordered_json parseErrorJson(const hgrd::ParseResult &r) {
  ordered_json e = ordered_json::array();
  for (const auto &d : r.diagnostics)
    e.push_back(d.str());
  return ordered_json{{"error", e}};
}

ordered_json resultJson(const hgrd::OracleResult &r) {
  ordered_json j;
  j["races"] = ordered_json::array();
  for (const auto &race : r.races) {
    j["races"].push_back(ordered_json{{"kind", hgrd::raceKindName(race.kind)},
                                      {"locA", locJson(race.locA)},
                                      {"locB", locJson(race.locB)},
                                      {"array", race.array},
                                      {"address", race.address}});
  }
  j["traps"] = r.traps;
  j["launchesRun"] = r.launchesRun;
  j["launchesSkipped"] = r.launchesSkipped;
  j["assertStopped"] = r.assertStopped;
  j["indirectIndexing"] = r.indirectIndexing;
  j["launchRecords"] = ordered_json::array();
  for (const auto &rec : r.launchRecords) {
    ordered_json lr;
    lr["site"] = rec.launchStmt ? rec.launchStmt->nodeId : -1;
    lr["line"] = rec.launchStmt ? rec.launchStmt->loc.line : 0;
    lr["column"] = rec.launchStmt ? rec.launchStmt->loc.column : 0;
    lr["grid"] = rec.grid;
    lr["block"] = rec.block;
    lr["scalarArgs"] = rec.scalarArgs;
    std::vector<int> isScalar(rec.isScalar.begin(), rec.isScalar.end());
    lr["isScalar"] = isScalar;
    ordered_json dv = ordered_json::array();
    for (const auto &[k, v] : rec.defValues)
      dv.push_back(ordered_json::array({k.site, k.aux, k.name, v}));
    lr["defValues"] = dv;
    j["launchRecords"].push_back(lr);
  }
  return j;
}

} // namespace

extern "C" {

void hgrd_ref_free(char *p) { std::free(p); }

// runConcrete(parse(src), cfg) -> OracleResult JSON.
char *hgrd_ref_run_concrete(const char *src, const char *file,
                            const char *cfgJson) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return dupString(parseErrorJson(parsed).dump());
  hgrd::OracleResult r = hgrd::runConcrete(*parsed.program, parseExec(cfgJson));
  return dupString(resultJson(r).dump());
}

// enumerateVerdict(parse(src), caps) -> {"races":[{kind,locA,locB,warpSize}]}
// in discovery order (reference src/oracle.cpp:863-903).
char *hgrd_ref_enumerate_verdict(const char *src, const char *file,
                                 const char *capsJson) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return dupString(parseErrorJson(parsed).dump());
  auto races = hgrd::enumerateVerdict(*parsed.program, parseCaps(capsJson));
  ordered_json j;
  j["races"] = ordered_json::array();
  for (const auto &r : races)
    j["races"].push_back(ordered_json{{"kind", hgrd::raceKindName(r.kind)},
                                      {"locA", locJson(r.locA)},
                                      {"locB", locJson(r.locB)},
                                      {"warpSize", r.warpSize}});
  return dupString(j.dump());
}

int hgrd_ref_count_inputs(const char *src, const char *file) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return -1;
  return hgrd::countInputs(*parsed.program);
}

// Bench reference arm: parse once, then run runConcrete on `nThreads` host
// threads at once, `reps` times each (runConcrete is re-entrant: one
// Interpreter per call, no globals). Returns wall seconds; the races found
// by the first call are returned through *nRaces.
double hgrd_ref_time_parallel(const char *src, const char *file,
                              const char *cfgJson, int nThreads, int reps,
                              int *nRaces) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return -1.0;
  hgrd::ExecConfig cfg = parseExec(cfgJson);
  std::atomic<int> found{-1};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < nThreads; ++t)
    pool.emplace_back([&, t] {
      for (int r = 0; r < reps; ++r) {
        hgrd::OracleResult res = hgrd::runConcrete(*parsed.program, cfg);
        if (t == 0 && r == 0)
          found = static_cast<int>(res.races.size());
      }
    });
  for (auto &th : pool)
    th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (nRaces)
    *nRaces = found;
  return std::chrono::duration<double>(t1 - t0).count();
}

// The reference's STATIC analyzer (analyzeProgram, src/report.cpp:82-211),
// for the static-verdict cross-check (tests/crosscheck.py): its race
// entries {kind, locA, locB, status} under AnalyzeOptions
// {hostAnalysis, warpSize, domainBound, maxGrid, maxBlock} from optsJson.
char *hgrd_ref_analyze(const char *src, const char *file, const char *optsJson) {
  hgrd::ParseResult parsed = hgrd::parseTranslationUnit(src, file);
  if (!parsed.ok())
    return dupString(parseErrorJson(parsed).dump());
  ordered_json o = ordered_json::parse(optsJson && *optsJson ? optsJson : "{}");
  hgrd::AnalyzeOptions opts;
  if (o.contains("hostAnalysis"))
    opts.hostAnalysis = o["hostAnalysis"].get<bool>();
  if (o.contains("warpSize"))
    opts.warpSize = o["warpSize"].get<long long>();
  if (o.contains("domainBound"))
    opts.domainBound = o["domainBound"].get<long long>();
  if (o.contains("maxGrid"))
    opts.maxGrid = o["maxGrid"].get<long long>();
  if (o.contains("maxBlock"))
    opts.maxBlock = o["maxBlock"].get<long long>();
  hgrd::RaceReport rep = hgrd::analyzeProgram(*parsed.program, opts);
  ordered_json j;
  j["races"] = ordered_json::array();
  for (const auto &r : rep.races)
    j["races"].push_back(ordered_json{
        {"kind", hgrd::raceKindName(r.kind)},
        {"locA", locJson(r.locA)},
        {"locB", locJson(r.locB)},
        {"array", r.array},
        {"status", r.status == hgrd::RaceStatus::Race ? "race" : "undecided"}});
  j["hadErrors"] = rep.hadErrors;
  return dupString(j.dump());
}

// Bench reference arm of the sweep workloads (BASELINE config 5): every
// job's enumerateVerdict (parse included), the jobs spread over `nThreads`
// host threads (enumerateVerdict is re-entrant). Returns wall seconds; the
// total number of sweep races found goes to *nRaces.
double hgrd_ref_time_sweeps(const char *const *srcs, const char *const *files,
                            const char *const *capsJson, int n, int nThreads, int *nRaces) {
  std::vector<hgrd::SweepCaps> caps;
  for (int i = 0; i < n; ++i)
    caps.push_back(parseCaps(capsJson[i]));
  std::atomic<int> next{0}, races{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(nThreads, 1); ++t)
    pool.emplace_back([&] {
      for (int i; (i = next.fetch_add(1)) < n;) {
        hgrd::ParseResult parsed = hgrd::parseTranslationUnit(srcs[i], files[i]);
        if (!parsed.ok())
          continue;
        races += static_cast<int>(hgrd::enumerateVerdict(*parsed.program, caps[i]).size());
      }
    });
  for (auto &th : pool)
    th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (nRaces)
    *nRaces = races;
  return std::chrono::duration<double>(t1 - t0).count();
}

} // extern "C"

// TEST INFRASTRUCTURE ONLY — ExecConfig / SweepCaps JSON (the schema of
// the product's hgrd_gpu_run_concrete_json) parsed into the reference's own
// types (reference include/hgrd/oracle.hpp:17-25, 59-66).  Shared by
// ref_shim.cpp and gpu_adapter_test.cpp.
#pragma once

#include "hgrd/oracle.hpp"

#include <nlohmann/json.hpp>

#include <vector>

namespace {

using nlohmann::ordered_json;

template <class A> void readArr3(const ordered_json &j, const char *k, A &dst) {
  if (!j.contains(k))
    return;
  const auto &v = j.at(k);
  for (size_t i = 0; i < 3 && i < v.size(); ++i)
    dst[i] = v[i].get<long long>();
}

inline hgrd::ExecConfig parseExec(const char *cfgJson) {
  hgrd::ExecConfig c;
  ordered_json j = ordered_json::parse(cfgJson ? cfgJson : "{}");
  readArr3(j, "gridCap", c.gridCap);
  readArr3(j, "blockCap", c.blockCap);
  if (j.contains("warpSize"))
    c.warpSize = j["warpSize"].get<long long>();
  if (j.contains("inputs"))
    c.inputs = j["inputs"].get<std::vector<long long>>();
  if (j.contains("maxThreads"))
    c.maxThreads = j["maxThreads"].get<long long>();
  if (j.contains("maxArrayElems"))
    c.maxArrayElems = j["maxArrayElems"].get<long long>();
  if (j.contains("maxSteps"))
    c.maxSteps = j["maxSteps"].get<long long>();
  return c;
}

inline hgrd::SweepCaps parseCaps(const char *capsJson) {
  hgrd::SweepCaps c;
  ordered_json j = ordered_json::parse(capsJson ? capsJson : "{}");
  readArr3(j, "gridCap", c.gridCap);
  readArr3(j, "blockCap", c.blockCap);
  if (j.contains("inputSet"))
    c.inputSet = j["inputSet"].get<std::vector<long long>>();
  if (j.contains("warpSizes"))
    c.warpSizes = j["warpSizes"].get<std::vector<long long>>();
  if (j.contains("maxThreads"))
    c.maxThreads = j["maxThreads"].get<long long>();
  if (j.contains("maxConfigs"))
    c.maxConfigs = j["maxConfigs"].get<size_t>();
  return c;
}

} // namespace

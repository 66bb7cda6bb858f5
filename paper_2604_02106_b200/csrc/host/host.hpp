// Host side of the race-check stage: the reference's concrete host
// interpreter (reference src/oracle.cpp:55-437), mirrored so that every
// kernel launch is handed, fully parameterised, to a launch backend
// (the B200 kernels in the product; the CPU restatement in oracle/).
#pragma once

#include "hgrd_gpu.h"
#include "lower.hpp"
#include "minicu.hpp"

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace hgrdgpu {

// reference include/hgrd/oracle.hpp:17-25
struct ExecConfig {
  std::array<int64_t, 3> gridCap{2, 2, 1};
  std::array<int64_t, 3> blockCap{4, 1, 1};
  int64_t warpSize = 32;
  std::vector<int64_t> inputs;
  int64_t maxThreads = 64;
  int64_t maxArrayElems = 1 << 20;
  int64_t maxSteps = 1 << 20;
};

// reference include/hgrd/oracle.hpp:59-66
struct SweepCaps {
  std::array<int64_t, 3> gridCap{2, 2, 1};
  std::array<int64_t, 3> blockCap{4, 1, 1};
  std::vector<int64_t> inputSet{0, 1, 2, 3, 127};
  std::vector<int64_t> warpSizes{2, 4};
  int64_t maxThreads = 64;
  uint64_t maxConfigs = 100000;
};

// reference ObservedRace (oracle.hpp:27-32) + witness pair
struct Race {
  Loc locA, locB;
  int kind = 0;
  std::string array;
  int64_t address = 0;
  int launch = 0;           // index into launchRecords
  int64_t threadX = 0, threadY = 0;
  int seqX = 0, seqY = 0;
  int64_t blockX[3] = {0, 0, 0}, tidX[3] = {0, 0, 0};
  int64_t blockY[3] = {0, 0, 0}, tidY[3] = {0, 0, 0};
};

struct DefVal {
  std::string name;
  int64_t value = 0;
};

// reference LaunchRecord (oracle.hpp:38-45)
struct LaunchRec {
  int site = -1;
  Loc loc;
  std::array<int64_t, 3> grid{1, 1, 1}, block{1, 1, 1};
  std::vector<int64_t> scalarArgs;
  std::vector<bool> isScalar;
  std::map<std::pair<int, int>, DefVal> defValues;
};

struct RunStats {
  uint64_t instances = 0, records = 0;
  int64_t kernelSteps = 0;
  double deviceMs = 0;
  int parLaunches = 0, seqLaunches = 0, restarts = 0;
  int batchedLaunches = 0; // checked by a batched backend call (sweeps)
};

// reference OracleResult (oracle.hpp:47-55)
struct RunResult {
  std::vector<Race> races;
  std::vector<std::string> traps;
  int launchesRun = 0;
  int launchesSkipped = 0;
  bool assertStopped = false;
  bool indirectIndexing = false;
  std::vector<LaunchRec> launchRecords;
  RunStats stats;
  int error = 0; // backend failure (negative hgrd_gpu code)
  std::string errorMessage;
};

struct SweepRace {
  Loc locA, locB;
  int kind = 0;
  int64_t warpSize = 0;
};

struct SweepResult {
  std::vector<SweepRace> races;
  RunStats stats;
  uint64_t configs = 0;
  int error = 0;
  std::string errorMessage;
};

// Device (or restated) execution of the race-check stage for one launch,
// plus the int64 buffers it runs against.
class LaunchBackend {
public:
  virtual ~LaunchBackend() = default;
  virtual int reset() = 0;
  virtual int alloc(int64_t elems, int32_t *handle) = 0;
  virtual int write(int32_t h, int64_t off, int64_t n, const int64_t *src) = 0;
  virtual int read(int32_t h, int64_t off, int64_t n, int64_t *dst) = 0;
  virtual int checkLaunch(const hgrd_gpu_launch &launch, hgrd_gpu_result &res) = 0;
  // Many small launches at once (hgrd_gpu_check_batch); HGRD_GPU_ENOTSUP
  // when the backend has no batched path.
  virtual int checkBatch(const hgrd_gpu_batch_launch *, uint32_t, hgrd_gpu_result *) {
    return HGRD_GPU_ENOTSUP;
  }
  virtual bool hasBatch() const { return false; }
  virtual std::string lastError() = 0;
};

// Lowered kernels are cached per program.
struct CompiledProgram {
  std::unique_ptr<Program> program;
  std::map<const Function *, LoweredKernel> kernels;
  bool indirectIndexing = false;
  int inputs = 0;
  const LoweredKernel &kernel(const Function *k);
};

std::unique_ptr<CompiledProgram> compileProgram(std::unique_ptr<Program> p);

// lean: a sweep's run (launch records without defValues; races, traps and
// counters as always)
RunResult runConcrete(CompiledProgram &prog, const ExecConfig &cfg,
                      LaunchBackend &backend, bool lean = false);
SweepResult enumerateVerdict(CompiledProgram &prog, const SweepCaps &caps,
                             LaunchBackend &backend);
// One rank's share of enumerateVerdict's configuration lattice: the
// configs with canonical index k (warp-size major, input odometer minor,
// k <= maxConfigs) and k % world == rank, each with its sorted races.
struct ShardConfig {
  uint64_t index = 0;
  int64_t warpSize = 0;
  std::vector<Race> races;
};
struct SweepShard {
  uint64_t total = 0; // configs the full sweep runs
  std::vector<ShardConfig> configs;
  RunStats stats;
  int error = 0;
  std::string errorMessage;
};
SweepShard sweepShard(CompiledProgram &prog, const SweepCaps &caps, int rank, int world,
                      LaunchBackend &backend);
std::string sweepShardJson(const SweepShard &r, const std::string &file);
// enumerateVerdict over several backends at once (one host thread each, a
// strided share of the lattice per backend), merged in canonical order with
// the reference's first-wins dedup: the result equals enumerateVerdict's.
SweepResult enumerateVerdictParallel(CompiledProgram &prog, const SweepCaps &caps,
                                     const std::vector<LaunchBackend *> &backends);
// enumerateVerdict with the configurations' host runs done speculatively on
// `hostThreads` threads (assuming no kernel traps, no step-budget abort and
// no device values read back) and all their launches checked by one batched
// backend call; a configuration whose speculation fails is re-run exactly
// through runConcrete.  Same result as enumerateVerdict.  Falls back to it
// when the backend has no batched path.
// `workers` (optional): backends 1..nWorkers-1 run the configurations that
// cannot be speculated (sequential / lock-idiom launches, host reads of
// device results) while the batch is checked on `backend`.
SweepResult enumerateVerdictBatched(CompiledProgram &prog, const SweepCaps &caps,
                                    LaunchBackend &backend, int hostThreads,
                                    const std::function<LaunchBackend *(int)> *workers = nullptr,
                                    int nWorkers = 0);
SweepShard sweepShardBatched(CompiledProgram &prog, const SweepCaps &caps, int rank, int world,
                             LaunchBackend &backend, int hostThreads);
// Host threads for the speculative runs of a batched sweep
// (HGRD_SWEEP_THREADS, default: the hardware threads, at most 32).
int sweepHostThreads();
// Configurations enumerateVerdict runs (warp sizes x input odometer, capped).
uint64_t sweepSize(const CompiledProgram &prog, const SweepCaps &caps);
int sweepShardJsonRun(LaunchBackend &be, const char *src, const char *file,
                      const char *capsJson, int rank, int world, std::string &out);
int countInputs(const Program &p);                 // oracle.cpp:805-861
bool hasIndirectIndexing(const Program &p);        // oracle.cpp:86-123

// JSON bridges shared by the product C ABI and the oracle library.
bool parseExecConfigJson(const char *json, ExecConfig &cfg, std::string &err);
bool parseSweepCapsJson(const char *json, SweepCaps &caps, std::string &err);
std::string runResultJson(const RunResult &r, const std::string &file);
std::string sweepResultJson(const SweepResult &r, const std::string &file);
std::string errorJson(const std::vector<std::string> &diags);
const char *raceKindName(int kind);

// Full pipeline from source text (parse -> run), used by both C ABIs.
int runConcreteJson(LaunchBackend &be, const char *src, const char *file,
                    const char *cfgJson, std::string &out);
int enumerateVerdictJson(LaunchBackend &be, const char *src, const char *file,
                         const char *capsJson, std::string &out);
// Same with the configurations spread over `workers` backends.  `workers`
// returns backend i (0 = the caller's) or nullptr; used when the lattice has
// at least 4 configurations per worker.
SweepResult enumerateVerdictOnWorkers(const std::function<LaunchBackend *(int)> &workers, int n,
                                      CompiledProgram &cp, const SweepCaps &caps);
// Many programs' sweeps at once (BASELINE config 5: thousands of program x
// configuration jobs).  jobsJson: [{"source", "file", "caps"}, ...].  Every
// job's configurations (this rank's share: canonical index % world == rank)
// are run together, batched when workers(0) has a batched path.  out: one
// entry per job — its enumerateVerdict result (world 1) or its sweep shard
// (world > 1, merged by parallel.merge_shards) or its parse error.
int sweepManyJson(const std::function<LaunchBackend *(int)> &workers, int n,
                  const char *jobsJson, int rank, int world, std::string &out);
int enumerateVerdictJsonParallel(const std::function<LaunchBackend *(int)> &workers, int n,
                                 const char *src, const char *file, const char *capsJson,
                                 std::string &out);

} // namespace hgrdgpu

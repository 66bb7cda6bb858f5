/*
 * hgrd_gpu.h — C ABI of the B200 race-check stage (libhgrd_gpu.so).
 *
 * Drop-in for the data-parallel core of the reference's concrete oracle
 * (arXiv 2604.02106 "HGRD"; reference /root/reference/proj):
 *
 *   reference                                   replaced by
 *   ------------------------------------------  ------------------------------
 *   Interpreter::execLaunch thread loop +       hgrd_gpu_check_launch
 *     runThread/runThreadStmt                     (one lowered launch: expansion
 *     src/oracle.cpp:440-646                       of every (blockIdx, threadIdx)
 *   Interpreter::detectRaces                       instance + conflict detection
 *     src/oracle.cpp:730-784                       on the GPU)
 *   Interpreter buffers_ (vector<long long>)    hgrd_gpu_buffer_alloc/_write/_read
 *     src/oracle.cpp:283, 789                     (device-resident int64 buffers)
 *   hgrd::runConcrete                           hgrd_gpu_run_concrete_json
 *     include/hgrd/oracle.hpp:57                  (host front end + GPU stage)
 *   hgrd::enumerateVerdict                      hgrd_gpu_enumerate_verdict_json
 *     include/hgrd/oracle.hpp:75
 *   hgrd::countInputs  oracle.hpp:79            hgrd_gpu_count_inputs
 *
 * Conventions: plain pointers and sizes only; negative return codes are
 * errors (no exceptions cross the ABI); the caller owns every descriptor and
 * output array, a context owns its device memory; calls on one context are
 * serialised on its CUDA stream, distinct contexts may be driven from
 * distinct host threads.  There is no CPU fallback: on a machine without a
 * usable sm_100 device hgrd_gpu_create fails with HGRD_GPU_ENODEV.
 */
#ifndef HGRD_GPU_H
#define HGRD_GPU_H

#if defined(__CUDACC_RTC__) /* NVRTC (JIT-compiled race-check kernels) */
#include <cuda/std/cstdint>
#else
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------- */
#define HGRD_GPU_OK 0
#define HGRD_GPU_EINVAL (-22)   /* malformed descriptor */
#define HGRD_GPU_E2BIG (-7)     /* an output array was too small */
#define HGRD_GPU_ENODEV (-19)   /* no CUDA device / not sm_100 */
#define HGRD_GPU_ENOMEM (-12)   /* device allocation failed */
#define HGRD_GPU_ECUDA (-5)     /* CUDA runtime error (message: hgrd_gpu_last_error) */
#define HGRD_GPU_ENOTSUP (-95)  /* launch outside the supported envelope */

/* ---- lowered kernel bytecode (register machine over wrapping int64) ---- */
/* One MiniCU kernel body (reference include/hgrd/ast.hpp:101-178) lowered by
 * the host to straight-line code.  Evaluation order follows the reference
 * interpreter exactly: binary operators evaluate their RIGHT operand first
 * (src/oracle.cpp:500 as compiled by GCC), stores evaluate index then value
 * (:569-570), atomics index, value, compare (:580-583), loops re-evaluate
 * their bound every iteration (:629-631), and one STEP is charged per
 * executed statement and per loop test (:561, :630). */
enum hgrd_gpu_opcode {
  HGRD_OP_END = 0,      /* thread done (falls off the body / return)      */
  HGRD_OP_CONST = 1,    /* r[a] = imm                                      */
  HGRD_OP_MOV = 2,      /* r[a] = r[b]                                     */
  HGRD_OP_BUILTIN = 3,  /* r[a] = builtin[sub/3][sub%3] (tid,bid,bdim,gdim)*/
  HGRD_OP_BIN = 4,      /* r[a] = r[b] <sub> r[c]   (enum hgrd_gpu_binop)  */
  HGRD_OP_LOAD = 5,     /* r[a] = site imm [r[b]]; sub&1: value is needed  */
  HGRD_OP_STORE = 6,    /* site imm [r[a]] = r[b]                          */
  HGRD_OP_ATOMIC = 7,   /* site imm [r[a]] op= r[b] (cmp r[c] for CAS)     */
  HGRD_OP_SYNCTHREADS = 8,
  HGRD_OP_SYNCWARP = 9,
  HGRD_OP_FENCE = 10,   /* sub = scope                                     */
  HGRD_OP_STEP = 11,    /* charge one step; imm = statement id (trap loc)  */
  HGRD_OP_JZ = 12,      /* if r[a] == 0 goto imm                           */
  HGRD_OP_JMP = 13      /* goto imm                                        */
};

/* reference BinOp order, include/hgrd/ast.hpp:31-45 */
enum hgrd_gpu_binop {
  HGRD_ADD, HGRD_SUB, HGRD_MUL, HGRD_DIV, HGRD_MOD, HGRD_LT, HGRD_LE,
  HGRD_GT, HGRD_GE, HGRD_EQ, HGRD_NE, HGRD_AND, HGRD_OR
};

typedef struct hgrd_gpu_insn {
  uint8_t op;
  uint8_t sub;
  uint16_t a, b, c;
  uint16_t pad;
  int64_t imm;
} hgrd_gpu_insn; /* 16 bytes */

/* Access sites: one per ArrayLoad / ArrayStoreStmt / AtomicStmt node. */
enum hgrd_gpu_site_kind { HGRD_SITE_LOAD = 0, HGRD_SITE_STORE = 1, HGRD_SITE_ATOMIC = 2 };
enum hgrd_gpu_atomic_op { HGRD_ATOMIC_CAS = 0, HGRD_ATOMIC_EXCH = 1, HGRD_ATOMIC_ADD = 2 };
enum hgrd_gpu_scope { HGRD_SCOPE_NONE = 0, HGRD_SCOPE_BLOCK = 1, HGRD_SCOPE_DEVICE = 2 };

typedef struct hgrd_gpu_site {
  int32_t loc;       /* source-location id; id order == SourceLoc order      */
  int32_t param;     /* kernel parameter index the access goes through      */
  uint8_t kind;      /* hgrd_gpu_site_kind                                  */
  uint8_t atomic_op; /* hgrd_gpu_atomic_op (atomics only)                   */
  uint8_t scope;     /* hgrd_gpu_scope (atomics only; reference Event.atomicScope) */
  uint8_t pad0;
  int32_t pad1;
} hgrd_gpu_site; /* 16 bytes */

/* ---- one launch after host analysis fixed its parameters --------------- */
#define HGRD_LAUNCH_SEQUENTIAL 1u /* loaded values feed addresses/control:
                                     run instances in canonical order with
                                     memory effects (reference :440-465) */
#define HGRD_LAUNCH_PAIRWISE 2u   /* force the exhaustive pairwise detector
                                     (always used when the kernel holds
                                     fence + CAS/Exch lock idioms) */
#define HGRD_LAUNCH_NO_WITNESS 4u /* skip first-pair witness extraction */
#define HGRD_LAUNCH_GENERAL 8u    /* bypass the fused block-local check (testing) */

typedef struct hgrd_gpu_launch {
  const hgrd_gpu_insn *code;
  uint32_t n_code;
  uint32_t n_regs;
  const int64_t *reg_init;       /* n_regs initial values (scalar params)   */
  const hgrd_gpu_site *sites;
  uint32_t n_sites;
  uint32_t n_locs;
  const int32_t *param_handle;   /* per kernel param: buffer handle or -1    */
  uint32_t n_params;
  uint32_t flags;
  int64_t grid[3];
  int64_t block[3];
  int64_t warp_size;
  int64_t step_budget;           /* steps left before "step budget exhausted" */
} hgrd_gpu_launch;

/* One realised race key (locA, locB, kind) with the reference's
 * first-found report fields (array = site_x's parameter name, address =
 * index; src/oracle.cpp:766-780) and the witness pair: the first (x, y)
 * in reference iteration order, i.e. the minimum (handle, index) element,
 * then the lexicographically first event pair on it. */
typedef struct hgrd_gpu_race {
  int32_t loc_a, loc_b; /* loc_a <= loc_b */
  int32_t kind;         /* 0 INTER-BLOCK, 1 INTRA-BLOCK, 2 INTRA-WARP */
  int32_t site_x, site_y;
  int32_t handle;
  int64_t index;
  int64_t thread_x, thread_y; /* dense launch thread numbers (:457-460) */
  int32_t seq_x, seq_y;       /* per-thread event sequence numbers (:538) */
} hgrd_gpu_race;

enum hgrd_gpu_trap_kind { HGRD_TRAP_OOB = 0, HGRD_TRAP_UNALLOCATED = 1 };
typedef struct hgrd_gpu_trap {
  int32_t site;
  int32_t kind;
  int64_t thread;
} hgrd_gpu_trap;

typedef struct hgrd_gpu_result {
  hgrd_gpu_race *races;  /* caller-owned */
  uint32_t race_cap;
  uint32_t n_races;      /* set; > race_cap with HGRD_GPU_E2BIG */
  hgrd_gpu_trap *traps;  /* first trap_cap traps in canonical order */
  uint32_t trap_cap;
  uint32_t n_traps;      /* traps recorded (<= trap_cap)               */
  uint64_t n_traps_total;/* traps raised before the end / abort        */
  int64_t steps;         /* steps charged by this launch               */
  uint64_t instances;    /* in-bounds accesses = reference Events      */
  uint64_t records;      /* events kept for detection (written buffers)*/
  int32_t aborted;       /* step budget ran out inside this launch     */
  int32_t abort_stmt;    /* STEP imm at which it ran out               */
  uint32_t mode;         /* flags actually used                        */
  float device_ms;       /* device time of the check (CUDA events)     */
} hgrd_gpu_result;

/* ---- contexts and device-resident buffers ------------------------------ */
typedef struct hgrd_gpu_ctx hgrd_gpu_ctx;

#if !defined(__CUDACC_RTC__) /* host API (not visible to JIT-compiled kernels) */

int hgrd_gpu_create(int device, hgrd_gpu_ctx **out);
void hgrd_gpu_destroy(hgrd_gpu_ctx *ctx);
const char *hgrd_gpu_last_error(hgrd_gpu_ctx *ctx);

/* Drop every buffer (start of a runConcrete). */
int hgrd_gpu_buffers_reset(hgrd_gpu_ctx *ctx);
/* Zero-filled int64 buffer (reference :282-285); handles are dense from 0. */
int hgrd_gpu_buffer_alloc(hgrd_gpu_ctx *ctx, int64_t elems, int32_t *handle);
int hgrd_gpu_buffer_write(hgrd_gpu_ctx *ctx, int32_t handle, int64_t offset,
                          int64_t count, const int64_t *src);
/* hgrd_gpu_buffer_write on the context's copy stream: returns once the copy
   is queued.  The copy starts after the work already queued on the context
   (which may still read the buffer); the next check, read or write that
   touches the buffer waits for it on the device, so uploading the next
   batch overlaps the current check (B200-side addition: the reference keeps
   its buffers in host memory).  src must stay valid until that point and
   be pinned for the copy to run asynchronously. */
int hgrd_gpu_buffer_write_async(hgrd_gpu_ctx *ctx, int32_t handle, int64_t offset,
                                int64_t count, const int64_t *src);
int hgrd_gpu_buffer_read(hgrd_gpu_ctx *ctx, int32_t handle, int64_t offset,
                         int64_t count, int64_t *dst);

/* The race-check stage for one launch. */
int hgrd_gpu_check_launch(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                          hgrd_gpu_result *result);

/* ---- instrumentation --------------------------------------------------- */
/* Per-stage CUDA-event timing of the next checks (off by default). */
int hgrd_gpu_set_profiling(hgrd_gpu_ctx *ctx, int on);
/* JSON [{"name":..., "ms":...}] of the last check's stages (ctx-owned). */
const char *hgrd_gpu_last_profile(hgrd_gpu_ctx *ctx);
/* Enable (default) / disable the fused block-local check for PARALLEL launches. */
int hgrd_gpu_set_fused(hgrd_gpu_ctx *ctx, int enabled);
/* NVRTC specialisation of the expansion for each MiniCU kernel:
 * 0 off (bytecode interpreter), 1 auto (launches >= 2^14 threads, default),
 * 2 always. */
int hgrd_gpu_set_jit(hgrd_gpu_ctx *ctx, int mode);
/* JSON {"mode","compiles","compileMs","failures","lastError"} (ctx-owned). */
const char *hgrd_gpu_jit_info(hgrd_gpu_ctx *ctx);
/* Number of this library's own kernels launched by the context so far. */
unsigned long long hgrd_gpu_kernel_launches(hgrd_gpu_ctx *ctx);
/* Bytes copied host->device and device->host by this context (lifetime):
 * buffer writes/reads, launch descriptors, counters, race/trap records. */
int hgrd_gpu_transfer_bytes(hgrd_gpu_ctx *ctx, unsigned long long *h2d, unsigned long long *d2h);

/* ---- reference-shaped entry points (JSON in / JSON out) ---------------- */
/* cfg: {"gridCap":[3],"blockCap":[3],"warpSize":n,"inputs":[..],
 *       "maxThreads":n,"maxArrayElems":n,"maxSteps":n}  (ExecConfig)
 * out: {"races":[{kind,locA,locB,array,address}],"traps":[..],
 *       "launchesRun","launchesSkipped","assertStopped","indirectIndexing",
 *       "launchRecords":[..],"witnesses":[..],"stats":{..}}  (OracleResult)
 * *out must be released with hgrd_gpu_free. */
int hgrd_gpu_run_concrete_json(hgrd_gpu_ctx *ctx, const char *source,
                               const char *file_name, const char *cfg_json,
                               char **out);
/* caps: {"gridCap","blockCap","inputSet","warpSizes","maxThreads","maxConfigs"}
 * out: {"races":[{kind,locA,locB,warpSize}]} in discovery order. */
int hgrd_gpu_enumerate_verdict_json(hgrd_gpu_ctx *ctx, const char *source,
                                    const char *file_name,
                                    const char *caps_json, char **out);
/* One rank's share of the enumerateVerdict lattice for multi-GPU sweeps:
 * configs whose canonical index k satisfies k % world == rank, each with its
 * sorted races: {"total":N,"configs":[{index,warpSize,races:[{kind,locA,locB}]}]}.
 * Merging all shards in index order with first-wins (locs, kind, warpSize)
 * dedup reproduces hgrd_gpu_enumerate_verdict_json exactly. */
/* Many programs' sweeps at once (BASELINE config 5, the launch-config sweep
 * of thousands of program x configuration jobs).  jobs_json:
 * [{"source": MiniCU text, "file": name, "caps": SweepCaps}, ...].  All the
 * jobs' configurations (with world > 1 only this rank's: canonical index
 * % world == rank) are speculated on host threads and their launches
 * checked by one batched kernel.  out: a JSON array with, per job, its
 * enumerateVerdict result (world == 1), its sweep shard as
 * hgrd_gpu_sweep_shard_json returns it (world > 1), or {"error": [...]}. */
int hgrd_gpu_enumerate_verdict_many_json(hgrd_gpu_ctx *ctx, const char *jobs_json, int rank,
                                         int world, char **out);
int hgrd_gpu_sweep_shard_json(hgrd_gpu_ctx *ctx, const char *source,
                              const char *file_name, const char *caps_json,
                              int rank, int world, char **out);
int hgrd_gpu_count_inputs(const char *source, const char *file_name);
/* Lowering only: bytecode, sites, locs and per-kernel facts of one kernel as
 * JSON (for callers that fix launch parameters themselves). */
/* ---- sharded single-launch check (one launch over several GPUs) -------
 * Each rank checks the whole-block range [block_begin, block_end) of the
 * launch's dense block index:
 *  1. hgrd_gpu_shard_check: INTRA-BLOCK / INTRA-WARP races of these blocks
 *     (complete: same-block pairs never leave a shard; per key the minimum
 *     element and its first pair, merged across ranks by the caller as the
 *     lexicographic minimum of (handle, index, x, y)), the shard's counters
 *     and, when a written buffer may be reached from two blocks, the
 *     shard's INTER summary: two device tables of inter_n u32 entries per
 *     (element, site) — min and max (block + 1), empty = 0x7F7F7F7F / 0 —
 *     which the caller combines across ranks (MIN on lo, MAX on hi);
 *  2. either (a) reduce-scatter: each rank reduces one element range of the
 *     tables (e.g. ncclReduceScatter, MIN / MAX, after padding the tables to
 *     world x ranks' elements x n_sites entries) and scans it with
 *     hgrd_gpu_shard_inter_scan -> per INTER key its minimum element in the
 *     range; the ranks MIN all-reduce that n_keys table; then
 *     hgrd_gpu_shard_inter_records gives this shard's packed records of the
 *     realised keys' first-found elements (key layout identical on every
 *     rank), copied to host;
 *     or (b) all-reduce: the tables reduced in place, then
 *     hgrd_gpu_shard_inter (scan of the whole tables + the records);
 *  3. hgrd_gpu_shard_detect: the INTER-BLOCK races (with witnesses) of the
 *     records gathered from all ranks.
 * HGRD_GPU_ENOTSUP means the launch (or a shard: traps, step budget) needs
 * the ordered path: run hgrd_gpu_check_launch on every rank instead. */
typedef struct hgrd_gpu_shard {
  int64_t block_begin, block_end; /* in: dense block range of this rank   */
  uint32_t *inter_lo, *inter_hi;  /* out: device tables (or NULL)         */
  uint64_t inter_n;               /* out: entries per table (0: no INTER)  */
} hgrd_gpu_shard;

int hgrd_gpu_shard_check(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                         hgrd_gpu_shard *shard, hgrd_gpu_result *result);
int hgrd_gpu_shard_inter(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                         const hgrd_gpu_shard *shard, uint64_t *keys, uint32_t *vals,
                         uint64_t cap, uint64_t *n);
/* lo / hi: device tables of elements [elem_begin, elem_begin + n_elems)
 * (n_sites entries per element), already reduced across ranks; key_elem:
 * host, n_keys >= 3 * n_locs^2 entries, UINT64_MAX where a key has no
 * element in the range.  Runs on the context's stream (hgrd_gpu_stream):
 * the caller orders it after the collective that produced lo / hi
 * (cudaStreamWaitEvent). */
int hgrd_gpu_shard_inter_scan(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                              const void *lo, const void *hi, uint64_t elem_begin,
                              uint64_t n_elems, uint64_t *key_elem, uint32_t n_keys);
int hgrd_gpu_shard_inter_records(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                                 const hgrd_gpu_shard *shard, const uint64_t *key_elem,
                                 uint32_t n_keys, uint64_t *keys, uint32_t *vals, uint64_t cap,
                                 uint64_t *n);
/* The context's CUDA stream (cudaStream_t): every kernel of the context
 * runs on it, so a caller orders its own work (a collective on another
 * stream) before or after the context's with events. */
void *hgrd_gpu_stream(hgrd_gpu_ctx *ctx);
int hgrd_gpu_shard_detect(hgrd_gpu_ctx *ctx, const hgrd_gpu_launch *launch,
                          const uint64_t *keys, const uint32_t *vals, uint64_t n,
                          hgrd_gpu_result *result);

/* ---- batched check of many small launches (sweeps) --------------------
 * Reference enumerateVerdict (src/oracle.cpp:863-903) runs thousands of
 * configurations whose launches have a few dozen MiniCU threads; one
 * hgrd_gpu_check_launch per launch is one GPU round trip each.
 * hgrd_gpu_check_batch checks n such launches with one H2D, one kernel and
 * one D2H.  Each launch brings its own buffers (the launch's param_handle
 * indexes buffer_elems / buffer_data, which hold every buffer's size and,
 * for buffers read by value-needed loads, the launch-entry contents; NULL
 * data means zeros).  results[i] is what hgrd_gpu_check_launch would report
 * (race handles index the launch's buffers; the first trap_cap traps in
 * canonical order, n_traps_total all of them), or carries
 * HGRD_RESULT_UNCHECKED in `mode` when the launch is outside the batch
 * envelope (sequential / lock-idiom launches, more than 512 threads or 256
 * blocks, record capacity, more than 1024 traps) or needs the ordered path
 * (the step budget runs out, a hot element): check those with
 * hgrd_gpu_check_launch. */
typedef struct hgrd_gpu_batch_launch {
  hgrd_gpu_launch launch;
  const int64_t *buffer_elems;       /* n_buffers sizes */
  const int64_t *const *buffer_data; /* per buffer: contents or NULL (zeros); may be NULL */
  uint32_t n_buffers;
} hgrd_gpu_batch_launch;
#define HGRD_RESULT_UNCHECKED 0x80000000u
int hgrd_gpu_check_batch(hgrd_gpu_ctx *ctx, const hgrd_gpu_batch_launch *launches, uint32_t n,
                         hgrd_gpu_result *results);

/* Host analysis (no GPU needed): out[s] = 1 when site s's buffer is proven
 * block-private for this launch (affine indices whose per-block element
 * ranges are disjoint), so the fused path skips its ownership exchange.
 * out has launch->n_sites entries. */
int hgrd_gpu_block_private(const hgrd_gpu_launch *launch, uint8_t *out);

/* Host analysis (no GPU needed): out[s] = c when site s is a load whose
 * index is always the MiniCU thread's dense id plus the constant c (one
 * contiguous stream per fused iteration: its values are staged in shared
 * memory by TMA bulk copies), else INT64_MIN.  out has launch->n_sites
 * entries. */
int hgrd_gpu_stream_sites(const hgrd_gpu_launch *launch, int64_t *out);

/* Development check (no GPU needed): lower `kernel`, generate its NVRTC
 * thread body for the given geometry (scalar parameters 0, every site
 * recording) and compile every specialised kernel for sm_100a without
 * loading them (k_expand_par, k_fused<256,4>, <256,16>, <256,8>,
 * k_expand_seq).  *out = {"variants":[{"cubin_bytes":N,"error":"..."}x5]}.
 * Returns HGRD_GPU_ENOTSUP when a variant does not compile. */
int hgrd_gpu_jit_check(const char *source, const char *file_name, const char *kernel,
                       const int64_t grid[3], const int64_t block[3], int64_t warp_size,
                       char **out);
int hgrd_gpu_lower_json(const char *source, const char *file_name,
                        const char *kernel, char **out);
void hgrd_gpu_free(char *p);
#endif /* !__CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif
#endif /* HGRD_GPU_H */

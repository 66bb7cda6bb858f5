/*
 * hgrd_gpu_program.h — the reference's own oracle API over the C ABI.
 *
 * include/hgrd_gpu.h exports the per-launch seam (hgrd_gpu_check_launch) and
 * source-text entry points (hgrd_gpu_run_concrete_json).  This header is the
 * drop-in for the reference's public oracle API itself:
 *
 *   reference                                    replaced by
 *   -------------------------------------------  ---------------------------------
 *   hgrd::runConcrete(const Program&,            hgrd_gpu_run_concrete_program
 *                     const ExecConfig&)
 *     include/hgrd/oracle.hpp:57
 *   hgrd::enumerateVerdict(const Program&,       hgrd_gpu_enumerate_verdict_program
 *                          const SweepCaps&)
 *     include/hgrd/oracle.hpp:75
 *
 * The caller passes its already-parsed Program (reference
 * include/hgrd/ast.hpp:12-209) as flat node tables: every Expr / Stmt node
 * with its SourceLoc and nodeId, children as indices.  Nothing is re-parsed,
 * so the race reports' SourceLocs and the LaunchRecord DefKeys (keyed by node
 * ids, include/hgrd/host_facts.hpp:22-33) are the caller's own.  Results come
 * back as C structs; a LaunchRecord names its launch statement by node id.
 *
 * oracle/gpu_adapter.cpp is the reference-side binding (C++ over the
 * reference's types: hgrd_gpu::runConcrete / hgrd_gpu::enumerateVerdict with
 * the reference signatures), compiled against the reference headers.
 */
#ifndef HGRD_GPU_PROGRAM_H
#define HGRD_GPU_PROGRAM_H

#include "hgrd_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Expr::node alternatives, reference ast.hpp:84-95 (variant order) */
enum hgrd_gpu_expr_kind {
  HGRD_EXPR_INT = 0,     /* IntLit      value                       */
  HGRD_EXPR_VAR = 1,     /* VarRef      name                        */
  HGRD_EXPR_BUILTIN = 2, /* BuiltinRef  builtin (BuiltinVar), axis  */
  HGRD_EXPR_BINARY = 3,  /* BinaryExpr  op (BinOp), lhs, rhs        */
  HGRD_EXPR_LOAD = 4,    /* ArrayLoad   name (array), index         */
  HGRD_EXPR_INPUT = 5    /* InputExpr                               */
};

/* Stmt::node alternatives, reference ast.hpp:165-178 (variant order);
 * BarrierStmt and AllocStmt carry their kind in `sub`. */
enum hgrd_gpu_stmt_kind {
  HGRD_STMT_ASSIGN = 0,  /* name = value (value -1: declaration only) */
  HGRD_STMT_STORE = 1,   /* name[index] = value                       */
  HGRD_STMT_IF = 2,      /* cond, body (then), orelse                 */
  HGRD_STMT_FOR = 3,     /* aux = iterator, init, bound, step, body   */
  HGRD_STMT_BARRIER = 4, /* sub: 0 __syncthreads, 1 __syncwarp        */
  HGRD_STMT_FENCE = 5,   /* scope                                     */
  HGRD_STMT_ATOMIC = 6,  /* sub = AtomicKind, scope, name[index], value, cmp */
  HGRD_STMT_ASSERT = 7,  /* cond                                      */
  HGRD_STMT_ALLOC = 8,   /* sub: 0 cudaMalloc, 1 cudaMallocPitch; name, aux = pitch var,
                            width, height */
  HGRD_STMT_LAUNCH = 9,  /* name = kernel, grid[3], block[3], args    */
  HGRD_STMT_CALL = 10,   /* name = callee, args                       */
  HGRD_STMT_RETURN = 11  /* value (-1: none)                          */
};

enum hgrd_gpu_stmt_flags {
  HGRD_STMT_IS_DECL = 1,       /* AssignStmt::isDecl            */
  HGRD_STMT_INCLUSIVE = 2,     /* ForStmt::inclusiveBound        */
  HGRD_STMT_DECLARES_ITER = 4  /* ForStmt::declaresIter          */
};

typedef struct hgrd_gpu_expr {
  int32_t kind;       /* enum hgrd_gpu_expr_kind */
  int32_t line, col;  /* SourceLoc (the file is the program's) */
  int32_t node_id;    /* Expr::nodeId */
  int64_t value;      /* INT */
  int32_t name;       /* VAR / LOAD: string index */
  int32_t builtin;    /* BUILTIN: BuiltinVar (threadIdx, blockIdx, blockDim, gridDim) */
  int32_t axis;       /* BUILTIN: 0 x, 1 y, 2 z */
  int32_t op;         /* BINARY: BinOp (enum hgrd_gpu_binop) */
  int32_t lhs, rhs;   /* BINARY: expr indices */
  int32_t index;      /* LOAD: expr index */
} hgrd_gpu_expr;

typedef struct hgrd_gpu_stmt {
  int32_t kind;       /* enum hgrd_gpu_stmt_kind */
  int32_t line, col;  /* SourceLoc */
  int32_t node_id;    /* Stmt::nodeId */
  int32_t sub;        /* BARRIER / ALLOC kind, ATOMIC AtomicKind */
  int32_t name, aux;  /* string indices (-1: none) */
  int32_t flags;      /* enum hgrd_gpu_stmt_flags */
  int32_t decl_type;  /* ASSIGN: ParamType of a declaration */
  int32_t scope;      /* FENCE / ATOMIC: Scope (0 none, 1 block, 2 device) */
  int64_t step;       /* FOR */
  /* expr indices, -1 when absent */
  int32_t value, index, cmp, cond, init, bound, width, height;
  int32_t grid[3], block[3];
  /* ranges: args into hgrd_gpu_program.expr_list, bodies into stmt_list */
  int32_t args_begin, n_args;
  int32_t body_begin, n_body;
  int32_t else_begin, n_else;
} hgrd_gpu_stmt;

typedef struct hgrd_gpu_param {
  int32_t name;       /* string index */
  int32_t type;       /* ParamType: 0 int, 1 float*, 2 int*, 3 lock* */
  int32_t line, col;
} hgrd_gpu_param;

typedef struct hgrd_gpu_function {
  int32_t name;       /* string index */
  int32_t kernel;     /* 1: KernelDecl, 0: FunctionDecl (host) */
  int32_t line, col;
  int32_t params_begin, n_params; /* into hgrd_gpu_program.params */
  int32_t body_begin, n_body;     /* into hgrd_gpu_program.stmt_list */
} hgrd_gpu_function;

typedef struct hgrd_gpu_program {
  const char *file_name;          /* Program::fileName */
  const char *const *strings;  uint32_t n_strings;
  const hgrd_gpu_expr *exprs;  uint32_t n_exprs;
  const hgrd_gpu_stmt *stmts;  uint32_t n_stmts;
  const int32_t *expr_list;    uint32_t n_expr_list;  /* argument lists */
  const int32_t *stmt_list;    uint32_t n_stmt_list;  /* statement bodies */
  const hgrd_gpu_param *params; uint32_t n_params;
  const hgrd_gpu_function *functions; uint32_t n_functions; /* hosts, then kernels */
} hgrd_gpu_program;

/* reference ExecConfig, include/hgrd/oracle.hpp:17-25 */
typedef struct hgrd_gpu_exec_config {
  int64_t grid_cap[3];
  int64_t block_cap[3];
  int64_t warp_size;
  const int64_t *inputs; uint32_t n_inputs;
  int64_t max_threads;
  int64_t max_array_elems;
  int64_t max_steps;
} hgrd_gpu_exec_config;

/* reference SweepCaps, include/hgrd/oracle.hpp:59-66 */
typedef struct hgrd_gpu_sweep_caps {
  int64_t grid_cap[3];
  int64_t block_cap[3];
  const int64_t *input_set; uint32_t n_input_set;
  const int64_t *warp_sizes; uint32_t n_warp_sizes;
  int64_t max_threads;
  uint64_t max_configs;
} hgrd_gpu_sweep_caps;

/* ObservedRace, oracle.hpp:27-32 (+ the witness pair) */
typedef struct hgrd_gpu_observed_race {
  int32_t line_a, col_a, line_b, col_b; /* locA <= locB */
  int32_t kind;                         /* RaceKind */
  const char *array;                    /* owned by the result */
  int64_t address;
  int64_t thread_a, thread_b;           /* witness (dense thread ids) */
  int32_t launch;                       /* index into the launch records */
} hgrd_gpu_observed_race;

/* DefKey + value, host_facts.hpp:22-33 */
typedef struct hgrd_gpu_def_value {
  int32_t site, aux;
  const char *name;
  int64_t value;
} hgrd_gpu_def_value;

/* LaunchRecord, oracle.hpp:38-45 */
typedef struct hgrd_gpu_launch_record {
  int32_t launch_node_id;   /* node id of the LaunchStmt */
  int64_t grid[3], block[3];
  const int64_t *scalar_args; const uint8_t *is_scalar; uint32_t n_args;
  const hgrd_gpu_def_value *defs; uint32_t n_defs; /* ordered by DefKey */
} hgrd_gpu_launch_record;

/* OracleResult, oracle.hpp:47-55 */
typedef struct hgrd_gpu_oracle_result {
  const hgrd_gpu_observed_race *races; uint32_t n_races;  /* sorted (operator<) */
  const char *const *traps; uint32_t n_traps;
  int32_t launches_run, launches_skipped;
  int32_t assert_stopped, indirect_indexing;
  const hgrd_gpu_launch_record *launch_records; uint32_t n_launch_records;
  uint64_t instances;       /* access instances checked (not in the reference) */
} hgrd_gpu_oracle_result;

/* SweepRace, oracle.hpp:68-72 */
typedef struct hgrd_gpu_sweep_race {
  int32_t line_a, col_a, line_b, col_b;
  int32_t kind;
  int64_t warp_size;
} hgrd_gpu_sweep_race;

typedef struct hgrd_gpu_sweep_result {
  const hgrd_gpu_sweep_race *races; uint32_t n_races;  /* discovery order */
  uint64_t configs;
} hgrd_gpu_sweep_result;

/* hgrd::runConcrete.  *out is owned by the library
 * (hgrd_gpu_oracle_result_free).  HGRD_GPU_EINVAL for a malformed program
 * (message: hgrd_gpu_last_error). */
int hgrd_gpu_run_concrete_program(hgrd_gpu_ctx *ctx, const hgrd_gpu_program *program,
                                  const hgrd_gpu_exec_config *config,
                                  hgrd_gpu_oracle_result **out);
void hgrd_gpu_oracle_result_free(hgrd_gpu_oracle_result *r);

/* hgrd::enumerateVerdict (configurations spread over the context's sweep
 * workers like hgrd_gpu_enumerate_verdict_json). */
int hgrd_gpu_enumerate_verdict_program(hgrd_gpu_ctx *ctx, const hgrd_gpu_program *program,
                                       const hgrd_gpu_sweep_caps *caps,
                                       hgrd_gpu_sweep_result **out);
void hgrd_gpu_sweep_result_free(hgrd_gpu_sweep_result *r);

/* hgrd::countInputs over a flat program (no GPU needed). */
int hgrd_gpu_count_inputs_program(const hgrd_gpu_program *program);

/* Canonical dump of the program as the library sees it (node kinds, locs,
 * ids, names, values) — no GPU needed.  hgrd_gpu_source_dump gives the same
 * dump for source text parsed by the library's own front end, so a caller
 * can verify its flattening against the library's parse.  *out: free with
 * hgrd_gpu_free.  0, or HGRD_GPU_EINVAL (the dump then holds the reason). */
int hgrd_gpu_program_dump(const hgrd_gpu_program *program, char **out);
int hgrd_gpu_source_dump(const char *source, const char *file_name, char **out);

#ifdef __cplusplus
}
#endif
#endif /* HGRD_GPU_PROGRAM_H */

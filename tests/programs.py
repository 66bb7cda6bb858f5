"""MiniCU programs used by the parity tests and the bench.

* ``synthetic_*`` — the north-star workloads of SURVEY.md §8(d) / Appendix A
  (1D stencil, tiled transpose, indirect histogram), parameterised by size.
* ``EDGE_PROGRAMS`` — programs written for this repo that drive the corners
  of the reference's semantics (src/oracle.cpp): step-budget aborts, trap
  ordering and the 256-trap cap, unallocated arrays, host reads of device
  results, parameter aliasing, cross-launch first-wins, locks, loops with
  barriers, pitch allocations, host calls.
"""
from __future__ import annotations

from typing import Dict


def stencil(n_threads: int, block: int = 256, barrier: bool = False) -> str:
    """1D stencil through a per-block tile; `barrier`
    inserts the missing __syncthreads() as line 5."""
    sync = "  __syncthreads();\n" if barrier else ""
    return (
        "__global__ void st(int *in_, int *tile, int *out_) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  int base = blockIdx.x * (blockDim.x + 2);\n"
        "  tile[base + threadIdx.x + 1] = in_[t];\n"
        f"{sync}"
        "  out_[t] = tile[base + threadIdx.x] + tile[base + threadIdx.x + 2];\n"
        "}\n"
        "void main() { int *in_; int *tile; int *out_;\n"
        f"  cudaMalloc(&in_, {n_threads}); cudaMalloc(&tile, {n_threads // block * (block + 2)});"
        f" cudaMalloc(&out_, {n_threads});\n"
        f"  st<<<({n_threads // block},1,1),({block},1,1)>>>(in_, tile, out_); }}\n")


def transpose(n: int, barrier: bool = False) -> str:
    """Tiled n x n transpose through a padded 32x33 tile per block (SURVEY
    Appendix A); `barrier` inserts __syncthreads() as line 6."""
    sync = "  __syncthreads();\n" if barrier else ""
    return (
        "__global__ void tr(int *tile, int *out_, int n) {\n"
        "  int gx = blockIdx.x * 32 + threadIdx.x;\n"
        "  int gy = blockIdx.y * 32 + threadIdx.y;\n"
        "  int tb = (blockIdx.y * gridDim.x + blockIdx.x) * 1056;\n"
        "  tile[tb + threadIdx.y * 33 + threadIdx.x] = gy * n + gx;\n"
        f"{sync}"
        "  out_[(blockIdx.x * 32 + threadIdx.y) * n + blockIdx.y * 32 + threadIdx.x] = "
        "tile[tb + threadIdx.x * 33 + threadIdx.y];\n"
        "}\n"
        f"void main() {{ int *tile; int *out_; int n = {n};\n"
        "  cudaMalloc(&tile, (n/32)*(n/32)*1056); cudaMalloc(&out_, n * n);\n"
        "  tr<<<(n / 32, n / 32, 1),(32, 32, 1)>>>(tile, out_, n); }\n")


HIST_UPDATES = {
    "atomic": "  atomicAdd(hist[b], 1);\n",            # (i)  clean: device atomics cover
    "atomic_block": "  atomicAdd_block(hist[b], 1);\n",  # (ii) INTER-BLOCK only
    "store": "  hist[b] = t;\n",                          # (iii) every kind collisions allow
}

HIST_MULT = 2654435761
HIST_SEED = 0x5EED


def histogram(n_threads: int, bins: int, update: str = "store", block: int = 256,
              host_init: bool = True) -> str:
    """Global-memory histogram with data-dependent bins:
    data[i] = (i*2654435761 + 0x5eed) % bins filled by a host loop, then
    `b = data[t]` and one update per thread.  With host_init=False the host
    loop is omitted and the caller fills `data` through the buffer API."""
    init = (f"  for (int i = 0; i < {n_threads}; i++) {{ data[i] = (i * {HIST_MULT} + {HIST_SEED})"
            f" % {bins}; }}\n") if host_init else ""
    return (
        "__global__ void h(int *data, int *hist) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  int b = data[t];\n"
        f"{HIST_UPDATES[update]}"
        "}\n"
        f"void main() {{ int *data; int *hist; cudaMalloc(&data, {n_threads});"
        f" cudaMalloc(&hist, {bins});\n"
        f"{init}"
        f"  h<<<({n_threads // block},1,1),({block},1,1)>>>(data, hist); }}\n")


def histogram_data(n_threads: int, bins: int):
    """Host-side contents of `data` for histogram(host_init=False)."""
    import numpy as np
    i = np.arange(n_threads, dtype=np.int64)
    return (i * HIST_MULT + HIST_SEED) % bins


def synthetic_config(**over) -> Dict:
    """ExecConfig with the caps raised as in SURVEY Appendix A."""
    cfg = {"gridCap": [1 << 40, 1 << 40, 1 << 40], "blockCap": [1024, 1024, 64],
           "warpSize": 32, "maxThreads": 1 << 40, "maxArrayElems": 1 << 40,
           "maxSteps": 1 << 60}
    cfg.update(over)
    return cfg


EDGE_PROGRAMS: Dict[str, str] = {
    # step budget runs out inside the second launch; races of launch 1 kept
    "budget_mid_launch": (
        "__global__ void k(int *A, int n) {\n"
        "  for (int i = 0; i < n; i++) {\n"
        "    A[i] = A[i + 1];\n"
        "  }\n"
        "}\n"
        "void main() { int *A; int n = __input(); cudaMalloc(&A, 64);\n"
        "  k<<<(2,1,1),(2,1,1)>>>(A, 2);\n"
        "  k<<<(2,1,1),(4,1,1)>>>(A, n); }\n"),
    # out-of-bounds loads/stores in many threads: trap order and the 256 cap
    "trap_flood": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  A[t + 3] = A[t - 1] + A[t * 2];\n"
        "  A[t] = 1;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 4);\n"
        "  k<<<(2,1,1),(4,1,1)>>>(A);\n"
        "  for (int r = 0; r < 40; r++) { k<<<(2,1,1),(4,1,1)>>>(A); } }\n"),
    # kernel touches an array that was never allocated
    "unallocated": (
        "__global__ void k(int *A, int *B) {\n"
        "  int t = threadIdx.x;\n"
        "  B[t] = A[t];\n"
        "  A[0] = t;\n"
        "}\n"
        "void main() { int *A; int *B; cudaMalloc(&A, 4);\n"
        "  k<<<(1,1,1),(4,1,1)>>>(A, B); }\n"),
    # host reads a device result and uses it for the next launch's shape
    "host_reads_result": (
        "__global__ void fill(int *A, int v) {\n"
        "  A[threadIdx.x] = v + threadIdx.x;\n"
        "}\n"
        "__global__ void use(int *A, int *B) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  B[A[t]] = t;\n"
        "}\n"
        "void main() { int *A; int *B; int v = __input();\n"
        "  cudaMalloc(&A, 8); cudaMalloc(&B, 16);\n"
        "  fill<<<(1,1,1),(4,1,1)>>>(A, v);\n"
        "  int g = A[1];\n"
        "  if (g > 2) { use<<<(2,1,1),(2,1,1)>>>(A, B); } else { use<<<(1,1,1),(4,1,1)>>>(A, B); } }\n"),
    # value-dependent control inside a launch that writes the same buffer
    "value_control": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  if (A[0] == 0) {\n"
        "    A[t + 1] = t;\n"
        "  }\n"
        "  A[0] = 1;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 8);\n"
        "  k<<<(2,1,1),(2,1,1)>>>(A); }\n"),
    # aliasing: the same buffer behind two parameters (array = earlier event)
    "aliasing": (
        "__global__ void k(int *P, int *Q) {\n"
        "  int t = threadIdx.x;\n"
        "  Q[t] = 1;\n"
        "  int v = P[t + 1];\n"
        "}\n"
        "void main() { int *X; cudaMalloc(&X, 8);\n"
        "  k<<<(1,1,1),(4,1,1)>>>(X, X); }\n"),
    # the first launch that realises a key wins over a smaller later element
    "cross_launch_first_wins": (
        "__global__ void k(int *A, int off) {\n"
        "  A[off + threadIdx.x / 2] = 1;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 16);\n"
        "  k<<<(1,1,1),(4,1,1)>>>(A, 5);\n"
        "  k<<<(1,1,1),(4,1,1)>>>(A, 0); }\n"),
    # loop with barriers: phases beyond one per statement
    "loop_barriers": (
        "__global__ void k(int *A, int n) {\n"
        "  int t = threadIdx.x;\n"
        "  for (int i = 0; i < n; i++) {\n"
        "    A[t + i] = i;\n"
        "    if (t < 2) { __syncthreads(); }\n"
        "    __syncwarp();\n"
        "  }\n"
        "  A[t] = A[t + 1];\n"
        "}\n"
        "void main() { int *A; int n = __input(); cudaMalloc(&A, 32);\n"
        "  k<<<(2,1,1),(4,1,1)>>>(A, n); }\n"),
    # spinlock-style critical sections with mixed scopes
    "locks_mixed": (
        "__global__ void k(int *acc, lock *L) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  atomicCAS(L[t % 2], 0, 1);\n"
        "  __threadfence_block();\n"
        "  acc[0] = acc[0] + t;\n"
        "  __threadfence();\n"
        "  atomicExch(L[t % 2], 0);\n"
        "  acc[1] = t;\n"
        "}\n"
        "void main() { int *acc; lock *L; cudaMalloc(&acc, 4); cudaMalloc(&L, 2);\n"
        "  k<<<(2,1,1),(2,1,1)>>>(acc, L); }\n"),
    # cudaMallocPitch, host calls, nested ifs, unary minus, division/modulo
    "pitch_calls": (
        "__global__ void k(float *A, int pitch, int w) {\n"
        "  int x = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  int y = blockIdx.y;\n"
        "  if (x < w) {\n"
        "    A[y * pitch + x] = -x / 2 + x % 3;\n"
        "    if (x > 0) { A[y * pitch + x - 1] = A[(y + 1) % 2 * pitch + x]; }\n"
        "  }\n"
        "}\n"
        "void go(float *A, int p, int w) { k<<<(2, 2, 1),(2, 1, 1)>>>(A, p, w); }\n"
        "void main() { float *A; int pitch; int w = __input();\n"
        "  cudaMallocPitch(&A, &pitch, w, 2);\n"
        "  go(A, pitch, w); }\n"),
    # atomics of every kind/scope plus plain accesses on the same cells
    "atomic_mix": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  atomicAdd(A[t % 3], 1);\n"
        "  atomicAdd_block(A[t % 2], 1);\n"
        "  atomicExch_block(A[3], t);\n"
        "  atomicCAS(A[4], 0, t);\n"
        "  int v = A[t % 5];\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 8);\n"
        "  k<<<(2,1,1),(4,1,1)>>>(A); }\n"),
    # 3-D grids and blocks, warps spanning y
    "dims3": (
        "__global__ void k(int *A) {\n"
        "  int b = blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y;\n"
        "  int l = threadIdx.x + threadIdx.y * blockDim.x + threadIdx.z * blockDim.x * blockDim.y;\n"
        "  A[(b * 7 + l) % 11] = l;\n"
        "  A[l % 4] = A[(l + 1) % 4] + b;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 16);\n"
        "  k<<<(2,2,2),(2,2,2)>>>(A); }\n"),
    # return inside a kernel (loads in the return value are never evaluated)
    "early_return": (
        "__global__ void k(int *A, int n) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  if (t >= n) { return A[t]; }\n"
        "  A[t] = A[t + 1];\n"
        "}\n"
        "void main() { int *A; int n = __input(); cudaMalloc(&A, 16);\n"
        "  k<<<(2,1,1),(4,1,1)>>>(A, n); }\n"),
}

# Launch configs the edge programs are checked at (ExecConfig overrides).
EDGE_CONFIGS = [
    {"warpSize": 2, "inputs": [3], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2]},
    {"warpSize": 4, "inputs": [1], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2]},
    {"warpSize": 2, "inputs": [100], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2],
     "maxSteps": 300},
    {"warpSize": 32, "inputs": [2], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2],
     "maxSteps": 40},
    {"warpSize": 1, "inputs": [0], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2]},
    {"warpSize": 3, "inputs": [2, 2], "gridCap": [2, 4, 2], "blockCap": [4, 2, 2]},
]


def chain_kernel(n, a_elems):
    """Each thread reads what the previous one stored (value-relevant loads:
    canonical order, k_expand_seq); with a_elems == n the last thread's
    store is out of bounds (a trap in canonical order)."""
    return ("__global__ void k(int *A, int *B) {\n"
            "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
            "  int v = A[t];\n"
            f"  B[(v + t) % {n}] = t;\n"
            "  A[t + 1] = v + 1;\n"
            "}\n"
            f"void main() {{ int *A; int *B; cudaMalloc(&A, {a_elems}); cudaMalloc(&B, {n});\n"
            f"  k<<<({n // 256},1,1),(256,1,1)>>>(A, B); }}\n")


def lock_kernel(n, variant):
    """CAS / fence / critical section / fence / Exch on two lock words with
    64 shared cells (groups of hundreds of events: the tiled pairwise pass);
    `block` uses block-scope fences (ordering only within a block), `leak`
    adds an unprotected write after the release."""
    fence = "__threadfence_block();" if variant == "block" else "__threadfence();"
    leak = "  acc[64 + t % 7] = t;\n" if variant == "leak" else ""
    return ("__global__ void k(int *acc, lock *L) {\n"
            "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
            "  atomicCAS(L[t % 2], 0, 1);\n"
            f"  {fence}\n"
            "  acc[t % 64] = acc[t % 64] + t;\n"
            f"  {fence}\n"
            "  atomicExch(L[t % 2], 0);\n"
            f"{leak}"
            "}\n"
            f"void main() {{ int *acc; lock *L; cudaMalloc(&acc, 128); cudaMalloc(&L, 2);\n"
            f"  k<<<({n // 256},1,1),(256,1,1)>>>(acc, L); }}\n")

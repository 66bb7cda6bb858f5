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
              host_init: bool = True, seed: int = HIST_SEED) -> str:
    """Global-memory histogram with data-dependent bins:
    data[i] = (i*2654435761 + 0x5eed) % bins filled by a host loop, then
    `b = data[t]` and one update per thread.  With host_init=False the host
    loop is omitted and the caller fills `data` through the buffer API."""
    init = (f"  for (int i = 0; i < {n_threads}; i++) {{ data[i] = (i * {HIST_MULT} + {seed})"
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


def histogram_data(n_threads: int, bins: int, seed: int = HIST_SEED):
    """Host-side contents of `data` for histogram(host_init=False)."""
    import numpy as np
    i = np.arange(n_threads, dtype=np.int64)
    return (i * HIST_MULT + seed) % bins


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


# Permutation scatter ("B = n, conflict-free, with k
# injected duplicates"): data[i] = (i*M + S) mod n is a bijection for
# power-of-two n and odd M, so every bin has exactly one thread except the
# duplicated ones.  PERM_DUPS: (j, j2) host assignments data[j] = data[j2],
# chosen so the duplicate pairs realise each kind at block 256 / warp 32:
#   (9, 5)        same warp                 -> INTRA-WARP
#   (100, 37)     block 0, warps 3 and 1    -> INTRA-BLOCK
#   (1000, 70000) blocks 3 and 273          -> INTER-BLOCK
#   (600, 601)    block 2, same warp        -> INTRA-WARP (a later element)
#   (n-1, 3)      last block and block 0    -> INTER-BLOCK
PERM_DUPS = ((9, 5), (100, 37), (1000, 70000), (600, 601), (-1, 3))


def perm_dups(n_threads: int):
    return [((j if j >= 0 else n_threads + j), j2) for j, j2 in PERM_DUPS]


def permutation_scatter(n_threads: int, update: str = "store", block: int = 256,
                        host_init: bool = True) -> str:
    """Scatter through a permutation with injected duplicate targets; with
    host_init=False the host loop and duplicate assignments are omitted and
    the caller writes `data` (permutation_data)."""
    init = ""
    if host_init:
        init = (f"  for (int i = 0; i < {n_threads}; i++) {{ data[i] = (i * {HIST_MULT} + "
                f"{HIST_SEED}) % {n_threads}; }}\n")
        for j, j2 in perm_dups(n_threads):
            init += f"  data[{j}] = data[{j2}];\n"
    return (
        "__global__ void h(int *data, int *hist) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  int b = data[t];\n"
        f"{HIST_UPDATES[update]}"
        "}\n"
        f"void main() {{ int *data; int *hist; cudaMalloc(&data, {n_threads});"
        f" cudaMalloc(&hist, {n_threads});\n"
        f"{init}"
        f"  h<<<({n_threads // block},1,1),({block},1,1)>>>(data, hist); }}\n")


def permutation_data(n_threads: int):
    import numpy as np
    i = np.arange(n_threads, dtype=np.int64)
    d = (i * HIST_MULT + HIST_SEED) % n_threads
    for j, j2 in perm_dups(n_threads):
        d[j] = d[j2]
    return d


# Launches of many tiny MiniCU blocks: more blocks than one fused iteration
# holds (the per-iteration block field of k_fused's records is 8 bits).
TINY_BLOCK_PROGRAMS: Dict[str, str] = {
    # clean: each single-thread block reads and writes its own element
    "own_rw_300": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x;\n"
        "  A[t] = A[t] + 1;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 300);\n"
        "  k<<<(300,1,1),(1,1,1)>>>(A); }\n"),
    # INTER-BLOCK only: every block stores element 0
    "hot_store_300": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  A[0] = t;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 4);\n"
        "  k<<<(300,1,1),(1,1,1)>>>(A); }\n"),
    "hot_store_1024": (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  A[0] = t;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 4);\n"
        "  k<<<(1024,1,1),(1,1,1)>>>(A); }\n"),
    # hot element over > 512 two-thread blocks (radix grouping in k_fused):
    # INTRA kinds inside each block plus INTER, and block-private pairs
    "hot_pairs_600": (
        "__global__ void k(int *A, int *B) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  A[0] = t;\n"
        "  B[blockIdx.x] = B[blockIdx.x] + threadIdx.x;\n"
        "  A[1 + t % 3] = A[1 + blockIdx.x % 2];\n"
        "}\n"
        "void main() { int *A; int *B; cudaMalloc(&A, 8); cudaMalloc(&B, 600);\n"
        "  k<<<(600,1,1),(2,1,1)>>>(A, B); }\n"),
    # 3-D grid of single-thread blocks, private and shared elements
    "grid3_800": (
        "__global__ void k(int *A) {\n"
        "  int b = blockIdx.x + blockIdx.y * gridDim.x + blockIdx.z * gridDim.x * gridDim.y;\n"
        "  A[b] = A[b] + 1;\n"
        "  A[800 + b % 5] = A[800 + (b + 1) % 7];\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 816);\n"
        "  k<<<(20,20,2),(1,1,1)>>>(A); }\n"),
}


def permutation_expected(n_threads: int, update: str = "store", block: int = 256,
                         ws: int = 32):
    """The report of permutation_scatter(n_threads, update) derived from its
    structure, for sizes no CPU run reaches (2^27): only the duplicated bins
    hold two events (threads j < j2, store seq 1 each).  Reference rules
    (src/oracle.cpp:745-784): kind by block / warp, block-scope atomics cover
    pairs inside one block, and each key keeps its first-found element =
    the minimum element (ordered map by (handle, index)), witness = its pair.
    Pinned against the reference at 2^20 (tests/test_golden_extra.py).
    Returns [(kind, address, threadA, threadB)] in report order."""
    d = permutation_data(n_threads)
    best = {}
    for j, j2 in perm_dups(n_threads):
        a, b = sorted((j, j2))
        if a // block != b // block:
            kind = "INTER-BLOCK"
        elif (a % block) // ws != (b % block) // ws:
            kind = "INTRA-BLOCK"
        else:
            kind = "INTRA-WARP"
        if update == "atomic" or (update == "atomic_block" and kind != "INTER-BLOCK"):
            continue
        e = int(d[j2])
        if kind not in best or e < best[kind][0]:
            best[kind] = (e, a, b)
    order = ("INTER-BLOCK", "INTRA-BLOCK", "INTRA-WARP")
    return [(k, *best[k]) for k in order if k in best]


def histogram_pow2_expected(n_threads: int, bins: int, update: str = "store",
                            seed: int = HIST_SEED):
    """The report of histogram(n_threads, bins, update) for power-of-two
    bins >= 256 (one block of 256 never repeats a bin: the multiplier is
    odd) and n_threads >= 2 * bins: only INTER-BLOCK pairs exist, the
    first-found element is bin 0 (the minimum element, src/oracle.cpp:745),
    and its first pair is (i0, i0 + bins), i0 = the first thread mapped to
    bin 0.  [(kind, address, threadA, threadB)]; pinned against the reference
    at 2^20 / 2^22 threads x 2^16 bins (test_golden_extra.py)."""
    assert bins >= 256 and bins & (bins - 1) == 0 and n_threads >= 2 * bins
    if update == "atomic":
        return []
    i0 = (-seed * pow(HIST_MULT, -1, bins)) % bins
    return [("INTER-BLOCK", 0, i0, i0 + bins)]


def wide_lock_kernel(n_locks: int, variant: str, threads: int = 64, block: int = 16) -> str:
    """Critical sections guarded by `n_locks` locks at once: lock sets wider
    than the GPU detector's fixed sets (8), evaluated exactly
    (detect.cuh lockOrderedDirect).  `clean`: every thread takes every lock;
    `partial`: odd threads skip lock 0 (the others still order them);
    `leaky`: threads of block 1 touch the cell without taking any lock;
    `blockscope`: block-scope CAS on lock 0 (device-scope on the rest)."""
    acq, rel = [], []
    for i in range(n_locks):
        cas = "atomicCAS_block" if (variant == "blockscope" and i == 0) else "atomicCAS"
        guard = "if (t % 2 == 0) { " if (variant == "partial" and i == 0) else ""
        close = " }" if guard else ""
        acq.append(f"  {guard}{cas}(L[{i}], 0, 1);{close}\n")
        rel.append(f"  {guard}atomicExch(L[{i}], 0);{close}\n")
    body = "".join(acq) + "  __threadfence();\n"
    cs = "  acc[t % 3] = acc[t % 3] + t;\n"
    if variant == "leaky":
        body = ("  if (blockIdx.x != 1) {\n" + "".join("  " + a for a in acq) +
                "    __threadfence();\n  }\n")
        cs = "  acc[t % 3] = acc[t % 3] + t;\n"
        tail = ("  if (blockIdx.x != 1) {\n    __threadfence();\n" +
                "".join("  " + r for r in rel) + "  }\n")
    else:
        tail = "  __threadfence();\n" + "".join(rel)
    return ("__global__ void k(int *acc, lock *L) {\n"
            "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
            f"{body}{cs}{tail}"
            "}\n"
            f"void main() {{ int *acc; lock *L; cudaMalloc(&acc, 4); cudaMalloc(&L, {n_locks});\n"
            f"  k<<<({threads // block},1,1),({block},1,1)>>>(acc, L); }}\n")


WIDE_LOCK_CASES = [(n, v) for n in (9, 12) for v in ("clean", "partial", "leaky", "blockscope")]


def _overflow_programs() -> Dict[str, str]:
    """Launches past the fused kernel's fixed fields, which must fall back
    to the general / pairwise paths exactly: more than 255 barrier phases in
    a thread, more than 8 written buffers, more than 64 access sites."""
    out = {}
    out["barriers_300"] = (
        "__global__ void k(int *A, int n) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  for (int i = 0; i < n; i++) {\n"
        "    A[t] = i;\n"
        "    __syncthreads();\n"
        "  }\n"
        "  A[(t + 1) % 64] = t;\n"
        "  A[64 + t % 4] = t;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 68);\n"
        "  k<<<(2,1,1),(32,1,1)>>>(A, 300); }\n")
    params = ", ".join(f"int *B{i}" for i in range(9))
    stores = "".join(f"  B{i}[(t + {i}) % 5] = t;\n" for i in range(9))
    decls = " ".join(f"int *B{i}; cudaMalloc(&B{i}, 16);" for i in range(9))
    args = ", ".join(f"B{i}" for i in range(9))
    out["written_9"] = (
        f"__global__ void k({params}) {{\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        f"{stores}"
        "}\n"
        f"void main() {{ {decls}\n"
        f"  k<<<(2,1,1),(8,1,1)>>>({args}); }}\n")
    lines = "".join(f"  A[t * 34 + {i}] = A[t * 34 + {i + 1}];\n" for i in range(33))
    out["sites_67"] = (
        "__global__ void k(int *A) {\n"
        "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
        f"{lines}"
        "  A[t % 3] = t;\n"
        "}\n"
        "void main() { int *A; cudaMalloc(&A, 1100);\n"
        "  k<<<(2,1,1),(16,1,1)>>>(A); }\n")
    return out


OVERFLOW_PROGRAMS = _overflow_programs()


def long_thread(n_acc: int, sites: int = 2) -> str:
    """Thread 0 of one warp stores A[0 .. n_acc) (n_acc accesses, one site),
    thread 1 then stores A[n_acc - 1]: an INTRA-WARP race whose first
    witness is thread 0's access number n_acc - 1.  sites > 64 adds
    per-thread private stores so the pairwise detector runs (more sites than
    the summary detector's masks)."""
    extra = "".join(f"  P[t * {sites} + {i}] = {i};\n" for i in range(max(0, sites - 2)))
    return ("__global__ void k(int *A, int *P, int n) {\n"
            "  int t = threadIdx.x;\n"
            f"{extra}"
            "  if (t == 0) {\n"
            "    for (int i = 0; i < n; i++) {\n"
            "      A[i] = i;\n"
            "    }\n"
            "  }\n"
            "  if (t == 1) {\n"
            "    A[n - 1] = 5;\n"
            "  }\n"
            "}\n"
            f"void main() {{ int *A; int *P; cudaMalloc(&A, {n_acc}); cudaMalloc(&P, {2 * sites});\n"
            f"  k<<<(1,1,1),(2,1,1)>>>(A, P, {n_acc}); }}\n")


def wide_group(n_threads: int, block: int = 256) -> str:
    """Every thread reads B[0] after thread 0 wrote it (one element group of
    n_threads + 1 events) and stores 65 private elements (more sites than
    the summary detector's 64-bit masks: the pairwise detector runs, with
    66 * n_threads events).  Races: B[0] write / read at INTRA-WARP,
    INTRA-BLOCK and INTER-BLOCK, first witnesses thread 0 against threads
    1, 32 and `block`."""
    stores = "".join(f"  A[t * 65 + {i}] = {i};\n" for i in range(65))
    return ("__global__ void k(int *A, int *B) {\n"
            "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
            "  if (t == 0) {\n"
            "    B[0] = 7;\n"
            "  }\n"
            "  int r = B[0];\n"
            f"{stores}"
            "}\n"
            f"void main() {{ int *A; int *B; cudaMalloc(&A, {65 * n_threads}); cudaMalloc(&B, 1);\n"
            f"  k<<<({n_threads // block},1,1),({block},1,1)>>>(A, B); }}\n")

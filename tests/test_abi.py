"""CPU-side checks of the product library: it loads, exports every function
include/*.h declares, fails loudly without a device (no CPU
fallback), and its lowering honours the reference's evaluation order."""
import ctypes
import os
import re

import pytest

import paper_2604_02106_b200 as hg
import programs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    inc = os.path.join(ROOT, "include")
    for h in sorted(os.listdir(inc)):
        if h.endswith(".h"):
            text = re.sub(r"/\*.*?\*/", "", open(os.path.join(inc, h)).read(), flags=re.S)
            names |= set(re.findall(r"\b(hgrd_gpu_[a-z_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = hg.load_library()
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        hg.GpuContext(0)


def test_lowering_right_operand_first():
    """Kernel binary operators evaluate RHS first (reference oracle.cpp:500
    under GCC): in `B[t] = A[t] + A[t+1]` the A[t+1] load gets the lower seq."""
    src = ("__global__ void k(int *A, int *B) {\n  int t = threadIdx.x;\n"
           "  B[t] = A[t] + A[t + 1];\n}\n"
           "void main() { int *A; int *B; cudaMalloc(&A, 8); cudaMalloc(&B, 8);\n"
           "  k<<<1,4>>>(A, B); }\n")
    low = hg.lower(src, "k")
    loads = [s for s in low["sites"] if s["kind"] == 0]
    assert [(s["line"], s["column"]) for s in loads] == [(3, 17), (3, 10)]
    assert low["locs"] == sorted(low["locs"])


def test_value_relevance():
    low = hg.lower(programs.histogram(4096, 64, "store"), "h")
    data = [s for s in low["sites"] if s["array"] == "data"][0]
    assert data["valueNeeded"]  # b = data[t] feeds the index of hist[b]
    low = hg.lower(programs.stencil(4096), "st")
    assert not any(s["valueNeeded"] for s in low["sites"])


def test_count_inputs_matches_goldens():
    from conftest import load_golden
    for e in load_golden("corpus"):
        n = hg.count_inputs(e["source"], e["file"])
        assert n == e["source"].count("__input()")


@pytest.mark.parametrize("name", ["stencil", "transpose", "histogram"])
def test_jit_bodies_compile_for_sm100a(name):
    """The NVRTC thread bodies (jit.cpp) and all three kernels they are
    specialised into compile for sm_100a (NVRTC needs no device)."""
    src, kernel, grid, block = {
        "stencil": (programs.stencil(1 << 12), "st", (16, 1, 1), (256, 1, 1)),
        "transpose": (programs.transpose(256), "tr", (8, 8, 1), (32, 32, 1)),
        "histogram": (programs.histogram(1 << 12, 64, "store"), "h", (16, 1, 1), (256, 1, 1)),
    }[name]
    d = hg.jit_check(src, kernel, grid, block)
    assert all(v["cubin_bytes"] > 0 for v in d["variants"]), d


def _block_private(src, kernel, grid, block, handles, scalars=None):
    low = hg.lower(src, kernel)
    spec = hg.LaunchSpec(low, grid, block, 32, handles=handles, scalars=scalars)
    return {(s["array"], s["kind"]): p for s, p in zip(low["sites"], spec.block_private())}


def test_block_private_analysis():
    """Affine partition proof (csrc/gpu/affine.cpp) that lets the fused path
    skip ownership exchanges: per-block tiles are private, a transposed
    store and data-dependent bins are not, aliasing defeats the proof."""
    st = programs.stencil(1 << 12)
    got = _block_private(st, "st", (16, 1, 1), (256, 1, 1), {"in_": 0, "tile": 1, "out_": 2})
    assert all(got.values())
    # tile and out_ aliased: strides 258 vs 256 per block -> no proof
    got = _block_private(st, "st", (16, 1, 1), (256, 1, 1), {"in_": 0, "tile": 1, "out_": 1})
    assert not got[("tile", 1)] and not got[("out_", 1)] and got[("in_", 0)]
    tr = programs.transpose(256)
    got = _block_private(tr, "tr", (8, 8, 1), (32, 32, 1), {"tile": 0, "out_": 1}, {"n": 256})
    # out_'s per-block ranges interleave, but its single index form is
    # injective over (threadIdx, blockIdx) in mixed radix (test B)
    assert got[("tile", 1)] and got[("out_", 1)]
    for n, ok in ((64, True), (4, True), (3, False)):  # A[tx * n + bx], 4 blocks
        src = ("__global__ void k(int *A, int n) {\n  A[threadIdx.x * n + blockIdx.x] = 1;\n}\n"
               "void main() { int *A; cudaMalloc(&A, 8192); k<<<4,32>>>(A, 64); }\n")
        assert _block_private(src, "k", (4, 1, 1), (32, 1, 1), {"A": 0}, {"n": n})[("A", 1)] is ok
    src = ("__global__ void k(int *A, int n) {\n  A[threadIdx.x * n + blockIdx.y] = 1;\n}\n"
           "void main() { int *A; cudaMalloc(&A, 8192); k<<<(2,4,1),(32,1,1)>>>(A, 64); }\n")
    # blockIdx.x does not move the index: blocks (0, y) and (1, y) share elements
    assert not _block_private(src, "k", (2, 4, 1), (32, 1, 1), {"A": 0}, {"n": 64})[("A", 1)]
    hist = programs.histogram(1 << 12, 64)
    got = _block_private(hist, "h", (16, 1, 1), (256, 1, 1), {"data": 0, "hist": 1})
    assert got[("data", 0)] and not got[("hist", 1)]
    # a block stride equal to the tile width still separates; one less does not
    for stride, ok in ((256, True), (255, False)):
        src = ("__global__ void k(int *A) {\n"
               f"  A[blockIdx.x * {stride} + threadIdx.x] = 1;\n}}\n"
               "void main() { int *A; cudaMalloc(&A, 8192);\n"
               "  k<<<16,256>>>(A); }\n")
        assert _block_private(src, "k", (16, 1, 1), (256, 1, 1), {"A": 0})[("A", 1)] is ok
    # loops: no proof
    src = ("__global__ void k(int *A) {\n  for (int i = 0; i < 2; i++) {\n"
           "    A[blockIdx.x * 512 + threadIdx.x + i] = 1;\n  }\n}\n"
           "void main() { int *A; cudaMalloc(&A, 8192);\n  k<<<4,256>>>(A); }\n")
    assert not _block_private(src, "k", (4, 1, 1), (256, 1, 1), {"A": 0})[("A", 1)]


def _stream(src, kernel, grid, block, handles, scalars=None):
    low = hg.lower(src, kernel)
    spec = hg.LaunchSpec(low, grid, block, 32, handles=handles, scalars=scalars)
    return {(s["array"], s["kind"]): p for s, p in zip(low["sites"], spec.stream_sites())}


def test_stream_sites_analysis():
    """Streamed loads (affine.cpp streamSites): an index that is always the
    dense thread id (blockLin * tpb + threadLin, reference oracle.cpp:443-460)
    plus a constant, whose values k_fused stages by TMA bulk copies."""
    hist = programs.histogram(1 << 12, 64)
    got = _stream(hist, "h", (16, 1, 1), (256, 1, 1), {"data": 0, "hist": 1})
    assert got[("data", 0)] == 0 and got[("hist", 1)] is None
    perm = programs.permutation_scatter(1 << 17, host_init=False)
    assert _stream(perm, "h", (512, 1, 1), (256, 1, 1), {"data": 0, "hist": 1})[("data", 0)] == 0
    st = programs.stencil(1 << 12)  # in_[t]: the stream; tile loads are not
    got = _stream(st, "st", (16, 1, 1), (256, 1, 1), {"in_": 0, "tile": 1, "out_": 2})
    assert got[("in_", 0)] == 0 and got[("tile", 0)] is None
    # 2-D: t = (by * gx + bx) * tpb + ty * bdx + tx, offset 5
    src = ("__global__ void k(int *A, int *B) {\n"
           "  int t = (blockIdx.y * gridDim.x + blockIdx.x) * (blockDim.x * blockDim.y)"
           " + threadIdx.y * blockDim.x + threadIdx.x;\n"
           "  B[A[t + 5]] = 1;\n}\n"
           "void main() { int *A; int *B; cudaMalloc(&A, 8192); cudaMalloc(&B, 64);\n"
           "  k<<<(4,2,1),(8,4,1)>>>(A, B); }\n")
    assert _stream(src, "k", (4, 2, 1), (8, 4, 1), {"A": 0, "B": 1})[("A", 0)] == 5
    # transposed thread order: not the dense id
    src2 = src.replace("threadIdx.y * blockDim.x + threadIdx.x", "threadIdx.x * blockDim.y + threadIdx.y")
    assert _stream(src2, "k", (4, 2, 1), (8, 4, 1), {"A": 0, "B": 1})[("A", 0)] is None

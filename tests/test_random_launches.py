"""Randomised launch-level parity at GPU-relevant sizes.

Straight-line MiniCU kernels with affine, modular and data-dependent
indices, barriers, warp syncs, branches and atomics of every scope, on 1-D
and 2-D grids of up to a few thousand threads, checked through every GPU
pipeline — the fused kernel with NVRTC bodies (push-time pairing, affine
privacy proofs, the single-site INTER scan), the general global-sort
pipeline and the ordered SEQUENTIAL path — against the CPU restatement of
the reference (oracle/cpu_oracle.cpp, pinned to the reference by
test_oracle_pin.py).  Races (with witness pairs), traps, steps and instance
counts must be identical."""
import random

import numpy as np
import pytest

import paper_2604_02106_b200 as hg

ARRAYS = {"A": 97, "B": 256, "C": 4096, "D": 64}  # D: read-only index data


def _index(rng, arr, size):
    if arr == "C" and rng.random() < 0.3:  # exact affine forms: block-private proofs
        return rng.choice(["t2", "blockIdx.x * blockDim.x + threadIdx.x",
                           "threadIdx.x * 64 + blockIdx.x"])
    if arr == "A" and rng.random() < 0.05:  # out of bounds for larger launches: traps
        return "t"
    t = rng.choice(["t", "threadIdx.x", "blockIdx.x", "l", "t2"])
    form = rng.randrange(7)
    c = rng.randrange(1, 5)
    k = rng.randrange(0, 9)
    if form == 0:
        e = f"{t}"
    elif form == 1:
        e = f"{t} + {k}"
    elif form == 2:
        e = f"{t} * {c} + {k}"
    elif form == 3:
        e = f"blockIdx.x * {size // 8 or 1} + threadIdx.x"
    elif form == 4:
        e = f"D[{t} % 64]"  # data-dependent (read-only buffer: PARALLEL mode)
    elif form == 5:
        e = f"({t} * 7 + {k}) / {c}"
    else:
        e = f"{k}"
    return f"({e}) % {size}"


def _kernel(rng):
    lines = ["  int t = blockIdx.x * blockDim.x + threadIdx.x;",
             "  int l = threadIdx.x + threadIdx.y * blockDim.x;",
             "  int t2 = t + blockIdx.y * gridDim.x * blockDim.x * blockDim.y;",
             "  int x = 0;"]
    depth = 0
    for _ in range(rng.randrange(3, 9)):
        arr = rng.choice("ABC")
        idx = _index(rng, arr, ARRAYS[arr])
        op = rng.randrange(14)
        pad = "  " * (depth + 1)
        if op < 4:
            lines.append(f"{pad}{arr}[{idx}] = t;")
        elif op < 7:
            lines.append(f"{pad}x = x + {arr}[{idx}];")
        elif op == 7:
            lines.append(f"{pad}__syncthreads();")
        elif op == 8:
            lines.append(f"{pad}__syncwarp();")
        elif op == 9:
            lines.append(f"{pad}atomicAdd({arr}[{idx}], 1);")
        elif op == 10:
            lines.append(f"{pad}atomicAdd_block({arr}[{idx}], 1);")
        elif op == 11:
            lines.append(f"{pad}atomicExch({arr}[{idx}], t);")
        elif op == 12 and depth == 0:
            lines.append(f"{pad}if (l % {rng.randrange(2, 5)} == {rng.randrange(2)}) {{")
            depth = 1
        elif depth:
            lines.append("  }")
            depth = 0
    if depth:
        lines.append("  }")
    return ("__global__ void k(int *A, int *B, int *C, int *D) {\n" + "\n".join(lines) +
            "\n}\nvoid main() { }\n")


def _case(seed):
    rng = random.Random(seed)
    src = _kernel(rng)
    grid = rng.choice([(8, 1, 1), (33, 1, 1), (64, 1, 1), (4, 3, 1)])
    block = rng.choice([(32, 1, 1), (64, 1, 1), (96, 1, 1), (16, 4, 1)])
    ws = rng.choice([32, 32, 16, 5])
    data = np.array([rng.randrange(0, 4096) for _ in range(ARRAYS["D"])], dtype=np.int64)
    return src, grid, block, ws, data


def _specs(src, grid, block, ws, data, ctx):
    low = hg.lower(src, "k")
    names = list(ARRAYS)
    bufs = [np.zeros(ARRAYS[n], np.int64) for n in names]
    bufs[names.index("D")] = data
    if ctx is not None:
        ctx.reset()
        h = {n: ctx.alloc(ARRAYS[n]) for n in names}
        ctx.write(h["D"], data)
    else:
        h = {n: i for i, n in enumerate(names)}
    return hg.LaunchSpec(low, grid, block, ws, handles=h), bufs


def _same(a, b):
    keys = ("races", "traps", "steps", "instances", "aborted")
    return {k: a[k] for k in keys} == {k: b[k] for k in keys}


def test_generator_lowers():
    """The generator only produces kernels the front end accepts (CPU)."""
    for seed in range(40):
        src, *_ = _case(seed)
        hg.lower(src, "k")


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", range(4))
def test_random_launches(gpu, cpu_oracle, chunk):
    try:
        mismatches = []
        for seed in range(chunk * 50, chunk * 50 + 50):
            # every 4th case through NVRTC bodies (compile ~1 s), the rest
            # through the bytecode interpreter
            gpu.set_jit(2 if seed % 4 == 0 else 0)
            src, grid, block, ws, data = _case(seed)
            spec, bufs = _specs(src, grid, block, ws, data, gpu)
            ref_spec, _ = _specs(src, grid, block, ws, data, None)
            want = cpu_oracle.check_launch(ref_spec, bufs)
            got = gpu.check_launch(spec)
            if not _same(got, want):
                mismatches.append((seed, "fused", got["races"], want["races"]))
                continue
            spec.launch.flags |= hg.LAUNCH_GENERAL
            if not _same(gpu.check_launch(spec), want):
                mismatches.append((seed, "general"))
                continue
            spec.launch.flags |= hg.LAUNCH_SEQUENTIAL
            if not _same(gpu.check_launch(spec), want):
                mismatches.append((seed, "sequential"))
        assert not mismatches, mismatches[:3]
    finally:
        gpu.set_jit(1)

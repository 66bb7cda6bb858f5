"""JitBody::run2 (two MiniCU threads per call, both value loads in flight):
branch-free bodies with a value-needed global load, at geometries whose
iterations end on a lone thread (the single-thread tail), with out-of-range
loads (traps: the fused attempt hands over to the ordered path), forced
through the NVRTC bodies and compared with the CPU restatement field by
field, witnesses included."""
import pytest

import programs
from oracles import strip_extras

pytestmark = pytest.mark.gpu

GATHER = """__global__ void g(int *A, int *B, int *C) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int v = A[(t * 7) % MOD];
  B[t] = v + 1;
  UPDATE
}
void main() { int *A; int *B; int *C; cudaMalloc(&A, 997); cudaMalloc(&B, NT);
  cudaMalloc(&C, 50);
  for (int i = 0; i < 997; i++) { A[i] = i * 3; }
  g<<<(GRID,1,1),(BLOCK,1,1)>>>(A, B, C); }
"""

UPDATES = {"store": "C[v % 50] = t;", "atomic": "atomicAdd(C[v % 50], 1);",
           "none": "B[t] = B[t] + v;"}


def _src(grid, block, update, mod=997):
    return (GATHER.replace("MOD", str(mod)).replace("NT", str(grid * block))
            .replace("GRID", str(grid)).replace("BLOCK", str(block))
            .replace("UPDATE", UPDATES[update]))


def _same(got, want, what):
    assert "error" not in want, want
    assert strip_extras(got) == strip_extras(want), what
    assert got["witnesses"] == want["witnesses"], what
    assert got["stats"]["instances"] == want["stats"]["instances"], what


@pytest.mark.parametrize("grid,block", [(333, 100), (41, 1024), (1000, 7), (3, 33)])
@pytest.mark.parametrize("update", sorted(UPDATES))
def test_pair_bodies(gpu, cpu_oracle, grid, block, update):
    src = _src(grid, block, update)
    gpu.set_jit(2)
    try:
        for ws in (32, 4):
            cfg = programs.synthetic_config(warpSize=ws)
            _same(gpu.run_concrete(src, cfg, "pair.mcu"),
                  cpu_oracle.run_concrete(src, cfg, "pair.mcu"), (grid, block, update, ws))
    finally:
        gpu.set_jit(1)


def test_pair_bodies_with_traps(gpu, cpu_oracle):
    src = _src(333, 100, "store", mod=1000)  # A[997..999]: out of range
    gpu.set_jit(2)
    try:
        cfg = programs.synthetic_config()
        want = cpu_oracle.run_concrete(src, cfg, "pair.mcu")
        assert want["traps"]
        _same(gpu.run_concrete(src, cfg, "pair.mcu"), want, "traps")
    finally:
        gpu.set_jit(1)

"""One launch split over several ranks by whole-block ranges
(paper_2604_02106_b200.parallel.check_launch_sharded)
must report exactly what the unsharded check reports.

The driver gives these tests one GPU, so the ranks are threads of this
process, each with its own context on cuda:0, and the collectives are an
in-process exchange (ThreadComm).  The kernels of different ranks never
wait on one another: every collective is a host-side rendezvous between
kernel launches, exactly as the NCCL path (TorchComm) runs them."""
import threading

import numpy as np
import pytest

import paper_2604_02106_b200 as hg
from paper_2604_02106_b200.parallel import block_ranges, check_launch_sharded
from test_gpu_parity import _same, _spec_hist, _spec_stencil, _spec_transpose
import programs


class ThreadComm:
    """In-process stand-in for TorchComm: rank threads rendezvous on a barrier."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def rank(self, r):
        outer = self

        class Rank:
            rank, world = r, outer.world

            def allgather(self, obj):
                outer.slots[r] = obj
                outer.barrier.wait()
                out = list(outer.slots)
                outer.barrier.wait()
                return out

            def reduce_scatter_minmax(self, lo, hi, unit):
                import torch
                from paper_2604_02106_b200.parallel import element_slices
                parts = self.allgather((lo.cpu(), hi.cpu()))
                rlo = torch.stack([p[0] for p in parts]).min(0).values
                rhi = torch.stack([p[1] for p in parts]).max(0).values
                b, e = element_slices(lo.numel() // unit, self.world)[r]
                return (rlo[b * unit: e * unit].to(lo.device),
                        rhi[b * unit: e * unit].to(lo.device), b, e - b)

            def allreduce_min_u64(self, v, device=None):
                return np.minimum.reduce(self.allgather(v.copy()))

        return Rank()


def run_sharded(make_spec, world):
    """make_spec(ctx) -> (spec, bufs); returns (sharded results per rank, full result)."""
    comm = ThreadComm(world)
    ctxs = [hg.GpuContext(0) for _ in range(world)]
    specs = [make_spec(c)[0] for c in ctxs]
    out = [None] * world
    errs = []

    def work(r):
        try:
            out[r] = check_launch_sharded(ctxs[r], specs[r], comm.rank(r))
        except Exception as e:  # surfaced below
            errs.append(e)
            comm.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    full_ctx = hg.GpuContext(0)
    full = full_ctx.check_launch(make_spec(full_ctx)[0])
    for c in ctxs + [full_ctx]:
        c.close()
    return out, full


def test_block_ranges():
    assert block_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert block_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("barrier", [False, True])
def test_sharded_stencil(world, barrier):
    out, full = run_sharded(lambda c: _spec_stencil(c, 1 << 14, barrier), world)
    assert full["races"] or barrier
    for o in out:
        assert o["path"] == "sharded" and o["interRecords"] == 0  # block-private buffers
        assert _same(o, full), (o["races"], full["races"])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("update", ["store", "atomic_block", "atomic"])
@pytest.mark.parametrize("bins", [64, 61])
def test_sharded_histogram(world, update, bins):
    out, full = run_sharded(lambda c: _spec_hist(c, 1 << 13, bins, update), world)
    assert bool(full["races"]) == (update != "atomic")
    for o in out:
        assert o["path"] == "sharded"
        assert (o["interRecords"] > 0) == (update != "atomic")
        assert _same(o, full), (o["races"], full["races"])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("barrier", [False, True])
def test_sharded_transpose(world, barrier):
    out, full = run_sharded(lambda c: _spec_transpose(c, 128, barrier), world)
    for o in out:
        assert o["path"] == "sharded"
        assert _same(o, full)


def _spec_mixed(ctx, n=4096, ws=32):
    """INTER and INTRA races on one buffer plus an out-of-range shard-local
    pattern: A[t % 97] is written by every block, B[t / 2] by thread pairs."""
    src = ("__global__ void k(int *A, int *B) {\n"
           "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
           "  A[t % 97] = B[t / 2];\n"
           "  B[t / 2] = t;\n"
           "}\n"
           f"void main() {{ int *A; int *B; cudaMalloc(&A, 97); cudaMalloc(&B, {n}); "
           f"k<<<{n // 128},128>>>(A, B); }}\n")
    low = hg.lower(src, "k")
    if ctx is not None:
        ctx.reset()
        h = {"A": ctx.alloc(97), "B": ctx.alloc(n)}
    else:
        h = {"A": 0, "B": 1}
    return hg.LaunchSpec(low, (n // 128, 1, 1), (128, 1, 1), ws, handles=h), None


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 5])
@pytest.mark.parametrize("ws", [32, 5])
def test_sharded_mixed_kinds(world, ws):
    out, full = run_sharded(lambda c: _spec_mixed(c, ws=ws), world)
    kinds = {r["kind"] for r in full["races"]}
    assert "INTER-BLOCK" in kinds and "INTRA-WARP" in kinds
    for o in out:
        assert o["path"] == "sharded" and o["interRecords"] > 0
        assert _same(o, full), (o["races"], full["races"])


def _spec_trapping(ctx):
    """The last thread stores past the end: the ordered path is required."""
    src = ("__global__ void k(int *A) {\n"
           "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n"
           "  A[t + 1] = A[t];\n}\n"
           "void main() { int *A; cudaMalloc(&A, 1024); k<<<8,128>>>(A); }\n")
    low = hg.lower(src, "k")
    h = {"A": ctx.alloc(1024)} if ctx is not None else {"A": 0}
    return hg.LaunchSpec(low, (8, 1, 1), (128, 1, 1), 32, handles=h), None


@pytest.mark.gpu
def test_sharded_falls_back_on_traps():
    out, full = run_sharded(_spec_trapping, 2)
    assert full["traps"]
    for o in out:
        assert o["path"] == "replicas"
        assert _same(o, full)

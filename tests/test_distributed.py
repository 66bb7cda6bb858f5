"""Multi-rank sharding of the sweep (paper_2604_02106_b200/parallel.py).

CPU tests: world_size-2 gloo process groups where each rank runs its shard of
the configuration lattice through the CPU restatement (the same host code the
GPU library runs, behind the same shard entry point), gathers, merges, and
must reproduce the reference's own single-process enumerateVerdict output
(tests/golden).  The GPU test checks hgrd_gpu_sweep_shard_json on one device
for every (rank, world) split."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden
from paper_2604_02106_b200.parallel import (enumerate_verdict_distributed, merge_shards,
                                            shard_jobs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_merge_shards_any_world(cpu_oracle):
    corpus = load_golden("corpus")
    for e in corpus:
        for world in (1, 2, 3, 8):
            shards = [cpu_oracle.sweep_shard(e["source"], e["caps"], e["file"], r, world)
                      for r in range(world)]
            got = merge_shards(shards)
            assert got["races"] == e["sweep_manifest"]["races"], (e["name"], world)
            assert sum(len(s["configs"]) for s in shards) == got["configs"]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracles import CpuOracle
    ora = CpuOracle()
    bad = []
    for e in load_golden("corpus"):
        got = enumerate_verdict_distributed(ora.sweep_shard, e["source"], e["caps"], e["file"])
        if got["races"] != e["sweep_manifest"]["races"]:
            bad.append(e["name"])
    for f in load_golden("fuzz")[:60]:
        got = enumerate_verdict_distributed(ora.sweep_shard, f["source"], {}, "fuzz.mcu")
        if got["races"] != f["sweep"]["races"]:
            bad.append(f["index"])
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write(repr(bad))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sweep_matches_reference(tmp_path):
    world = 2
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{out}.{r}").read() == "[]"


def test_shard_jobs_partition():
    jobs = [{"id": i, "cost": (i % 7) + 1} for i in range(100)]
    parts = [shard_jobs(jobs, r, 4) for r in range(4)]
    ids = sorted(j["id"] for p in parts for j in p)
    assert ids == list(range(100))
    loads = [sum(j["cost"] for j in p) for p in parts]
    assert max(loads) - min(loads) <= 7


@pytest.mark.gpu
def test_gpu_sweep_shards(gpu):
    for e in load_golden("corpus"):
        for world in (1, 2, 4):
            shards = [gpu.sweep_shard(e["source"], e["caps"], e["file"], r, world)
                      for r in range(world)]
            assert merge_shards(shards)["races"] == e["sweep_manifest"]["races"], e["name"]


def _comm_worker(rank, world, port, out):
    """TorchComm over gloo: the sharded launch's collectives (MIN / MAX of the
    INTER summary tables, gather of the per-rank INTRA races and records)."""
    import numpy as np
    import torch
    from paper_2604_02106_b200.parallel import TorchComm, block_ranges
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        assert (comm.rank, comm.world, comm.nccl) == (rank, world, False)
        empty = 0x7F7F7F7F  # kShardEmpty: positive as int32
        # element e touched by block 2e+rank on rank `rank` when e % world == rank,
        # element 0 by every rank (-> MULTI after the reduction)
        lo = torch.full((8,), empty, dtype=torch.int32)
        hi = torch.zeros(8, dtype=torch.int32)
        for e in range(8):
            if e % world == rank or e == 0:
                lo[e] = hi[e] = 2 * e + rank + 1
        rlo, rhi, e0, ne = comm.reduce_scatter_minmax(lo.clone(), hi.clone(), 2)
        ke = np.full(6, (1 << 64) - 1, dtype=np.uint64)
        ke[rank] = 10 + rank
        ke[3] = 7 - rank
        ke_red = comm.allreduce_min_u64(ke)
        comm.allreduce_minmax(lo, hi)
        got = comm.allgather({"rank": rank, "keys": np.arange(rank + 1, dtype=np.uint64)})
        res = {"lo": lo.tolist(), "hi": hi.tolist(), "ranks": [g["rank"] for g in got],
               "rs": [rank, rlo.tolist(), rhi.tolist(), e0, ne], "ke": ke_red.tolist(),
               "nkeys": [len(g["keys"]) for g in got], "ranges": block_ranges(9, world)}
        open(f"{out}.{rank}", "w").write(repr(res))
    finally:
        dist.destroy_process_group()


def _sharded_worker(rank, world, port, out):
    """check_launch_sharded end to end: one process per rank, each with its
    own context on cuda:0, collectives over gloo (host-side rendezvous between
    kernels: no kernel waits on another rank's)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import paper_2604_02106_b200 as hg
    from paper_2604_02106_b200.parallel import TorchComm, check_launch_sharded
    from test_gpu_parity import _spec_hist, _spec_stencil, _spec_transpose
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys = ("races", "steps", "instances", "records")
    try:
        ctx = hg.GpuContext(0)
        comm = TorchComm()
        bad = []
        cases = [("stencil", lambda c: _spec_stencil(c, 1 << 14, False)),
                 ("transpose", lambda c: _spec_transpose(c, 128, False)),
                 ("hist64_store", lambda c: _spec_hist(c, 1 << 13, 64, "store")),
                 ("hist61_block", lambda c: _spec_hist(c, 1 << 13, 61, "atomic_block")),
                 ("hist1024_atomic", lambda c: _spec_hist(c, 1 << 13, 1024, "atomic"))]
        for name, mk in cases:
            spec = mk(ctx)[0]
            got = check_launch_sharded(ctx, spec, comm, device=0)
            full = ctx.check_launch(mk(ctx)[0])
            if got.get("path") != "sharded" or {k: got[k] for k in keys} != \
                    {k: full[k] for k in keys}:
                bad.append(name)
        open(f"{out}.{rank}", "w").write(repr(bad))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_check_launch_sharded_gpu(tmp_path):
    world = 2
    out = str(tmp_path / "sharded")
    mp.spawn(_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{out}.{r}").read() == "[]"


def test_gloo_world2_shard_collectives(tmp_path):
    world = 2
    out = str(tmp_path / "comm")
    mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [eval(open(f"{out}.{r}").read()) for r in range(world)]
    # reduce-scatter: rank r holds elements [2r, 2r + 2) of the 4 two-site elements
    for r in range(world):
        rank, rlo, rhi, e0, ne = res[r].pop("rs")
        assert (e0, ne) == (2 * rank, 2)
        assert rlo == res[r]["lo"][4 * rank: 4 * rank + 4]
        assert rhi == res[r]["hi"][4 * rank: 4 * rank + 4]
    big = (1 << 64) - 1
    assert res[0]["ke"] == [10, 11, big, 6, big, big]
    assert res[0] == res[1]
    lo, hi = res[0]["lo"], res[0]["hi"]
    assert (lo[0], hi[0]) == (1, 2)  # element 0: blocks of both ranks -> lo != hi (MULTI)
    for e in range(1, 8):
        assert lo[e] == hi[e] == 2 * e + (e % world) + 1  # one block: not MULTI
    assert res[0]["ranks"] == [0, 1] and res[0]["nkeys"] == [1, 2]
    assert res[0]["ranges"] == [(0, 5), (5, 9)]

"""Multi-GPU sharding of the race-check stage (one process per GPU).

The configuration lattice of ``enumerateVerdict`` (reference
src/oracle.cpp:863-903: warp sizes outer, input odometer inner, at most
``maxConfigs + 1`` configs) consists of independent ``runConcrete`` runs, so it
shards with no data-path collective: rank r runs the configs whose canonical
index k satisfies ``k % world == r`` (``hgrd_gpu_sweep_shard_json``), and the
per-config race lists are merged in index order with the reference's
first-wins ``(lineA, colA, lineB, colB, kind, warpSize)`` dedup — the output
is identical to the single-GPU sweep.  The only communication is gathering
the (small) per-config reports, done here with ``torch.distributed``
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Dict, Iterable, List, Optional


def merge_shards(shards: Iterable[dict]) -> dict:
    """Merge ``sweep_shard`` outputs of all ranks into the enumerateVerdict
    result (reference src/oracle.cpp:883-889 discovery order)."""
    configs: List[dict] = []
    total = 0
    for sh in shards:
        total = max(total, sh.get("total", 0))
        configs.extend(sh["configs"])
    configs.sort(key=lambda c: c["index"])
    seen = set()
    races = []
    for c in configs:
        ws = c["warpSize"]
        for r in c["races"]:  # each config's races are already sorted (:76)
            key = (r["locA"]["line"], r["locA"]["column"], r["locB"]["line"],
                   r["locB"]["column"], r["kind"], ws)
            if key in seen:
                continue
            seen.add(key)
            races.append({"kind": r["kind"], "locA": r["locA"], "locB": r["locB"],
                          "warpSize": ws})
    return {"races": races, "configs": total}


def enumerate_verdict_distributed(run_shard: Callable[..., dict], source: str, caps=None,
                                  file_name: str = "prog.mcu", group=None) -> dict:
    """Sweep sharded over the ranks of ``group`` (default: the world).

    ``run_shard(source, caps, file_name, rank, world)`` runs one rank's share —
    ``GpuContext.sweep_shard`` on a GPU rank.  Every rank returns the merged
    result."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return merge_shards([run_shard(source, caps, file_name, 0, 1)])
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    mine = run_shard(source, caps, file_name, rank, world)
    gathered: List[Optional[dict]] = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    return merge_shards(gathered)


def shard_jobs(jobs: List[dict], rank: int, world: int) -> List[dict]:
    """Longest-processing-time assignment of independent jobs (programs x
    configs) to ranks: heaviest first onto the currently lightest rank.
    ``jobs`` carry a ``cost`` estimate (e.g. threads x configs)."""
    loads = [0.0] * world
    owner: Dict[int, int] = {}
    order = sorted(range(len(jobs)), key=lambda i: (-jobs[i].get("cost", 1.0), i))
    for i in order:
        r = min(range(world), key=lambda q: (loads[q], q))
        owner[i] = r
        loads[r] += jobs[i].get("cost", 1.0)
    return [jobs[i] for i in range(len(jobs)) if owner[i] == rank]


__all__ = ["merge_shards", "enumerate_verdict_distributed", "shard_jobs"]

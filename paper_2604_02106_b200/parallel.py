"""Multi-GPU sharding of the race-check stage (one process per GPU).

Two shardings:

* independent jobs — sweep configs / programs — with no data-path
  collective (below), and
* one huge launch by whole-block ranges (``check_launch_sharded``): INTRA
  kinds stay rank-local; INTER-BLOCK takes one MIN / MAX reduce-scatter of
  the per-(element, site) block summaries over element ranges (NCCL over
  NVLink on GPUs), a scan of each rank's range, a MIN all-reduce of the
  per-key first-found elements (3 * locs^2 words), then the few witness
  records of the realised keys' elements are gathered.

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


# ------------------------------------------------- one launch over many GPUs
def block_ranges(n_blocks: int, world: int) -> List[tuple]:
    """Contiguous, near-equal whole-block ranges of the dense block index."""
    base, extra = divmod(n_blocks, world)
    out, b = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((b, b + n))
        b += n
    return out


EMPTY_LO = 0x7F7F7F7F  # kShardEmpty: an element / site no block of the shard reached
NO_ELEM = (1 << 64) - 1  # key without an element


def element_slices(n_elems: int, world: int) -> List[tuple]:
    """Equal element ranges of the reduce-scatter (the last ones may be
    short or empty): rank r reduces and scans elements [b, e)."""
    per = (n_elems + world - 1) // world if n_elems else 0
    return [(min(r * per, n_elems), min((r + 1) * per, n_elems)) for r in range(world)]


class TorchComm:
    """Collectives of ``check_launch_sharded`` over ``torch.distributed``.
    NCCL: the device tables are reduce-scattered (MIN / MAX) into equal
    element ranges, the per-key minima are MIN all-reduced on the device.
    gloo (CPU tests): the same results through host copies (all-reduce, then
    each rank keeps its range)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def allreduce_minmax(self, lo, hi):
        """In-place MIN / MAX all-reduce of whole tables (the all-reduce
        variant of the protocol, hgrd_gpu_shard_inter)."""
        d = self.dist
        if self.nccl:
            d.all_reduce(lo, op=d.ReduceOp.MIN, group=self.group)
            d.all_reduce(hi, op=d.ReduceOp.MAX, group=self.group)
            return
        hlo, hhi = lo.cpu(), hi.cpu()
        d.all_reduce(hlo, op=d.ReduceOp.MIN, group=self.group)
        d.all_reduce(hhi, op=d.ReduceOp.MAX, group=self.group)
        lo.copy_(hlo)
        hi.copy_(hhi)

    def reduce_scatter_minmax(self, lo, hi, unit: int):
        """lo / hi: int32 tables of n_elems * unit entries (unit = sites per
        element).  Returns this rank's reduced range (lo_r, hi_r, elem_begin,
        n_elems_r); lo_r / hi_r live on lo's device."""
        import torch
        d = self.dist
        n_elems = lo.numel() // unit
        b, e = element_slices(n_elems, self.world)[self.rank]
        per = (n_elems + self.world - 1) // self.world
        if self.nccl:
            pad = per * self.world * unit
            plo = torch.full((pad,), EMPTY_LO, dtype=torch.int32, device=lo.device)
            phi = torch.zeros(pad, dtype=torch.int32, device=lo.device)
            plo[: lo.numel()].copy_(lo)
            phi[: hi.numel()].copy_(hi)
            olo = torch.empty(per * unit, dtype=torch.int32, device=lo.device)
            ohi = torch.empty(per * unit, dtype=torch.int32, device=lo.device)
            d.reduce_scatter_tensor(olo, plo, op=d.ReduceOp.MIN, group=self.group)
            d.reduce_scatter_tensor(ohi, phi, op=d.ReduceOp.MAX, group=self.group)
            return olo[: (e - b) * unit], ohi[: (e - b) * unit], b, e - b
        hlo, hhi = lo.cpu(), hi.cpu()
        d.all_reduce(hlo, op=d.ReduceOp.MIN, group=self.group)
        d.all_reduce(hhi, op=d.ReduceOp.MAX, group=self.group)
        return (hlo[b * unit: e * unit].to(lo.device), hhi[b * unit: e * unit].to(lo.device),
                b, e - b)

    def allreduce_min_u64(self, values, device=None):
        """MIN all-reduce of a uint64 numpy vector (NO_ELEM = none)."""
        import numpy as np
        import torch
        d = self.dist
        v = values.astype(np.uint64)
        signed = np.where(v == np.uint64(NO_ELEM), np.int64(2 ** 63 - 1),
                          v.astype(np.int64))
        t = torch.from_numpy(signed)
        if self.nccl:
            t = t.to(device if device is not None else torch.cuda.current_device())
        d.all_reduce(t, op=d.ReduceOp.MIN, group=self.group)
        out = t.cpu().numpy()
        return np.where(out == np.int64(2 ** 63 - 1), np.uint64(NO_ELEM),
                        out.astype(np.uint64))

    def allgather(self, obj) -> list:
        out: List[Optional[object]] = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


def _race_key(r: dict):
    return (tuple(r["locA"]), tuple(r["locB"]), r["kind"])


def check_launch_sharded(ctx, spec, comm, device: int = 0) -> dict:
    """``ctx.check_launch(spec)`` of one launch split over the ranks of
    ``comm`` by whole-block ranges; every rank returns the same result, equal
    to the unsharded check (INTRA races merged as the lexicographic minimum
    of (element, x, y) per key — the single-GPU rule; INTER races detected on
    the gathered records of the realised keys' elements).  A launch or shard
    that needs the ordered path (traps, step budget, locks, sequential mode)
    falls back to the unsharded check on every rank."""
    from . import NotShardable
    g, b = spec.launch.grid, spec.launch.block
    n_blocks = g[0] * g[1] * g[2]
    b0, b1 = block_ranges(n_blocks, comm.world)[comm.rank]
    try:
        res, sh = ctx.shard_check(spec, b0, b1)
        stages = ctx.last_profile()  # (empty unless profiling is on)
        mine = {"ok": True, "steps": res["steps"], "instances": res["instances"],
                "records": res["records"], "mode": res["mode"], "ms": res["deviceMs"]}
    except NotShardable:
        res, sh, mine, stages = None, None, {"ok": False}, []
    import numpy as np
    # every rank shardable? (one small MIN all-reduce instead of a gather)
    if int(comm.allreduce_min_u64(np.array([1 if mine["ok"] else 0], np.uint64), device)[0]) == 0:
        out = ctx.check_launch(spec)  # replicas: the ordered path on every rank
        out["path"] = "replicas"
        return out
    if sh.inter_n:
        lo, hi = ctx.shard_tables(sh, device)
        if hasattr(comm, "reduce_scatter_minmax"):
            # reduce-scatter over element ranges, scan of this rank's range,
            # MIN all-reduce of the per-key first-found elements
            rlo, rhi, e0, ne = comm.reduce_scatter_minmax(lo, hi, spec.launch.n_sites)
            ke = ctx.shard_inter_scan(spec, rlo, rhi, e0, ne, device)
            ke = comm.allreduce_min_u64(ke, device)
            keys, vals = ctx.shard_inter_records(spec, sh, ke)
        else:
            comm.allreduce_minmax(lo, hi)
            ctx.wait_torch_stream(device)
            keys, vals = ctx.shard_inter(spec, sh)
    else:
        import numpy as np
        keys, vals = np.zeros(0, np.uint64), np.zeros(0, np.uint32)
    parts = comm.allgather({"races": res["races"], "keys": keys, "vals": vals, "stats": mine})
    stats = [p["stats"] for p in parts]
    steps = sum(s.get("steps", 0) for s in stats)
    if steps > spec.launch.step_budget:  # the budget runs out: the ordered path decides
        out = ctx.check_launch(spec)
        out["path"] = "replicas"
        return out
    best: Dict[tuple, dict] = {}
    for p in parts:  # INTRA: per key the minimum (element, x, y)
        for r in p["races"]:
            k = _race_key(r)
            o = (r["handle"], r["address"], r["threadA"], r["seqA"], r["threadB"], r["seqB"])
            if k not in best or o < best[k][0]:
                best[k] = (o, r)
    races = [v[1] for v in best.values()]
    all_keys = np.concatenate([p["keys"] for p in parts]) if parts else keys
    all_vals = np.concatenate([p["vals"] for p in parts]) if parts else vals
    if len(all_keys):
        races += ctx.shard_detect(spec, all_keys, all_vals)["races"]
    kinds = ["INTER-BLOCK", "INTRA-BLOCK", "INTRA-WARP"]
    races.sort(key=lambda d: (d["locA"], d["locB"], kinds.index(d["kind"])))
    return {"races": races, "traps": [], "steps": steps,
            "instances": sum(s["instances"] for s in stats),
            "records": sum(s["records"] for s in stats), "aborted": False, "abortStmt": -1,
            "mode": stats[0]["mode"], "deviceMs": max(s["ms"] for s in stats),
            "path": "sharded", "interRecords": int(len(all_keys)), "stages": stages}


__all__ = ["merge_shards", "enumerate_verdict_distributed", "shard_jobs", "block_ranges",
           "element_slices", "TorchComm", "check_launch_sharded"]

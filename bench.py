#!/usr/bin/env python
"""Race-check throughput on B200: access instances race-checked per second.

Default workload: BASELINE.json configs[3], the largest config that fits one
GPU — the global-memory histogram with data-dependent bins, 2^27 MiniCU
threads (2^28 access instances per launch), 2^16 bins; one step checks the
three update variants of SURVEY.md §8(d) row 4 (atomicAdd / atomicAdd_block /
store) over the same 1 GiB data array.  --workload selects the other configs
(stencil = configs[1], transpose = configs[2], permutation / histogram_2p24 =
configs[3] variants, corpus = configs[0] and lattice = configs[4] sweeps).

* ``value``: instances / device time of hgrd_gpu_check_launch (CUDA events on
  the context's stream) with the inputs resident in HBM; L2 flushed (256 MiB
  write) between steps (the data arrays exceed L2 too).
* ``e2e``: the same checks through the C ABI with HOST buffers: every step
  copies the host's input arrays from pinned memory (hgrd_gpu_buffer_write),
  checks and reads the reports back (workloads without host data go through
  hgrd_gpu_run_concrete_json: source text in, JSON out); wall clock.
* ``roofline``: the dominant kernel vs the measured HBM copy bandwidth, with
  SURVEY.md §8(d)'s algorithmic bytes (32 B per instance, +8 B per value-
  consumed load: 36 B for the histogram) x the instances of one launch.
* ``cpu_baseline``: the unmodified reference (oracle/_ref/libhgrd_ref.so,
  hgrd::runConcrete) on every host thread on a bounded sample.

--impl reference times that reference CPU implementation alone (rank 0).
--gpus N under torchrun: every rank checks its own independent launches (own
data, no data-path collective: weak scaling); --shard-launch instead splits
ONE launch of N x the per-GPU threads by whole-block ranges (INTER-BLOCK via
an NCCL reduce-scatter, parallel.check_launch_sharded).  The sweep workloads
shard their configurations by canonical index (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import programs  # noqa: E402

METRIC = "access instances race-checked/sec"
UNIT = "instances/s"


# ----------------------------------------------------------------- workloads
class Workload:
    """One BASELINE.json config as bench steps: `launches` are checked once
    per step (every variant of the config); `b_alg` is SURVEY.md §8(d)'s
    algorithmic bytes per instance; `cpu_sample` gives the reference CPU
    sample (sources with the launch, and the same host code without it so the
    host-side init loop can be subtracted)."""

    name = ""
    config_index = 0
    b_alg = 32
    shardable = False
    e2e_api = "hgrd_gpu_buffer_write + hgrd_gpu_check_launch"

    def variants(self):
        raise NotImplementedError


def _no_launch(src: str) -> str:
    """The same program without its kernel launch (host work only)."""
    lines = src.splitlines(keepends=True)
    out = []
    for ln in lines:
        if "<<<" in ln:
            head, tail = ln.split("<<<", 1)
            name = head.split()[-1]
            head = head[: len(head) - len(name)]
            ln = head + tail.split(";", 1)[1]
        out.append(ln)
    return "".join(out)


class Histogram(Workload):
    """configs[3]: global-memory histogram with data-dependent bins, 2^27
    MiniCU threads (2^28 instances per launch: the indexed load of data[t]
    and one update), bins 2^16 (hot, 2048 threads per bin) or 2^24; one
    step checks the three update variants of SURVEY §8(d) row 4 — (i)
    atomicAdd (clean), (ii) atomicAdd_block (INTER-BLOCK), (iii) store
    (every kind the collisions allow) — over the same 1 GiB data array."""

    config_index = 3
    b_alg = 36  # 32 B per instance + 8 B per value-consumed load (1 per 2 instances)
    updates = ("atomic", "atomic_block", "store")

    shardable = True  # --shard-launch: one launch of N x n threads, whole-block ranges per rank

    def __init__(self, n=1 << 27, bins=1 << 16):
        self.n, self.bins = n, bins
        self.name = (f"histogram_2^{n.bit_length() - 1}threads_2^{bins.bit_length() - 1}bins_"
                     f"block256_ws32_atomic+atomic_block+store")
        self.inst_per_launch = 2 * n
        self.world, self.rank = 1, 0
        self.seed = programs.HIST_SEED

    def independent(self, rank):
        """--gpus N (default): rank r checks its own launches over its own
        data (seed + r), independent units with no data-path collective."""
        self.seed = programs.HIST_SEED + rank

    def shard(self, world, rank):
        """Weak scaling: the launch grows to world x n threads; this rank
        checks (and supplies the data of) its n threads' whole blocks."""
        self.world, self.rank = world, rank
        self.name = self.name.replace(f"2^{self.n.bit_length() - 1}threads",
                                      f"{world}x2^{self.n.bit_length() - 1}threads")
        self.inst_per_launch = 2 * self.n * world

    def program(self, n, upd, host_init):
        return programs.histogram(n, self.bins, upd, host_init=host_init, seed=self.seed)

    def data(self, n, lo=0, hi=None):
        """data[lo:hi] of an n-thread launch."""
        import numpy as np
        i = np.arange(lo, n if hi is None else hi, dtype=np.int64)
        return (i * programs.HIST_MULT + self.seed) % self.bins

    def expected(self, upd):
        if self.bins & (self.bins - 1) == 0 and self.bins >= 256:
            return programs.histogram_pow2_expected(self.n * self.world, self.bins, upd,
                                                    self.seed)
        return None

    def table(self):
        return self.bins

    def build(self, hg, ctx, pinned):
        n = self.n * self.world
        lo = self.rank * self.n
        data_h = ctx.alloc(n)
        table_h = ctx.alloc(self.table())
        host = pinned(self.data(n, lo, lo + self.n))
        ctx.write(data_h, host, lo)  # (the other ranks' blocks never read this rank's range)
        out = []
        for upd in self.updates:
            low = hg.lower(self.program(n, upd, False), "h")
            spec = hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), 32,
                                 handles={"data": data_h, "hist": table_h})
            out.append((upd, spec))
        self.inputs = [(data_h, host, lo)]
        return out

    def check(self, upd, res):
        want = self.expected(upd)
        if want is not None:
            got = [(r["kind"], r["address"], r["threadA"], r["threadB"]) for r in res["races"]]
            assert got == want, (upd, got, want)
        assert res["instances"] == self.inst_per_launch, res["instances"]

    def cpu_sample(self, sample_n):
        return [(self.program(sample_n, u, True), _no_launch(self.program(sample_n, u, True)),
                 2 * sample_n) for u in self.updates]


class Permutation(Histogram):
    """configs[3] permutation-scatter variant: B = n = 2^27 bins, every bin
    hit once except the injected duplicates (programs.PERM_DUPS)."""

    updates = ("store", "atomic_block")

    def independent(self, rank):
        pass  # (one fixed permutation: every rank checks the same launches)
    shardable = False  # (the permutation spans the whole launch: replicas)

    def __init__(self, n=1 << 27):
        self.n = n
        self.name = f"permutation_scatter_2^{n.bit_length() - 1}threads_block256_ws32_store+atomic_block"
        self.inst_per_launch = 2 * n
        self.world, self.rank = 1, 0

    def program(self, n, upd, host_init):
        return programs.permutation_scatter(n, upd, host_init=host_init)

    def data(self, n, lo=0, hi=None):
        return programs.permutation_data(n)[lo:hi]

    def expected(self, upd):
        return programs.permutation_expected(self.n, upd)

    def table(self):
        return self.n


class ZeroInit(Workload):
    """Workloads whose buffers are all zero-initialised by cudaMalloc (the
    host supplies no data): e2e goes through hgrd_gpu_run_concrete_json,
    MiniCU source in, JSON report out."""

    e2e_api = "hgrd_gpu_run_concrete_json"
    inputs = []
    shardable = False

    def check(self, var, res):
        want = self.expect[var]
        got = sorted(r["kind"] for r in res["races"])
        assert got == want, (var, got, want)
        assert res["instances"] == self.inst_per_launch, res["instances"]


class Stencil(ZeroInit):
    """configs[1]: 1D stencil with a per-block tile, 2^20 threads, block 256,
    warp 32; missing-barrier and fixed variants."""

    config_index = 1
    expect = {"missing": ["INTRA-BLOCK", "INTRA-BLOCK", "INTRA-WARP", "INTRA-WARP"], "fixed": []}

    def __init__(self, n=1 << 20):
        self.n = n
        self.name = f"stencil1d_2^{n.bit_length() - 1}threads_block256_ws32_missing+fixed"
        self.inst_per_launch = 5 * n

    def source(self, n, var):
        return programs.stencil(n, 256, var == "fixed")

    def build(self, hg, ctx, pinned):
        n, out = self.n, []
        for var in ("missing", "fixed"):
            low = hg.lower(self.source(n, var), "st")
            h = {"in_": ctx.alloc(n), "tile": ctx.alloc(n // 256 * 258), "out_": ctx.alloc(n)}
            out.append((var, hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), 32, handles=h)))
        return out

    def cpu_sample(self, sample_n):
        return [(self.source(sample_n, v), None, 5 * sample_n) for v in ("missing", "fixed")]


class Transpose(ZeroInit):
    """configs[2]: tiled n x n transpose through a padded 32x33 tile per
    block, n = 8192: 2^26 instances per barrier interval, 3 * 2^26 per
    launch; missing-barrier and fixed variants."""

    config_index = 2
    expect = {"missing": ["INTRA-BLOCK"], "fixed": []}

    def __init__(self, n=8192):
        self.n = n
        self.name = f"transpose_{n}x{n}_block32x32_ws32_missing+fixed"
        self.inst_per_launch = 3 * n * n

    def source(self, n, var):
        return programs.transpose(n, var == "fixed")

    def build(self, hg, ctx, pinned):
        n, out = self.n, []
        for var in ("missing", "fixed"):
            low = hg.lower(self.source(n, var), "tr")
            ntile = (n // 32) * (n // 32) * 1056
            h = {"tile": ctx.alloc(ntile), "out_": ctx.alloc(n * n)}
            out.append((var, hg.LaunchSpec(low, (n // 32, n // 32, 1), (32, 32, 1), 32,
                                           scalars={"n": n}, handles=h)))
        return out

    def cpu_sample(self, sample_n):
        side = int(round(sample_n ** 0.5))
        return [(self.source(side, v), None, 3 * side * side) for v in ("missing", "fixed")]


WORKLOADS = {
    "histogram": lambda: Histogram(),
    "histogram_2p24": lambda: Histogram(bins=1 << 24),
    "permutation": lambda: Permutation(),
    "transpose": lambda: Transpose(),
    "stencil": lambda: Stencil(),
}
# reference CPU sample per host thread (MiniCU threads per launch)
CPU_SAMPLE = {"histogram": 1 << 18, "histogram_2p24": 1 << 18, "permutation": 1 << 18,
              "transpose": 1 << 18, "stencil": 1 << 16}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def init_dist(local):
    """NCCL process group (torchrun's env://; HGRD_BENCH_DIST=1 alone: a
    single-rank group on this GPU, to exercise the multi-rank code path)."""
    import torch
    import torch.distributed as dist
    if "RANK" not in os.environ:
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (clock / throttle record)."""

    def __init__(self, index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


def reference_rate(wl, threads: int, reps: int, sample: int):
    """The unmodified reference runConcrete, `threads` host threads at once,
    each running every variant of the workload at `sample` MiniCU threads;
    the host-only run of the same program (init loop, no launch) is timed
    the same way and subtracted, so the rate is the race-check stage's."""
    from oracles import RefOracle, REF_LIB, CpuOracle, ORACLE_LIB
    cfg = programs.synthetic_config()
    if os.path.exists(REF_LIB):
        ref, kind = RefOracle(), "reference"

        def run(src):
            return ref.time_parallel(src, cfg, threads, reps, "syn.mcu")[0]
    else:
        ora, kind = CpuOracle(ORACLE_LIB), "port"
        threads = 1

        def run(src):
            t0 = time.perf_counter()
            for _ in range(reps):
                ora.run_concrete(src, cfg, "syn.mcu")
            return time.perf_counter() - t0
    secs = host_secs = 0.0
    inst = 0
    for src, host_only, n_inst in wl.cpu_sample(sample):
        secs += run(src)
        if host_only is not None:
            host_secs += run(host_only)
        inst += threads * reps * n_inst
    return inst / max(secs - host_secs, 1e-9), kind, threads, secs, host_secs, inst


def _sample_text(wl, threads, reps, sample, inst, secs, host_secs):
    t = (f"{threads} host threads x {reps} reps x {len(wl.cpu_sample(sample))} variants of "
         f"{wl.name.split('_')[0]} at {sample} MiniCU threads per launch "
         f"({inst} instances, {secs:.1f} s")
    if host_secs:
        t += f", minus {host_secs:.1f} s of the same host init without the launch"
    return t + "; hgrd::runConcrete, caps raised)"


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]()
    sample = CPU_SAMPLE[args.workload]
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        reference_rate(wl, threads, 1, sample // 4)
    tot_inst, tot_secs, tot_host = 0, 0.0, 0.0
    kind = "reference"
    for _ in range(args.steps):
        _, kind, threads, secs, host_secs, inst = reference_rate(wl, threads, 1, sample)
        tot_inst += inst
        tot_secs += secs
        tot_host += host_secs
    v = tot_inst / (tot_secs - tot_host)
    sample_txt = _sample_text(wl, threads, 1, sample, tot_inst // args.steps,
                              tot_secs / args.steps, tot_host / args.steps) + " per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * (tot_secs - tot_host) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": wl.name, "baseline_config": wl.config_index,
                   "sample_threads_per_launch": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample_txt},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_gpu_arm(args):
    import torch
    import paper_2604_02106_b200 as hg

    ws, rank, local = dist_env()
    # (HGRD_BENCH_DIST=1: the multi-rank code path at world size 1, for testing)
    use_dist = ws > 1 or os.environ.get("HGRD_BENCH_DIST") == "1"
    if use_dist:
        init_dist(local)
    dev = torch.device("cuda", local)
    ctx = hg.GpuContext(local)
    ctx.set_profiling(True)
    wl = WORKLOADS[args.workload]()
    # --gpus N on a shardable workload: ONE launch of N x the per-GPU threads,
    # whole-block ranges per rank (INTRA kinds rank-local; INTER-BLOCK through
    # an NCCL reduce-scatter of the block summaries, parallel.py); otherwise
    # every rank checks its own replica of the workload
    sharded = use_dist and wl.shardable and args.shard_launch
    if sharded:
        from paper_2604_02106_b200.parallel import TorchComm, check_launch_sharded
        wl.shard(ws, rank)
        comm = TorchComm()
    elif use_dist and hasattr(wl, "independent"):
        wl.independent(rank)

    def pinned(a):
        t = torch.empty(a.size, dtype=torch.int64, pin_memory=True).numpy()
        t[:] = a
        return t

    launches = wl.build(hg, ctx, pinned)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    ext = torch.cuda.ExternalStream(ctx.stream(), device=dev)  # the context's stream

    def check(spec):
        if sharded:
            res = check_launch_sharded(ctx, spec, comm, device=local)
            return res, res["stages"]
        res = ctx.check_launch(spec)
        return res, ctx.last_profile()

    def step():
        out = []
        for var, spec in launches:
            res, prof = check(spec)
            out.append((var, res, prof))
        return out

    for _ in range(max(args.warmup, 3)):
        step()
    # correctness guard: the report must be the known one (tests pin it to the reference)
    ablate = bool(os.environ.get("HGRD_FUSED_ABLATE"))  # profiling ablations change reports
    if not ablate:
        for var, res, _ in step():
            wl.check(var, res)

    def barrier():
        if use_dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # clocks: sample across a >= 1 s run of the same steps right before the
    # timed region and through it
    clocks = Clocks(local)
    t_probe = time.perf_counter()
    while time.perf_counter() - t_probe < 1.0:
        step()
    launches0 = ctx.kernel_launches()
    barrier()
    dev_ms = 0.0
    stage_ms, stage_n = {}, {}
    inst = 0
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between steps (the data arrays exceed L2 as well)
        torch.cuda.synchronize()
        if sharded:  # the step spans collectives: events on the context's stream around it
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(ext)
        results = step()
        if sharded:
            ev1.record(ext)
            ev1.synchronize()
            dev_ms += ev0.elapsed_time(ev1)
        for var, res, prof in results:
            if not sharded:
                dev_ms += res["deviceMs"]
            inst += res["instances"]
            for s in prof:
                stage_ms[s["name"]] = stage_ms.get(s["name"], 0.0) + s["ms"]
                stage_n[s["name"]] = stage_n.get(s["name"], 0) + 1
    barrier()
    wall = time.perf_counter() - wall0
    n_launch = ctx.kernel_launches() - launches0
    clk = clocks.stop()

    # e2e through the C ABI with HOST buffers: every step copies the host's
    # input arrays (pinned) into the context's buffers (hgrd_gpu_buffer_write),
    # checks every variant and reads the reports back; workloads without
    # host data go through hgrd_gpu_run_concrete_json (source in, JSON out).
    cfg = programs.synthetic_config()

    def e2e_step():
        if wl.e2e_api.startswith("hgrd_gpu_run_concrete"):
            return [(var, ctx.run_concrete(wl.source(wl.n, var), cfg, "syn.mcu"))
                    for var, _ in launches]
        for h, host, off in wl.inputs:
            ctx.write(h, host, off)
        return [(var, check(spec)[0]) for var, spec in launches]

    e2e_step()  # warm (allocation arena, NVRTC cache)
    barrier()
    xfer0 = ctx.transfer_bytes()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        got = e2e_step()
    barrier()
    e2e_s = time.perf_counter() - t0
    xfer1 = ctx.transfer_bytes()
    h2d = (xfer1[0] - xfer0[0]) // max(args.steps, 1)
    d2h = (xfer1[1] - xfer0[1]) // max(args.steps, 1)
    e2e_serial_s = None
    if wl.inputs and not wl.e2e_api.startswith("hgrd_gpu_run_concrete"):
        # pipelined e2e: a second buffer set; step k+1's inputs upload on the
        # context's copy stream (hgrd_gpu_buffer_write_async) while step k is
        # checked. Every step still copies its whole input from pinned host
        # memory and reads its reports back inside the timed region.
        inputs_a = wl.inputs
        launches_b = wl.build(hg, ctx, pinned)
        sets = [(launches, inputs_a), (launches_b, wl.inputs)]
        wl.inputs = inputs_a

        def upload(k):
            for h, host, off in sets[k % 2][1]:
                ctx.write_async(h, host, off)

        def run_pipelined(steps):
            upload(0)
            res = None
            for k in range(steps):
                if k + 1 < steps:
                    upload(k + 1)
                res = [(var, check(spec)[0]) for var, spec in sets[k % 2][0]]
            return res

        run_pipelined(2)  # warm
        barrier()
        xfer0 = ctx.transfer_bytes()
        t0 = time.perf_counter()
        got = run_pipelined(args.steps)
        barrier()
        e2e_serial_s, e2e_s = e2e_s, time.perf_counter() - t0
        xfer1 = ctx.transfer_bytes()
        assert (xfer1[0] - xfer0[0]) // max(args.steps, 1) == h2d
        wl.e2e_api = ("hgrd_gpu_buffer_write_async (step k+1's inputs, two buffer sets) + "
                      "hgrd_gpu_check_launch")
    if not ablate:
        for var, res in got:
            if "stats" in res:
                assert sorted(r["kind"] for r in res["races"]) == wl.expect[var]
            else:
                wl.check(var, res)

    if use_dist:
        t = torch.tensor([dev_ms, e2e_s, e2e_serial_s or 0.0], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, e2e_s = float(t[0]), float(t[1])
        e2e_serial_s = float(t[2]) or None
    total_inst = inst if sharded else inst * ws  # (a sharded report counts every rank's)
    value = total_inst / (dev_ms / 1e3)
    e2e_value = total_inst / e2e_s

    peak, peak_kind = peaks()
    if not stage_ms:  # (no per-stage profile: the whole check as one stage)
        stage_ms, stage_n = {"check": dev_ms}, {"check": args.steps * len(launches)}
    dom = max(stage_ms, key=stage_ms.get)
    dom_avg_ms = stage_ms[dom] / stage_n[dom]
    # algorithmic bytes per launch of the dominant kernel: B_alg x instances
    # of one launch (it runs once per check)
    # (sharded: one rank's kernel processes its share of the launch)
    kernel_inst = wl.inst_per_launch // (ws if sharded else 1)
    achieved = wl.b_alg * kernel_inst / (dom_avg_ms / 1e3) / 1e9
    traffic, traffic_src = None, None  # DRAM bytes per launch, from a committed ncu capture
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath)).get(args.workload)
        if isinstance(tr, dict) and dom in tr:
            traffic, traffic_src = tr[dom], tr.get("source")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": wl.name, "baseline_config": wl.config_index,
                   "instances_per_launch": wl.inst_per_launch,
                   "launches_per_step": len(launches),
                   "instances_per_step": wl.inst_per_launch * len(launches),
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": (f"blockshard{ws}" if sharded else
                                   f"independent-launches{ws}" if use_dist else "1")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": wl.e2e_api,
                **({"serial_value": total_inst / e2e_serial_s,
                    "serial_api": "hgrd_gpu_buffer_write + hgrd_gpu_check_launch"}
                   if e2e_serial_s else {})},
        "gpu_launches": n_launch,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     **({"traffic_unit": "DRAM bytes per launch (ncu)",
                         "traffic_source": traffic_src,
                         "alg_bytes_per_launch": wl.inst_per_launch * wl.b_alg}
                        if traffic is not None else {}),
                     "kernel": dom,
                     "kernel_avg_ms": dom_avg_ms, "b_alg_per_instance": wl.b_alg,
                     "peak_source": peak_kind,
                     "stage_share": {k: v / sum(stage_ms.values()) for k, v in stage_ms.items()}},
        "clocks": clk,
        "wall_s": wall,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = CPU_SAMPLE[args.workload]
        v, kind, threads, secs, host_secs, n = reference_rate(wl, threads, 1, sample)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                                "sample": _sample_text(wl, threads, 1, sample, n, secs,
                                                       host_secs)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if use_dist:
        torch.distributed.destroy_process_group()


def run_paths(args):
    """--paths: the other GPU paths against the unmodified reference
    (hgrd::runConcrete / enumerateVerdict from oracle/_ref) on side
    workloads, one JSON line each (device wall clock through the public
    API; reports compared field by field).  Opt-in: the reference needs
    ~40 s of host time here."""
    import paper_2604_02106_b200 as hg
    from conftest import load_golden
    from oracles import RefOracle, REF_LIB, strip_extras
    if not os.path.exists(REF_LIB):
        print(json.dumps({"paths": "unavailable", "why": f"{REF_LIB} not built"}))
        return
    ctx, ref = hg.GpuContext(0), RefOracle()
    cfg = programs.synthetic_config()

    def timed(fn, reps):
        fn()  # warm (NVRTC cache, arena)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3, out

    n = 1 << 16
    for name, src, mode in (
            (f"locks_{n}threads", programs.lock_kernel(n, "leak"), "PARALLEL + pairwise lockInfo"),
            (f"sequential_chain_{n}threads", programs.chain_kernel(n, n + 1),
             "SEQUENTIAL (canonical order, NVRTC body)")):
        g_ms, g = timed(lambda: ctx.run_concrete(src, cfg, "paths.mcu"), 3)
        t0 = time.perf_counter()
        r = ref.run_concrete(src, cfg, "paths.mcu")
        r_ms = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"workload": name, "mode": mode, "gpu_ms": g_ms, "reference_ms": r_ms,
                          "reference_threads": 1,
                          "same_report": strip_extras(g) == strip_extras(r),
                          "instances": g["stats"]["instances"], "races": len(g["races"])}),
              flush=True)
    corpus = load_golden("corpus")
    sweep = lambda: [ctx.enumerate_verdict(e["source"], e["caps"], e["file"])  # noqa: E731
                     for e in corpus]
    g_ms, g = timed(sweep, 3)
    t0 = time.perf_counter()
    r = [ref.enumerate_verdict(e["source"], e["caps"], e["file"]) for e in corpus]
    r_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"workload": "corpus_sweep_29_entries_manifest_caps",
                      "mode": "enumerateVerdict, 8 worker contexts", "gpu_ms": g_ms,
                      "reference_ms": r_ms, "reference_threads": 1,
                      "same_report": [strip_extras(x) for x in g] == [strip_extras(x) for x in r]}),
          flush=True)
    # config 5: the launch-config sweep -- every corpus program over a
    # 10-value input set plus the reference's 200 soundness-fuzz programs
    # (tests/test_soundness.cpp:80-84), warp sizes {2,4,8,16,32}
    jobs = sweep_jobs(corpus, load_golden("fuzz"))
    n_cfg = sum(j["configs"] for j in jobs)
    sweep = lambda: [ctx.enumerate_verdict(j["source"], j["caps"], j["file"])  # noqa: E731
                     for j in jobs]
    g_ms, g = timed(sweep, 3)
    t0 = time.perf_counter()
    r = [ref.enumerate_verdict(j["source"], j["caps"], j["file"]) for j in jobs]
    r_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"workload": f"config5_sweep_{len(jobs)}programs_{n_cfg}configs",
                      "mode": "enumerateVerdict, 8 worker contexts", "gpu_ms": g_ms,
                      "reference_ms": r_ms, "reference_threads": 1,
                      "gpu_configs_per_s": n_cfg / g_ms * 1e3,
                      "reference_configs_per_s": n_cfg / r_ms * 1e3,
                      "same_report": [strip_extras(x) for x in g] == [strip_extras(x) for x in r]}),
          flush=True)
    ctx.close()


SWEEP_INPUTS = [-1, 0, 1, 2, 3, 4, 7, 16, 127, 255]
SWEEP_WARPS = [2, 4, 8, 16, 32]


def sweep_jobs(corpus, fuzz):
    """BASELINE config 5's job list: (program, SweepCaps) with the number
    of configurations each enumerates (|inputSet|^inputs x |warpSizes|)."""
    import paper_2604_02106_b200 as hg
    jobs = []
    for e in corpus:
        caps = dict(e["caps"], inputSet=SWEEP_INPUTS, warpSizes=SWEEP_WARPS)
        k = hg.count_inputs(e["source"], e["file"])
        jobs.append({"source": e["source"], "file": e["file"], "caps": caps,
                     "configs": len(SWEEP_INPUTS) ** k * len(SWEEP_WARPS)})
    for f in fuzz:
        k = hg.count_inputs(f["source"], "fuzz.mcu")
        jobs.append({"source": f["source"], "file": "fuzz.mcu",
                     "caps": {"warpSizes": SWEEP_WARPS},
                     "configs": 5 ** k * len(SWEEP_WARPS)})
    return jobs


# ------------------------------------------------------- sweep workloads
SWEEP_WORKLOADS = ("lattice", "corpus")


def sweep_job_list(name):
    """configs[4] ("lattice"): the 229-program x 10-input x 5-warp-size
    lattice (9695 configurations); configs[0] ("corpus"): the 29 corpus
    entries at their manifest SweepCaps (acceptance criterion 4).  Jobs are
    [{"source", "file", "caps"}]; the expected reports are the reference's
    (tests/golden)."""
    from conftest import load_golden
    if name == "lattice":
        gold = load_golden("lattice")
        return ([{"source": j["source"], "file": j["file"], "caps": j["caps"]} for j in gold],
                [j["sweep"] for j in gold], 4)
    gold = load_golden("corpus")
    return ([{"source": e["source"], "file": e["file"], "caps": e["caps"]} for e in gold],
            [e["sweep_manifest"] for e in gold], 0)


def sweep_instances(jobs):
    """Access instances the sweep checks (identical on every path by
    construction; counted by the CPU restatement, test infrastructure)."""
    from oracles import CpuOracle
    return sum(r["stats"]["instances"] for r in CpuOracle().enumerate_verdict_many(jobs))


def run_sweep_arm(args):
    """configs[0] / configs[4]: every job's enumerateVerdict per step through
    hgrd_gpu_enumerate_verdict_many_json (host runs speculated on host
    threads, the launches of all jobs in one batched kernel; configurations
    that cannot be speculated run exactly on worker contexts meanwhile).
    A sweep is a host-driven pipeline, so a step is timed end to end (wall
    clock around the synchronous call, max over ranks); `value` and `e2e`
    are the same measurement.  --gpus N: rank r runs the configurations with
    canonical index % N == r of every job (no data-path collective), the
    shards are gathered and merged (parallel.merge_shards)."""
    import torch
    import paper_2604_02106_b200 as hg
    from oracles import strip_extras
    from paper_2604_02106_b200.parallel import merge_shards
    ws, rank, local = dist_env()
    use_dist = ws > 1 or os.environ.get("HGRD_BENCH_DIST") == "1"
    if use_dist:
        init_dist(local)
    jobs, want, cfg_index = sweep_job_list(args.workload)
    ctx = hg.GpuContext(local)

    payload = hg.GpuContext.sweep_jobs_payload(jobs)  # the input: MiniCU sources + SweepCaps

    def step():
        """One sweep of every job; returns the report (world 1: the C ABI's
        JSON text, parsed only for checking outside the timed region)."""
        if ws == 1:
            return ctx.enumerate_verdict_many_raw(payload)
        mine = json.loads(ctx.enumerate_verdict_many_raw(payload, rank, ws))
        parts = [None] * ws
        torch.distributed.all_gather_object(parts, mine)
        return [merge_shards([p[q] for p in parts]) | {"stats": {}} for q in range(len(jobs))]

    def parsed(rep):
        return json.loads(rep) if isinstance(rep, str) else rep

    for _ in range(max(args.warmup, 3)):
        got = parsed(step())
    assert [strip_extras(g)["races"] for g in got] == [w["races"] for w in want]
    n_configs = sum(g.get("configs", 0) for g in got)
    inst = sweep_instances(jobs)
    clocks = Clocks(local)
    launches0 = ctx.kernel_launches()
    xfer0 = ctx.transfer_bytes()
    times = []
    for _ in range(args.steps):
        if use_dist:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        got = step()
        times.append(time.perf_counter() - t0)
        if os.environ.get("HGRD_SWEEP_TRACE"):
            print(f"[bench step] {1e3 * times[-1]:.2f} ms", file=sys.stderr)
    clk = clocks.stop()
    got = parsed(got)
    assert [strip_extras(g)["races"] for g in got] == [w["races"] for w in want]
    n_launch = ctx.kernel_launches() - launches0
    xfer1 = ctx.transfer_bytes()
    secs = sum(times)
    if use_dist:
        t = torch.tensor([secs], dtype=torch.float64, device=torch.device("cuda", local))
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs = float(t[0])
    value = inst * args.steps / secs
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{args.workload}_sweep_{len(jobs)}programs_{n_configs}configs",
                   "baseline_config": cfg_index, "instances_per_step": inst,
                   "configs_per_s": n_configs * args.steps / secs,
                   "timing": "wall clock around the synchronous sweep call, max over ranks",
                   "parallelism": f"configshard{ws}" if use_dist else "1 GPU + host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": (xfer1[0] - xfer0[0]) // args.steps,
                "d2h_bytes_per_step": (xfer1[1] - xfer0[1]) // args.steps,
                "api": "hgrd_gpu_enumerate_verdict_many_json (jobs JSON with the MiniCU sources "
                       "in, report JSON text out)"},
        "gpu_launches": n_launch, "clocks": clk,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracles import RefOracle
        threads = os.cpu_count() or 1
        tj = [(j["source"], j["file"], j["caps"]) for j in jobs]
        reps = 5
        t = sum(RefOracle().time_sweeps(tj, threads)[0] for _ in range(reps))
        line["cpu_baseline"] = {"value": inst * reps / t, "unit": UNIT, "cores": threads,
                                "kind": "reference",
                                "sample": f"the whole workload x {reps}: enumerateVerdict of "
                                          f"every job (parse included), jobs over {threads} "
                                          f"host threads ({t:.2f} s)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if use_dist:
        torch.distributed.destroy_process_group()


def run_sweep_reference_arm(args):
    """The unmodified reference's enumerateVerdict over the same jobs, the
    jobs spread over every host thread (re-entrant), whole workload per step."""
    from oracles import RefOracle
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    jobs, _, cfg_index = sweep_job_list(args.workload)
    tj = [(j["source"], j["file"], j["caps"]) for j in jobs]
    inst = sweep_instances(jobs)
    ref = RefOracle()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        ref.time_sweeps(tj, threads)
    secs = sum(ref.time_sweeps(tj, threads)[0] for _ in range(args.steps))
    v = inst * args.steps / secs
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}_sweep_{len(jobs)}programs",
                   "baseline_config": cfg_index},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"the whole workload per step: enumerateVerdict of every "
                                   f"job, jobs over {threads} host threads"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="histogram",
                    choices=sorted(WORKLOADS) + list(SWEEP_WORKLOADS),
                    help="BASELINE config to time (default: configs[3], the largest)")
    ap.add_argument("--shard-launch", action="store_true",
                    help="--gpus N: split ONE launch of N x the per-GPU threads by whole-block "
                         "ranges (INTER-BLOCK through NCCL reduce-scatter) instead of "
                         "independent launches per rank")
    ap.add_argument("--paths", action="store_true",
                    help="time the lock-idiom, SEQUENTIAL and sweep paths against the reference")
    args = ap.parse_args()
    if args.paths:
        run_paths(args)
    elif args.workload in SWEEP_WORKLOADS:
        (run_sweep_reference_arm if args.impl == "reference" else run_sweep_arm)(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()

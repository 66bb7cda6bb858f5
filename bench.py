#!/usr/bin/env python
"""Race-check throughput on B200: access instances race-checked per second.

Workload (BASELINE.json configs[1]): the synthetic 1D stencil with a
per-block tile, 2^20 MiniCU threads in blocks of 256, warp size 32; one step
checks BOTH variants of the config — the missing-barrier launch (4 racy keys)
and the fixed one (clean) — i.e. 2 x 5 x 2^20 = 10,485,760 instances/step.

* ``value``: instances / device time of hgrd_gpu_check_launch with the launch
  buffers already resident in HBM (CUDA events on the context's stream),
  L2 flushed (256 MiB write) between steps.
* ``e2e``: the same checks through the reference-facing entry point
  (hgrd_gpu_run_concrete_json = hgrd::runConcrete): MiniCU source text in,
  JSON race report out, wall clock; h2d/d2h bytes are the context's counted
  host<->device copies per step (launch descriptors, counters, race records).
* ``roofline``: dominant pipeline stage vs the measured HBM copy bandwidth,
  algorithmic bytes = 32 B per instance.
* ``cpu_baseline``: the unmodified reference (oracle/_ref/libhgrd_ref.so,
  hgrd::runConcrete) on this host's cores on a bounded sample.

--impl reference times that reference CPU implementation alone (rank 0).
With --gpus N under torchrun every rank checks its own replica of the
workload (weak scaling; the path has no cross-rank exchange for this config).
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

N_THREADS = 1 << 20
BLOCK = 256
WS = 32
INST_PER_THREAD = 5
B_ALG = 32  # algorithmic bytes per instance
SAMPLE_THREADS = 1 << 16  # CPU reference sample (per host thread, per step)
CPU_BASELINE_REPS = 24    # cpu_baseline leg of the GPU arm: ~10 s of reference work
METRIC = "access instances race-checked/sec"
UNIT = "instances/s"
WORKLOAD = "stencil1d_2^20threads_block256_ws32_missing+fixed"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def reference_rate(threads: int, reps: int, sample: int):
    """The unmodified reference runConcrete, `threads` host threads at once,
    each running both variants of the stencil on a `sample`-thread launch."""
    from oracles import RefOracle, REF_LIB, CpuOracle, ORACLE_LIB
    cfg = programs.synthetic_config()
    srcs = [programs.stencil(sample, barrier=b) for b in (False, True)]
    if os.path.exists(REF_LIB):
        ref, kind = RefOracle(), "reference"
        secs = 0.0
        for s in srcs:
            t, _ = ref.time_parallel(s, cfg, threads, reps, "syn.mcu")
            secs += t
    else:
        ora, kind = CpuOracle(ORACLE_LIB), "port"
        t0 = time.perf_counter()
        for _ in range(reps):
            for s in srcs:
                ora.run_concrete(s, cfg, "syn.mcu")
        secs = time.perf_counter() - t0
        threads = 1
    inst = threads * reps * len(srcs) * INST_PER_THREAD * sample
    return inst / secs, kind, threads, secs, inst


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        reference_rate(threads, 1, SAMPLE_THREADS)
    tot_inst, tot_secs = 0, 0.0
    kind = "reference"
    for _ in range(args.steps):
        _, kind, threads, secs, inst = reference_rate(threads, 1, SAMPLE_THREADS)
        tot_inst += inst
        tot_secs += secs
    v = tot_inst / tot_secs
    sample = (f"{threads} host threads x both stencil variants at {SAMPLE_THREADS} MiniCU "
              f"threads each per step (hgrd::runConcrete, caps raised)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_threads": SAMPLE_THREADS},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def build_specs(hg, ctx):
    import torch
    specs = []
    for barrier in (False, True):
        src = programs.stencil(N_THREADS, BLOCK, barrier)
        low = hg.lower(src, "st")
        sizes = {"in_": N_THREADS, "tile": N_THREADS // BLOCK * (BLOCK + 2), "out_": N_THREADS}
        handles = {k: ctx.alloc(v) for k, v in sizes.items()}
        spec = hg.LaunchSpec(low, (N_THREADS // BLOCK, 1, 1), (BLOCK, 1, 1), WS,
                             handles=handles)
        # the reference's buffers_ (zero-initialised int64), in pinned host memory
        host = {k: torch.zeros(v, dtype=torch.int64, pin_memory=True).numpy()
                for k, v in sizes.items()}
        specs.append((spec, handles, host))
    return specs


def run_gpu_arm(args):
    import torch
    import paper_2604_02106_b200 as hg

    ws, rank, local = dist_env()
    # (HGRD_BENCH_DIST=1: the multi-rank code path at world size 1, for testing)
    use_dist = ws > 1 or os.environ.get("HGRD_BENCH_DIST") == "1"
    if use_dist:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = hg.GpuContext(local)
    ctx.set_profiling(True)
    specs = build_specs(hg, ctx)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        out = []
        for spec, _, _ in specs:
            res = ctx.check_launch(spec)
            out.append((res, ctx.last_profile()))
        return out

    for _ in range(max(args.warmup, 3)):
        step()
    # correctness guard: the report must be the known one (tests pin it to the oracle)
    got = step()
    kinds = sorted(r["kind"] for r in got[0][0]["races"])
    if not os.environ.get("HGRD_FUSED_ABLATE"):  # profiling ablations change the report
        assert kinds == ["INTRA-BLOCK", "INTRA-BLOCK", "INTRA-WARP", "INTRA-WARP"], kinds
        assert not got[1][0]["races"]

    def barrier():
        if use_dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # clocks: sample across a >= 1 s run of the same steps right before the
    # timed region and through it (the timed region alone is milliseconds)
    clocks = Clocks(local)
    t_probe = time.perf_counter()
    while time.perf_counter() - t_probe < 1.0:
        step()
    launches0 = ctx.kernel_launches()
    barrier()
    dev_ms = 0.0
    stage_ms = {}
    stage_n = {}
    inst = 0
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        for res, prof in step():
            dev_ms += res["deviceMs"]
            inst += res["instances"]
            for s in prof:
                stage_ms[s["name"]] = stage_ms.get(s["name"], 0.0) + s["ms"]
                stage_n[s["name"]] = stage_n.get(s["name"], 0) + 1
    barrier()
    wall = time.perf_counter() - wall0
    launches = ctx.kernel_launches() - launches0
    clk = clocks.stop()

    # e2e: the reference-facing call (hgrd::runConcrete, src/oracle.cpp:378):
    # MiniCU source text in, JSON race report out — front end, host
    # interpretation of main(), zero-initialised cudaMalloc buffers, the
    # launch descriptor upload, the check and the report read-back, wall clock.
    sources = [programs.stencil(N_THREADS, BLOCK, b) for b in (False, True)]
    cfg = programs.synthetic_config()  # same ExecConfig as the reference arm
    for src in sources:  # warm (allocation arena, NVRTC cache)
        ctx.run_concrete(src, cfg, "syn.mcu")
    barrier()
    xfer0 = ctx.transfer_bytes()
    t0 = time.perf_counter()
    e2e_races = []
    for _ in range(args.steps):
        e2e_races = [ctx.run_concrete(src, cfg, "syn.mcu")["races"] for src in sources]
    barrier()
    e2e_s = time.perf_counter() - t0
    xfer1 = ctx.transfer_bytes()
    h2d = (xfer1[0] - xfer0[0]) // max(args.steps, 1)
    d2h = (xfer1[1] - xfer0[1]) // max(args.steps, 1)
    if not os.environ.get("HGRD_FUSED_ABLATE"):
        assert sorted(r["kind"] for r in e2e_races[0]) == kinds and not e2e_races[1]

    if use_dist:
        t = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, e2e_s = float(t[0]), float(t[1])
    total_inst = inst * ws
    value = total_inst / (dev_ms / 1e3)
    e2e_value = total_inst / e2e_s

    peak, peak_kind = peaks()
    dom = max(stage_ms, key=stage_ms.get)
    per_launch_inst = INST_PER_THREAD * N_THREADS
    dom_avg_ms = stage_ms[dom] / stage_n[dom]
    achieved = B_ALG * per_launch_inst / (dom_avg_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "threads_per_launch": N_THREADS,
                   "instances_per_step": 2 * per_launch_inst,
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"replicas{ws}"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "hgrd_gpu_run_concrete_json"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                     "kernel_avg_ms": dom_avg_ms, "peak_source": peak_kind,
                     "stage_share": {k: v / sum(stage_ms.values()) for k, v in stage_ms.items()}},
        "clocks": clk,
        "wall_s": wall,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        reps = CPU_BASELINE_REPS  # ~10 s of host work on the GPU box
        v, kind, threads, secs, n = reference_rate(threads, reps, SAMPLE_THREADS)
        line["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{threads} host threads x {reps} reps x both variants at {SAMPLE_THREADS} "
                      f"threads ({n} instances, {secs:.1f} s)"}
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--paths", action="store_true",
                    help="time the lock-idiom, SEQUENTIAL and sweep paths against the reference")
    args = ap.parse_args()
    if args.paths:
        run_paths(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()

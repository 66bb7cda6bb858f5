"""Static-verdict cross-check at scale.

The reference's static analyzer (analyzeProgram, src/report.cpp:82-211)
decides races with a DFS solver over finite domains: unknown inputs in
[-domainBound, domainBound), grid and block extents up to maxGrid / maxBlock
per axis, every (blockIdx, threadIdx) pair (src/solver.cpp:593-612).  Its
soundness claim — every race a concrete run can show is reported — is what
the reference's corpus runner checks on a handful of configurations
(src/corpus.cpp:219-236: every oracle race maps to a static race of the same
kind and line pair at the matching warp size).

This brute-forces a much larger part of the same domains on the GPU: every
corpus program swept over a wide input lattice, launch caps up to the
analyzer's own bounds and warp sizes 1..32, through the batched sweep
(hgrd_gpu_enumerate_verdict_many_json, or the CPU restatement for the CPU
test), then checks every concrete race against the static report at that
warp size.  It also reports how many static races the brute force realised.

Test infrastructure: the static verdicts come from the reference library
(oracle/_ref/libhgrd_ref.so).

    python tests/crosscheck.py [--out profiles/r02/static_crosscheck.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

# within the analyzer's default domains (constraints.hpp:19-26: inputs in
# [-1024, 1024), grid / block extents <= 64 per axis)
WIDE_INPUTS = [-2, -1, 0, 1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 255,
               1023]
WIDE_WARPS = [1, 2, 4, 8, 16, 32]
WIDE_CAPS = {"inputSet": WIDE_INPUTS, "warpSizes": WIDE_WARPS, "gridCap": [64, 64, 64],
             "blockCap": [64, 64, 64], "maxThreads": 1 << 14, "maxConfigs": 1 << 20}


def _key(r):
    return (r["kind"], r["locA"]["line"], r["locB"]["line"])


def crosscheck(sweep_many, ref, programs, caps=WIDE_CAPS):
    """sweep_many(jobs) -> per-job enumerateVerdict results (GPU or CPU);
    ref: oracles.RefOracle (the static analyzer).  Returns the report."""
    jobs = [{"source": p["source"], "file": p["file"], "caps": caps} for p in programs]
    t0 = time.perf_counter()
    sweeps = sweep_many(jobs)
    sweep_s = time.perf_counter() - t0
    out = []
    for p, sw in zip(programs, sweeps):
        static = {}  # warp size -> statically reported (kind, lineA, lineB)
        for ws in caps["warpSizes"]:
            rep = ref.analyze(p["source"], {"warpSize": ws, "hostAnalysis": True}, p["file"])
            static[ws] = {_key(x) for x in rep.get("races", [])}
        unsound, observed = [], set()
        for r in sw["races"]:
            ws, k = r["warpSize"], _key(r)
            observed.add((ws,) + k)
            if k not in static[ws]:
                unsound.append({"warpSize": ws, "kind": k[0], "lineA": k[1], "lineB": k[2]})
        reported = {(ws,) + k for ws, keys in static.items() for k in keys}
        out.append({"name": p["name"], "configs": sw.get("configs"),
                    "instances": sw.get("stats", {}).get("instances"),
                    "concrete_races": len(sw["races"]), "unsound": unsound,
                    "static_races": len(reported),
                    "static_races_realised": len(reported & observed)})
    return {"caps": caps, "sweep_seconds": sweep_s,
            "configs": sum(x["configs"] or 0 for x in out),
            "instances": sum(x["instances"] or 0 for x in out),
            "unsound_total": sum(len(x["unsound"]) for x in out),
            "static_races": sum(x["static_races"] for x in out),
            "static_races_realised": sum(x["static_races_realised"] for x in out),
            "programs": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--cpu", action="store_true", help="the CPU restatement instead of the GPU")
    args = ap.parse_args()
    from conftest import load_golden
    from oracles import CpuOracle, RefOracle
    programs = [{"name": e["name"], "source": e["source"], "file": e["file"]}
                for e in load_golden("corpus")]
    if args.cpu:
        ora = CpuOracle()
        sweep_many = ora.enumerate_verdict_many
    else:
        import paper_2604_02106_b200 as hg
        ctx = hg.GpuContext(0)
        sweep_many = ctx.enumerate_verdict_many
    rep = crosscheck(sweep_many, RefOracle(), programs)
    txt = json.dumps(rep, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    print(json.dumps({k: rep[k] for k in ("configs", "instances", "sweep_seconds",
                                          "unsound_total", "static_races",
                                          "static_races_realised")}))


if __name__ == "__main__":
    main()

"""GPU-backed `hgrd oracle`, `hgrd corpus` and a `run` subcommand.

    python -m paper_2604_02106_b200 oracle prog.mcu [--warp-size 2 4] [--input-set 0 1 2 3 127]
                                                  [--grid-cap 2 2 1] [--block-cap 4 1 1]
                                                  [--max-threads 64]
    python -m paper_2604_02106_b200 run prog.mcu [--warp-size 32] [--inputs 4 1] ...
    python -m paper_2604_02106_b200 corpus DIR

`oracle` mirrors the reference CLI (tools/hgrd.cpp:66-80, 114-137): the
enumerateVerdict sweep, printed as {"program", "races": [{kind, locA, locB,
warpSize}]} with exit status 1 when a race was observed.  `corpus` runs the
oracle half of the reference corpus runner (src/corpus.cpp:41-114,
203-216): every manifest with `oracle = racy | clean` is swept at its
`oracle_*` caps and must observe a race (racy) or none (clean).  The static
analyzer's half of that runner is not part of this build.  Everything runs
on the GPU through libhgrd_gpu.so (there is no CPU path).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import Dict, List

from . import ExecConfig, GpuContext, SweepCaps


def parse_manifest(path: str) -> Dict:
    """`key = value` lines (reference src/corpus.cpp:41-100)."""
    entry: Dict = {"path": path, "races": [], "oracle": "skip", "caps": {}}
    for raw in open(path):
        line = raw.split("#", 1)[0].strip()
        if not line or "=" not in line:
            continue
        key, value = (x.strip() for x in line.split("=", 1))
        nums = lambda: [int(x) for x in value.replace(",", " ").split()]  # noqa: E731
        if key == "race":
            entry["races"].append(value.split())
        elif key == "oracle":
            entry["oracle"] = value if value in ("racy", "clean") else "skip"
        elif key == "oracle_grid_cap":
            entry["caps"]["gridCap"] = nums()[:3]
        elif key == "oracle_block_cap":
            entry["caps"]["blockCap"] = nums()[:3]
        elif key == "oracle_inputs":
            entry["caps"]["inputSet"] = nums()
        elif key == "oracle_warp_sizes":
            entry["caps"]["warpSizes"] = nums()
        elif key == "oracle_max_threads":
            entry["caps"]["maxThreads"] = int(value)
        else:
            entry[key] = value
    return entry


def _sweep_caps(args) -> SweepCaps:
    return SweepCaps(gridCap=tuple(args.grid_cap), blockCap=tuple(args.block_cap),
                     inputSet=tuple(args.input_set), warpSizes=tuple(args.warp_size),
                     maxThreads=args.max_threads)


def cmd_oracle(args, ctx: GpuContext) -> int:
    src = open(args.file).read()
    res = ctx.enumerate_verdict(src, _sweep_caps(args), args.file)
    if "error" in res:
        print("\n".join(res["error"]), file=sys.stderr)
        return 2
    out = {"program": args.file, "races": []}
    for r in res["races"]:
        out["races"].append({"kind": r["kind"],
                             "locA": {"file": r["locA"].get("file", args.file),
                                      "line": r["locA"]["line"]},
                             "locB": {"file": r["locB"].get("file", args.file),
                                      "line": r["locB"]["line"]},
                             "warpSize": r["warpSize"]})
    print(json.dumps(out, indent=2))
    return 1 if out["races"] else 0


def cmd_run(args, ctx: GpuContext) -> int:
    src = open(args.file).read()
    cfg = ExecConfig(gridCap=tuple(args.grid_cap), blockCap=tuple(args.block_cap),
                     warpSize=args.warp_size[0], inputs=tuple(args.inputs),
                     maxThreads=args.max_threads)
    res = ctx.run_concrete(src, cfg, args.file)
    print(json.dumps(res, indent=2))
    if "error" in res:
        return 2
    return 1 if res.get("races") else 0


def run_corpus(directory: str, ctx: GpuContext) -> List[Dict]:
    rows = []
    for name in sorted(os.listdir(directory)):
        if not name.endswith(".manifest"):
            continue
        m = parse_manifest(os.path.join(directory, name))
        row = {"name": m.get("name", name[:-9]), "oracle": m["oracle"], "races": None,
               "pass": True, "why": ""}
        if m["oracle"] != "skip":
            src_path = os.path.join(directory, m.get("source", name[:-9] + ".mcu"))
            res = ctx.enumerate_verdict(open(src_path).read(), m["caps"], src_path)
            if "error" in res:
                row["pass"], row["why"] = False, "oracle: parse failed"
            else:
                row["races"] = len(res["races"])
                if m["oracle"] == "clean" and res["races"]:
                    row["pass"], row["why"] = False, "oracle observed a race in a clean program"
                if m["oracle"] == "racy" and not res["races"]:
                    row["pass"], row["why"] = False, "oracle saw no race in a racy program"
        rows.append(row)
    return rows


def cmd_corpus(args, ctx: GpuContext) -> int:
    rows = run_corpus(args.dir, ctx)
    width = max([len(r["name"]) for r in rows] + [4])
    print(f"{'name':<{width}}  oracle  races  result")
    for r in rows:
        races = "-" if r["races"] is None else str(r["races"])
        print(f"{r['name']:<{width}}  {r['oracle']:<6}  {races:>5}  "
              f"{'PASS' if r['pass'] else 'FAIL ' + r['why']}")
    bad = sum(not r["pass"] for r in rows)
    print(f"{len(rows) - bad}/{len(rows)} entries pass (oracle half; the static analyzer "
          "is not part of this build)")
    return 1 if bad else 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_02106_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("oracle", "run"):
        p = sub.add_parser(name)
        p.add_argument("file")
        p.add_argument("--max-threads", type=int, default=64)
        p.add_argument("--warp-size", type=int, nargs="+", default=[2, 4])
        p.add_argument("--input-set", type=int, nargs="+", default=[0, 1, 2, 3, 127])
        p.add_argument("--inputs", type=int, nargs="*", default=[])
        p.add_argument("--grid-cap", type=int, nargs=3, default=[2, 2, 1])
        p.add_argument("--block-cap", type=int, nargs=3, default=[4, 1, 1])
        p.add_argument("--device", type=int, default=0)
    p = sub.add_parser("corpus")
    p.add_argument("dir")
    p.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    ctx = GpuContext(args.device)
    try:
        return {"oracle": cmd_oracle, "run": cmd_run, "corpus": cmd_corpus}[args.cmd](args, ctx)
    finally:
        ctx.close()


if __name__ == "__main__":
    sys.exit(main())

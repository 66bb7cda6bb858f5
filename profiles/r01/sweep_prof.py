# Per-entry corpus sweep timing, GPU (1 and 8 worker contexts) vs the reference: python profiles/r01/sweep_prof.py
import os, sys, time, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2604_02106_b200 as hg
from conftest import load_golden
from oracles import RefOracle
corpus = load_golden("corpus")
ctx = hg.GpuContext(0); ref = RefOracle()
tot = {}
for w in ("1", "8"):
    os.environ["HGRD_SWEEP_WORKERS"] = w
    for e in corpus: ctx.enumerate_verdict(e["source"], e["caps"], e["file"])
    rows = []
    for e in corpus:
        k0 = ctx.kernel_launches()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); ctx.enumerate_verdict(e["source"], e["caps"], e["file"]); ts.append(time.perf_counter() - t0)
        k = (ctx.kernel_launches() - k0) // 3
        t0 = time.perf_counter(); ref.enumerate_verdict(e["source"], e["caps"], e["file"]); rt = time.perf_counter() - t0
        rows.append((e["file"], k, statistics.median(ts) * 1e3, rt * 1e3))
    print("workers", w, "total gpu ms %.2f ref ms %.2f launches %d" % (sum(r[2] for r in rows), sum(r[3] for r in rows), sum(r[1] for r in rows)))
    for r in rows: print("  %-40s launches %5d gpu %.3f ms ref %.3f ms" % r)

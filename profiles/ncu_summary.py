"""Summarise an ncu --set full report (raw metrics, stall shares, hottest
CUDA source lines) as JSON: python profiles/ncu_summary.py REPORT.ncu-rep."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:80]}
        for key in KEYS:
            if key in d:
                k[key] = f"{d[key]} {u.get(key, '')}".strip()
        st = {}
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith(
                    "not_issued"):
                try:
                    st[key.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(
                        v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        k["stall_share_pct"] = {n: round(100 * v / tot, 1)
                                for n, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        out.append(k)
    # hottest CUDA source lines (stall samples), first kernel
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv",
                                          "--print-source", "cuda,sass"))))
    agg, cur, line = {}, "", None
    for r in src:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0].isdigit():
            line = (cur, int(r[0]), r[1].strip()[:70])
        elif len(r) > 4 and r[0] == "" and r[2].startswith("0x") and line:
            try:
                agg[line] = agg.get(line, 0) + int(r[4] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    hot = [{"file": f, "line": ln, "source": s, "stall_pct": round(100 * v / tot, 1)}
           for (f, ln, s), v in sorted(agg.items(), key=lambda x: -x[1])[:15]]
    json.dump({"report": rep, "kernels": out, "hot_source_lines": hot}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])

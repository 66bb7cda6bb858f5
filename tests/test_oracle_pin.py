"""Pin the CPU restatement (oracle/cpu_oracle.cpp behind the shared host
front end) to the reference's own outputs: every golden fixture recorded
from the unmodified reference (tests/golden/make_golden.py) must be
reproduced field for field (races incl. array/address, traps, launch
counts, assert stop, indirect-indexing flag, launch records incl.
defValues).  Runs on CPU."""
import pytest

from conftest import load_golden
from oracles import strip_extras


def test_corpus_runs(cpu_oracle):
    n = 0
    for e in load_golden("corpus"):
        for run in e["runs"]:
            got = strip_extras(cpu_oracle.run_concrete(e["source"], run["config"], e["file"]))
            assert got == run["result"], (e["name"], run["config"])
            n += 1
    assert n == 29 * 22


def test_corpus_sweeps(cpu_oracle):
    racy = 0
    for e in load_golden("corpus"):
        got = strip_extras(cpu_oracle.enumerate_verdict(e["source"], e["caps"], e["file"]))
        assert got == e["sweep_manifest"], e["name"]
        got = strip_extras(cpu_oracle.enumerate_verdict(e["source"], {}, e["file"]))
        assert got == e["sweep_default"], e["name"]
        # manifest verdicts (reference corpus.cpp:213-216)
        if e["oracle"] == "clean":
            assert not e["sweep_manifest"]["races"], e["name"]
        elif e["oracle"] == "racy":
            assert e["sweep_manifest"]["races"], e["name"]
            racy += 1
    assert racy == 14


def test_unit_cases(cpu_oracle):
    for c in load_golden("unit_cases"):
        got = strip_extras(cpu_oracle.run_concrete(c["source"], c["config"], "oracle.mcu"))
        assert got == c["result"], (c["name"], c["config"])


def test_unit_case_known_answers():
    """The reference test_oracle.cpp assertions themselves, on the goldens."""
    by = {}
    for c in load_golden("unit_cases"):
        by.setdefault(c["name"], []).append(c)
    tri = [c for c in by["triangle"] if c["config"]["inputs"] == [4, 1]][0]["result"]
    assert any(r["kind"] == "INTER-BLOCK" and r["locA"]["line"] == 5 and r["locB"]["line"] == 5
               for r in tri["races"])  # :53-64
    for c in by["triangle"]:
        if c["config"]["inputs"][0] == c["config"]["inputs"][1]:
            assert not c["result"]["races"]  # :66-72
    assert not by["barrier_phases"][0]["result"]["races"]  # :74-93
    assert by["no_barrier"][0]["result"]["races"]
    assert not by["device_locks"][0]["result"]["races"]  # :95-108
    kinds = {r["kind"] for r in by["block_locks"][0]["result"]["races"]}
    assert kinds == {"INTER-BLOCK"}  # :110-129
    assert not by["handoff"][0]["result"]["races"]  # :131-147
    ws2 = [c for c in by["kind_by_warp"] if c["config"]["warpSize"] == 2][0]["result"]
    ws4 = [c for c in by["kind_by_warp"] if c["config"]["warpSize"] == 4][0]["result"]
    assert any(r["kind"] == "INTRA-BLOCK" for r in ws2["races"])  # :149-166
    assert all(r["kind"] == "INTRA-WARP" for r in ws4["races"])
    stop = [c for c in by["assert_stop"] if c["config"]["inputs"] == [5]][0]["result"]
    assert stop["assertStopped"] and stop["launchesRun"] == 0 and not stop["races"]  # :181-194
    assert by["oob_trap"][0]["result"]["traps"] and not by["oob_trap"][0]["result"]["races"]
    skip = by["cap_skip"][0]["result"]
    assert skip["launchesRun"] == 0 and skip["launchesSkipped"] == 1  # :205-212


def test_fuzz(cpu_oracle):
    total = 0
    for f in load_golden("fuzz"):
        got = strip_extras(cpu_oracle.enumerate_verdict(f["source"], {}, "fuzz.mcu"))
        assert got == f["sweep"], f["index"]
        total += len(f["sweep"]["races"])
        for run in f["runs"]:
            got = strip_extras(cpu_oracle.run_concrete(f["source"], run["config"], "fuzz.mcu"))
            assert got == run["result"], (f["index"], run["config"])
    assert total > 500  # reference test_soundness.cpp:106


def test_edge_programs(cpu_oracle):
    for c in load_golden("edge"):
        got = strip_extras(cpu_oracle.run_concrete(c["source"], c["config"], "edge.mcu"))
        assert got == c["result"], (c["name"], c["config"])


def test_synthetic_small(cpu_oracle):
    for c in load_golden("synthetic"):
        got = strip_extras(cpu_oracle.run_concrete(c["source"], c["config"], "syn.mcu"))
        assert got == c["result"], (c["name"], c["config"])


def test_survey_synthetic_goldens():
    """SURVEY §8(c) synthetic goldens (stencil / transpose missing barrier)."""
    syn = {c["name"]: c["result"] for c in load_golden("synthetic")
           if c["config"]["warpSize"] == 32}
    st = {(r["kind"], r["locA"]["line"], r["locB"]["line"]) for r in
          syn["stencil_4096_missing"]["races"]}
    assert st == {("INTRA-BLOCK", 4, 5), ("INTRA-WARP", 4, 5)}
    assert not syn["stencil_4096_fixed"]["races"]
    assert not syn["transpose_128_fixed"]["races"]
    tr = {(r["kind"], r["locA"]["line"], r["locB"]["line"]) for r in
          syn["transpose_128_missing"]["races"]}
    assert tr == {("INTRA-BLOCK", 5, 6)}
    assert not syn["histogram_4096_64_atomic"]["races"]
    assert {r["kind"] for r in syn["histogram_4096_64_atomic_block"]["races"]} == {"INTER-BLOCK"}
    assert {r["kind"] for r in syn["histogram_4096_64_store"]["races"]} == {"INTER-BLOCK",
                                                                          "INTRA-BLOCK"}


def test_live_reference_crosscheck(ref_oracle, cpu_oracle):
    """Where the reference itself is built here: a few fresh configs, live."""
    import programs
    for name, src in programs.EDGE_PROGRAMS.items():
        for ws in (1, 5):
            cfg = {"warpSize": ws, "inputs": [2, 3], "gridCap": [3, 3, 3], "blockCap": [3, 3, 3],
                   "maxThreads": 200}
            assert strip_extras(cpu_oracle.run_concrete(src, cfg)) == \
                ref_oracle.run_concrete(src, cfg), (name, ws)


def test_regress_tiny_blocks(cpu_oracle):
    """Launches of more MiniCU blocks than one k_fused iteration holds."""
    for c in load_golden("regress"):
        got = cpu_oracle.run_concrete(c["source"], c["config"], "tiny.mcu")
        assert strip_extras(got) == c["result"], (c["name"], c["config"])
        assert got["witnesses"] == c["witnesses_restatement"]


def test_envelope_goldens(cpu_oracle):
    """Long threads (> 2^20 accesses) and a wide pairwise group."""
    for c in load_golden("envelope"):
        got = cpu_oracle.run_concrete(c["source"], c["config"], "env.mcu")
        assert strip_extras(got) == c["result"], c["name"]
        assert got["witnesses"] == c["witnesses_restatement"]


def test_structural_predictors_pinned():
    """programs.permutation_expected / histogram_pow2_expected (used by the
    2^27 GPU tests) reproduce the reference's reports at 2^20 / 2^22."""
    import programs
    n_checked = 0
    for g in ("large", "xlarge"):
        for c in load_golden(g):
            name, res = c["name"], c["result"]
            got = [(r["kind"], r["address"]) for r in res["races"]]
            wit = [(w["threadA"], w["threadB"]) for w in c["witnesses_restatement"]]
            if name.startswith("permutation_"):
                n, upd = int(name.split("_")[1]), name.split("_", 2)[2]
                want = programs.permutation_expected(n, upd)
            elif name.startswith("histogram_") and name.split("_")[2] == "65536":
                n, upd = int(name.split("_")[1]), name.split("_", 3)[3]
                want = programs.histogram_pow2_expected(n, 65536, upd)
            else:
                continue
            assert got == [(k, a) for k, a, _, _ in want], name
            assert wit == [(x, y) for _, _, x, y in want], name
            n_checked += 1
    assert n_checked >= 5


def test_batched_sweeps(cpu_oracle):
    """The speculative batched sweep (configurations' host runs speculated,
    launches checked as one batch with traps merged in canonical order,
    failed speculations re-run exactly) reproduces the reference's
    enumerateVerdict on the corpus (manifest and default caps), the fuzz
    programs and the config-5 lattice."""
    restarts = configs = 0
    for e in load_golden("corpus"):
        for caps, want in ((e["caps"], e["sweep_manifest"]), ({}, e["sweep_default"])):
            got = cpu_oracle.enumerate_verdict_batched(e["source"], caps, e["file"])
            assert strip_extras(got) == want, e["name"]
    for f in load_golden("fuzz"):
        got = cpu_oracle.enumerate_verdict_batched(f["source"], {}, "fuzz.mcu")
        assert strip_extras(got) == f["sweep"], f["index"]
    for j in load_golden("lattice"):
        got = cpu_oracle.enumerate_verdict_batched(j["source"], j["caps"], j["file"])
        assert strip_extras(got) == j["sweep"], j["name"]
        restarts += got["stats"]["restarts"]
        configs += got["configs"]
    assert configs == 9695 and restarts < configs // 50  # most configurations batched


def test_many_sweeps_and_shards(cpu_oracle):
    """sweepManyJson (hgrd_gpu_enumerate_verdict_many_json's host side): all
    229 config-5 programs in one call reproduce the reference's sweeps, and
    per-rank shards (canonical index % world) merge back to them."""
    from paper_2604_02106_b200.parallel import merge_shards
    lat = load_golden("lattice")
    jobs = [{"source": j["source"], "file": j["file"], "caps": j["caps"]} for j in lat]
    got = cpu_oracle.enumerate_verdict_many(jobs)
    assert [strip_extras(g) for g in got] == [j["sweep"] for j in lat]
    world = 3
    shards = [cpu_oracle.enumerate_verdict_many(jobs, r, world) for r in range(world)]
    for q, j in enumerate(lat):
        assert merge_shards([shards[r][q] for r in range(world)])["races"] == j["sweep"]["races"]
    bad = cpu_oracle.enumerate_verdict_many([{"source": "int main(", "file": "x.mcu"}])
    assert "error" in bad[0]

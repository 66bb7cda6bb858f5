"""GPU parity: the B200 race-check stage (libhgrd_gpu.so, through its C ABI)
against the reference's recorded outputs (tests/golden, generated from the
unmodified reference) on every field the reference reports, and against the
CPU restatement (oracle/) on the witness pairs the reference does not
report.  Bit-exact: integer / index work, no tolerance."""
import numpy as np
import pytest

import paper_2604_02106_b200 as hg
import programs
from conftest import load_golden
from oracles import strip_extras

pytestmark = pytest.mark.gpu


def _check_run(gpu, cpu_oracle, src, cfg, file_name, want):
    got = gpu.run_concrete(src, cfg, file_name)
    assert strip_extras(got) == want, (cfg, got, want)
    ora = cpu_oracle.run_concrete(src, cfg, file_name)
    assert got["witnesses"] == ora["witnesses"], (cfg, got["witnesses"], ora["witnesses"])
    assert got["stats"]["instances"] == ora["stats"]["instances"]
    return got


@pytest.fixture(params=["fused", "general"])
def mode(request, gpu):
    gpu.set_fused(request.param == "fused")
    yield request.param
    gpu.set_fused(True)


def test_corpus_runs(gpu, cpu_oracle, mode):
    for e in load_golden("corpus"):
        for run in e["runs"]:
            _check_run(gpu, cpu_oracle, e["source"], run["config"], e["file"], run["result"])


def test_corpus_sweeps(gpu):
    """Acceptance criterion 4 / corpus.cpp:203-237 on the GPU."""
    for e in load_golden("corpus"):
        got = strip_extras(gpu.enumerate_verdict(e["source"], e["caps"], e["file"]))
        assert got == e["sweep_manifest"], e["name"]
        got = strip_extras(gpu.enumerate_verdict(e["source"], {}, e["file"]))
        assert got == e["sweep_default"], e["name"]


def test_unit_cases(gpu, cpu_oracle, mode):
    for c in load_golden("unit_cases"):
        _check_run(gpu, cpu_oracle, c["source"], c["config"], "oracle.mcu", c["result"])


def test_fuzz(gpu, cpu_oracle, mode):
    """reference tests/test_soundness.cpp programs (mt19937(31337))."""
    total = 0
    for f in load_golden("fuzz"):
        got = strip_extras(gpu.enumerate_verdict(f["source"], {}, "fuzz.mcu"))
        assert got == f["sweep"], f["index"]
        total += len(got["races"])
        for run in f["runs"]:
            _check_run(gpu, cpu_oracle, f["source"], run["config"], "fuzz.mcu", run["result"])
    assert total > 500


def test_edge_programs(gpu, cpu_oracle, mode):
    for c in load_golden("edge"):
        _check_run(gpu, cpu_oracle, c["source"], c["config"], "edge.mcu", c["result"])


def test_synthetic_small(gpu, cpu_oracle, mode):
    for c in load_golden("synthetic"):
        got = _check_run(gpu, cpu_oracle, c["source"], c["config"], "syn.mcu", c["result"])
        assert got["stats"]["parallelLaunches"] >= 1  # the data-parallel path ran


# --------------------------------------------------------------- launch level
def _spec_stencil(ctx, n, barrier, ws=32):
    src = programs.stencil(n, barrier=barrier)
    low = hg.lower(src, "st")
    bufs = [np.zeros(n, np.int64), np.zeros(n // 256 * 258, np.int64), np.zeros(n, np.int64)]
    handles = {}
    if ctx is not None:
        ctx.reset()
        handles = {"in_": ctx.alloc(n), "tile": ctx.alloc(n // 256 * 258), "out_": ctx.alloc(n)}
    else:
        handles = {"in_": 0, "tile": 1, "out_": 2}
    spec = hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), ws, handles=handles)
    return spec, bufs


def _spec_hist(ctx, n, bins, update, ws=32):
    src = programs.histogram(n, bins, update, host_init=False)
    low = hg.lower(src, "h")
    data = programs.histogram_data(n, bins)
    bufs = [data, np.zeros(bins, np.int64)]
    if ctx is not None:
        ctx.reset()
        h = {"data": ctx.alloc(n), "hist": ctx.alloc(bins)}
        ctx.write(h["data"], data)
    else:
        h = {"data": 0, "hist": 1}
    return hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), ws, handles=h), bufs


def _spec_transpose(ctx, n, barrier):
    src = programs.transpose(n, barrier=barrier)
    low = hg.lower(src, "tr")
    ntile = (n // 32) * (n // 32) * 1056
    bufs = [np.zeros(ntile, np.int64), np.zeros(n * n, np.int64)]
    if ctx is not None:
        ctx.reset()
        h = {"tile": ctx.alloc(ntile), "out_": ctx.alloc(n * n)}
    else:
        h = {"tile": 0, "out_": 1}
    return hg.LaunchSpec(low, (n // 32, n // 32, 1), (32, 32, 1), 32,
                         scalars={"n": n}, handles=h), bufs


def _same(a, b):
    keys = ("races", "traps", "steps", "instances", "records", "aborted")
    return {k: a[k] for k in keys} == {k: b[k] for k in keys}


@pytest.mark.parametrize("barrier", [False, True])
@pytest.mark.parametrize("ws", [32, 5])
def test_launch_stencil(gpu, cpu_oracle, barrier, ws):
    spec, bufs = _spec_stencil(gpu, 1 << 14, barrier, ws)
    got = gpu.check_launch(spec)
    ref_spec, _ = _spec_stencil(None, 1 << 14, barrier, ws)
    want = cpu_oracle.check_launch(ref_spec, bufs)
    assert _same(got, want), (got, want)
    spec.launch.flags |= hg.LAUNCH_GENERAL  # the general (global sort) pipeline too
    assert _same(gpu.check_launch(spec), want)
    spec.launch.flags |= hg.LAUNCH_SEQUENTIAL  # and the ordered path
    assert _same(gpu.check_launch(spec), want)


@pytest.mark.parametrize("update", list(programs.HIST_UPDATES))
@pytest.mark.parametrize("bins", [64, 1 << 10, 61])
def test_launch_histogram(gpu, cpu_oracle, update, bins):
    n = 1 << 13
    spec, bufs = _spec_hist(gpu, n, bins, update)
    got = gpu.check_launch(spec)
    ref_spec, _ = _spec_hist(None, n, bins, update)
    want = cpu_oracle.check_launch(ref_spec, bufs)
    assert _same(got, want), (got, want)
    spec.launch.flags |= hg.LAUNCH_GENERAL
    assert _same(gpu.check_launch(spec), want)


@pytest.mark.parametrize("barrier", [False, True])
def test_launch_transpose(gpu, cpu_oracle, barrier):
    spec, bufs = _spec_transpose(gpu, 128, barrier)
    got = gpu.check_launch(spec)
    ref_spec, _ = _spec_transpose(None, 128, barrier)
    want = cpu_oracle.check_launch(ref_spec, bufs)
    assert _same(got, want), (got, want)
    spec.launch.flags |= hg.LAUNCH_GENERAL
    assert _same(gpu.check_launch(spec), want)


# ------------------------------------------------ full size, size-independent
def test_full_stencil_2p20(gpu, cpu_oracle):
    """configs[1]: 2^20 threads.  The first-found element of every key lies in
    block 0, so the full-size report equals the 2^14 oracle report."""
    for barrier in (False, True):
        spec, _ = _spec_stencil(gpu, 1 << 20, barrier)
        got = gpu.check_launch(spec)
        small, bufs = _spec_stencil(None, 1 << 14, barrier)
        want = cpu_oracle.check_launch(small, bufs)
        assert got["races"] == want["races"]
        assert got["instances"] == 5 << 20
        assert got["records"] == 4 << 20


def test_full_transpose_8192(gpu, cpu_oracle):
    """configs[2]: 8192^2, 2^26 instances per interval."""
    for barrier in (False, True):
        spec, _ = _spec_transpose(gpu, 8192, barrier)
        got = gpu.check_launch(spec)
        small, bufs = _spec_transpose(None, 128, barrier)
        want = cpu_oracle.check_launch(small, bufs)
        assert [(r["kind"], r["locA"], r["locB"], r["address"], r["threadA"], r["seqA"],
                 r["threadB"], r["seqB"]) for r in got["races"]] == \
               [(r["kind"], r["locA"], r["locB"], r["address"], r["threadA"], r["seqA"],
                 r["threadB"], r["seqB"]) for r in want["races"]]
        assert got["instances"] == 3 << 26


# ------------------------------------------------------- NVRTC specialisation
def test_jit_forced_edge_and_synthetic(gpu, cpu_oracle):
    """Every launch through NVRTC-specialised kernels (mode 2)."""
    gpu.set_jit(2)
    try:
        for name, fn in (("edge", "edge.mcu"), ("synthetic", "syn.mcu")):
            for c in load_golden(name)[:: 6 if name == "edge" else 1]:
                _check_run(gpu, cpu_oracle, c["source"], c["config"], fn, c["result"])
        info = gpu.jit_info()
        assert info["compiles"] > 0 and info["failures"] == 0, info
    finally:
        gpu.set_jit(1)


def test_jit_used_for_large_launches(gpu):
    gpu.set_profiling(True)
    spec, _ = _spec_stencil(gpu, 1 << 16, False)
    gpu.check_launch(spec)
    names = [s["name"] for s in gpu.last_profile()]
    gpu.set_profiling(False)
    assert any(n.endswith("[jit]") for n in names), (names, gpu.jit_info())


@pytest.mark.parametrize("bins", [1 << 16, 65521])
@pytest.mark.parametrize("update", ["atomic_block", "store", "atomic"])
def test_full_histogram_2p27(gpu, cpu_oracle, bins, update):
    """configs[3]: 2^27 threads, 2^28 instances, data-dependent bins.  The
    first two threads that hit bin 0 are i0 and i0 + bins (< 2^17), so the
    full-size report (races, addresses, witnesses) equals the 2^17 oracle's."""
    spec, _ = _spec_hist(gpu, 1 << 27, bins, update)
    got = gpu.check_launch(spec)
    small, bufs = _spec_hist(None, 1 << 17, bins, update)
    want = cpu_oracle.check_launch(small, bufs)
    assert got["races"] == want["races"]
    assert got["instances"] == 2 << 27


# ------------------------------------------------- SEQUENTIAL at launch scale
@pytest.mark.parametrize("case", ["clean_bounds", "trap_last", "budget"])
def test_sequential_large(gpu, cpu_oracle, case):
    """A 2^16-thread SEQUENTIAL launch through the NVRTC canonical-order body
    (k_expand_seq[jit]): races, traps and the step-budget abort equal the
    CPU restatement's."""
    n = 1 << 16
    src = programs.chain_kernel(n, n if case == "trap_last" else n + 1)
    cfg = programs.synthetic_config(**({"maxSteps": 200000} if case == "budget" else {}))
    gpu.set_profiling(True)
    try:
        got = gpu.run_concrete(src, cfg, "seq.mcu")
        names = [s["name"] for s in gpu.last_profile()]
    finally:
        gpu.set_profiling(False)
    want = cpu_oracle.run_concrete(src, cfg, "seq.mcu")
    assert strip_extras(got) == strip_extras(want), (got, want)
    assert got["witnesses"] == want["witnesses"]
    assert got["stats"]["instances"] == want["stats"]["instances"]
    assert "k_expand_seq[jit]" in names, names
    if case == "trap_last":
        assert got["traps"]


# ------------------------------------------------ lock idioms at launch scale
@pytest.mark.parametrize("variant", ["device", "block", "leak"])
@pytest.mark.parametrize("n", [4096, 16384])
def test_lock_kernels_large(gpu, cpu_oracle, n, variant):
    """Lock-idiom launches with element groups far above the per-thread
    pairwise limit: k_lock_info + the tiled k_detect_pairwise_big against
    the CPU restatement of lockInfo / lockOrdered / detectRaces."""
    src = programs.lock_kernel(n, variant)
    cfg = programs.synthetic_config()
    got = gpu.run_concrete(src, cfg, "lk.mcu")
    want = cpu_oracle.run_concrete(src, cfg, "lk.mcu")
    assert strip_extras(got) == strip_extras(want), (got, want)
    assert got["witnesses"] == want["witnesses"]

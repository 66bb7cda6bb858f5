"""GPU parity at scale against the UNMODIFIED reference's own outputs
(tests/golden/{regress,large,xlarge,lattice}.json, made by make_golden.py):

* regress — launches of more single/two-thread MiniCU blocks than one
  k_fused iteration holds (the iteration's 8-bit block field), hot elements
  in radix mode, 3-D grids of tiny blocks;
* large / xlarge — the north-star workloads at the largest sizes the
  reference runs here: the 2^20 / 2^22 stencil (configs[1]), 2048^2 /
  4096^2 transposes (configs[2] shape), 2^20 / 2^22-thread histograms at
  2^16 and 2^24 bins, hot 64-bin histograms realising INTRA-BLOCK (and
  INTRA-WARP at warp size 128), the permutation scatter with injected
  duplicates (configs[3] variant);
* lattice — BASELINE config 5, enumerateVerdict of 229 programs.

Every reference field must match; witness pairs must match the CPU
restatement's (recorded next to the reference result by make_golden.py,
which asserts the restatement reproduces the reference on that run).
Bit-exact integer work: no tolerance."""
import pytest

import paper_2604_02106_b200 as hg
import programs
from conftest import load_golden
from oracles import strip_extras

pytestmark = pytest.mark.gpu


def _check(gpu, case, file_name="syn.mcu"):
    got = gpu.run_concrete(case["source"], case["config"], file_name)
    assert strip_extras(got) == case["result"], (case["name"], case["config"], got["races"])
    assert got["witnesses"] == case["witnesses_restatement"], case["name"]
    assert got["stats"]["instances"] == case["instances_restatement"], case["name"]
    return got


@pytest.fixture(params=["fused", "general"])
def mode(request, gpu):
    gpu.set_fused(request.param == "fused")
    yield request.param
    gpu.set_fused(True)


def test_regress_tiny_blocks(gpu, mode):
    for c in load_golden("regress"):
        _check(gpu, c, "tiny.mcu")


@pytest.mark.parametrize("jit", [0, 2])
def test_regress_tiny_blocks_jit(gpu, jit):
    """The same launches through the interpreter and the NVRTC bodies."""
    gpu.set_jit(jit)
    try:
        for c in load_golden("regress"):
            _check(gpu, c, "tiny.mcu")
    finally:
        gpu.set_jit(1)


def test_large(gpu):
    for c in load_golden("large"):
        got = _check(gpu, c)
        assert got["stats"]["parallelLaunches"] >= 1, c["name"]


def test_xlarge(gpu):
    for c in load_golden("xlarge"):
        _check(gpu, c)


def test_envelope(gpu, mode):
    """Round-1 ENOTSUP limits, now exact: a thread of more than 2^20
    accesses (record values site << bS | seq with bS = 32 - site bits), in
    the summary and the pairwise detector."""
    for c in load_golden("envelope"):
        _check(gpu, c, "env.mcu")


def test_wide_group_past_old_caps(gpu):
    """The pairwise detector (66 sites) on an element group of 2^20 + 257
    events and 2^26+ events in total (round 1: ENOTSUP past 2^20 / 2^24).
    Same program as the envelope golden's wide_group_4096, which pins the
    report: the races, their witnesses (thread 0 against 1, 32 and 256)
    and 66 instances per thread are size-independent."""
    small = next(c for c in load_golden("envelope") if c["name"] == "wide_group_4096")
    n = (1 << 20) + 256
    got = gpu.run_concrete(programs.wide_group(n), small["config"], "env.mcu")
    assert strip_extras(got)["races"] == small["result"]["races"]
    assert got["witnesses"] == small["witnesses_restatement"]
    assert got["stats"]["instances"] == 66 * n + 1


def test_lattice_config5(gpu):
    """BASELINE config 5: the reference's enumerateVerdict output for every
    program of the 10k-configuration lattice, through the batched sweep
    (k_batch: nearly every launch of the lattice in one batched check per
    program)."""
    jobs = load_golden("lattice")
    assert len(jobs) == 229
    batched = 0
    for j in jobs:
        got = gpu.enumerate_verdict(j["source"], j["caps"], j["file"])
        assert strip_extras(got) == j["sweep"], j["name"]
        batched += got["stats"]["batchedLaunches"]
    assert batched > 8000, batched


def test_sweeps_per_launch_path(gpu):
    """HGRD_SWEEP_BATCH=0: the per-launch sweep path over worker contexts
    gives the same reports (and batches nothing)."""
    import os
    os.environ["HGRD_SWEEP_BATCH"] = "0"
    try:
        for e in load_golden("corpus"):
            got = gpu.enumerate_verdict(e["source"], e["caps"], e["file"])
            assert strip_extras(got) == e["sweep_manifest"], e["name"]
            assert got["stats"]["batchedLaunches"] == 0
    finally:
        del os.environ["HGRD_SWEEP_BATCH"]


# ------------------------------------------- permutation scatter, full size
@pytest.mark.parametrize("update", ["store", "atomic_block", "atomic"])
def test_full_permutation_scatter_2p27(gpu, update):
    """configs[3] permutation variant at 2^27 threads (2^28 instances): B = n
    bins, every bin hit once except the injected duplicates.  Expected report
    from programs.permutation_expected (pinned to the reference at 2^20 and
    2^22 by test_golden_extra.py)."""
    n = 1 << 27
    src = programs.permutation_scatter(n, update, host_init=False)
    low = hg.lower(src, "h")
    gpu.reset()
    h = {"data": gpu.alloc(n), "hist": gpu.alloc(n)}
    gpu.write(h["data"], programs.permutation_data(n))
    spec = hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), 32, handles=h)
    got = gpu.check_launch(spec)
    want = programs.permutation_expected(n, update)
    assert [(r["kind"], r["address"], r["threadA"], r["threadB"]) for r in got["races"]] == want
    assert all(r["array"] == "hist" and r["seqA"] == 1 and r["seqB"] == 1 for r in got["races"])
    assert got["instances"] == 2 * n


@pytest.mark.parametrize("update", ["store", "atomic_block", "atomic"])
def test_full_histogram_2p27_2p24_bins(gpu, update):
    """configs[3] at 2^27 threads x 2^24 bins (8 threads per bin)."""
    n, bins = 1 << 27, 1 << 24
    src = programs.histogram(n, bins, update, host_init=False)
    low = hg.lower(src, "h")
    gpu.reset()
    h = {"data": gpu.alloc(n), "hist": gpu.alloc(bins)}
    gpu.write(h["data"], programs.histogram_data(n, bins))
    spec = hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), 32, handles=h)
    got = gpu.check_launch(spec)
    want = programs.histogram_pow2_expected(n, bins, update)
    assert [(r["kind"], r["address"], r["threadA"], r["threadB"]) for r in got["races"]] == want
    assert got["instances"] == 2 * n

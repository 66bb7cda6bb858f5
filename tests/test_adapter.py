"""The reference-side drop-in (oracle/gpu_adapter.cpp): hgrd_gpu::runConcrete
/ hgrd_gpu::enumerateVerdict take the REFERENCE's own parsed Program and
ExecConfig / SweepCaps and return its OracleResult / SweepRace types,
through the flat-program C ABI of include/hgrd_gpu_program.h.

* CPU: the reference's parse, flattened by the adapter, is the same program
  (every node kind, SourceLoc, node id, name, value) as the library's own
  parse of the source; countInputs agrees.
* GPU: in-process diff against the unmodified hgrd::runConcrete /
  hgrd::enumerateVerdict on every field of the reference's types, including
  LaunchRecord::launchStmt identity and DefKey-keyed defValues."""
import ctypes
import json
import os

import pytest

from conftest import load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ADAPTER = os.path.join(ROOT, "oracle", "_ref", "libhgrd_adapter.so")


@pytest.fixture(scope="module")
def adapter():
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter not built (oracle/Makefile needs /root/reference)")
    lib = ctypes.CDLL(ADAPTER)
    P = ctypes.c_void_p
    lib.hgrd_adapter_dumps.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(P),
                                       ctypes.POINTER(P)]
    lib.hgrd_adapter_count_inputs.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                              ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_int)]
    lib.hgrd_adapter_diff_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                          ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(P)]
    lib.hgrd_adapter_diff_sweep.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                            ctypes.POINTER(P)]
    lib.hgrd_adapter_free.argtypes = [P]
    return lib


def _take(lib, p):
    s = ctypes.string_at(p.value).decode() if p.value else ""
    lib.hgrd_adapter_free(p)
    return s


def _sources():
    """Every distinct (source, file name) of the golden fixtures."""
    seen = {}
    for e in load_golden("corpus"):
        seen[(e["source"], e["file"])] = None
    for g, fn in (("unit_cases", "oracle.mcu"), ("edge", "edge.mcu"), ("synthetic", "syn.mcu"),
                  ("regress", "tiny.mcu")):
        for c in load_golden(g):
            seen[(c["source"], fn)] = None
    for f in load_golden("fuzz"):
        seen[(f["source"], "fuzz.mcu")] = None
    return list(seen)


def test_flattening_is_the_same_program(adapter):
    n = 0
    for src, fn in _sources():
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        rc = adapter.hgrd_adapter_dumps(src.encode(), fn.encode(), ctypes.byref(a),
                                        ctypes.byref(b))
        via_adapter, via_source = _take(adapter, a), _take(adapter, b)
        assert rc == 0, (fn, via_adapter, via_source)
        assert via_adapter == via_source, fn
        ri, gi = ctypes.c_int(), ctypes.c_int()
        assert adapter.hgrd_adapter_count_inputs(src.encode(), fn.encode(), ctypes.byref(ri),
                                                 ctypes.byref(gi)) == 0
        assert ri.value == gi.value
        n += 1
    assert n > 250


def _diff_run(adapter, src, fn, cfg):
    rep = ctypes.c_void_p()
    inst = ctypes.c_ulonglong()
    rc = adapter.hgrd_adapter_diff_run(src.encode(), fn.encode(), json.dumps(cfg).encode(),
                                       ctypes.byref(inst), ctypes.byref(rep))
    return rc, _take(adapter, rep), inst.value


@pytest.mark.gpu
def test_run_concrete_drop_in(adapter):
    cases = []
    for e in load_golden("corpus"):
        cases += [(e["source"], e["file"], r["config"]) for r in e["runs"]]
    for g, fn in (("unit_cases", "oracle.mcu"), ("edge", "edge.mcu"), ("synthetic", "syn.mcu"),
                  ("regress", "tiny.mcu")):
        cases += [(c["source"], fn, c["config"]) for c in load_golden(g)]
    for f in load_golden("fuzz"):
        cases += [(f["source"], "fuzz.mcu", r["config"]) for r in f["runs"]]
    total = 0
    for src, fn, cfg in cases:
        rc, rep, inst = _diff_run(adapter, src, fn, cfg)
        assert rc == 0, (fn, cfg, rep)
        total += inst
    assert len(cases) > 1000 and total > 0


@pytest.mark.gpu
def test_run_concrete_drop_in_large(adapter):
    """The 2^20-thread stencil and the 2^20-thread histograms (host init
    loop included) through the reference's own types."""
    for c in load_golden("large"):
        if c["name"].startswith(("stencil", "histogram_1048576_65536")):
            rc, rep, inst = _diff_run(adapter, c["source"], "syn.mcu", c["config"])
            assert rc == 0, (c["name"], rep)
            assert inst == c["instances_restatement"]


@pytest.mark.gpu
def test_enumerate_verdict_drop_in(adapter):
    jobs = [(e["source"], e["file"], e["caps"]) for e in load_golden("corpus")]
    jobs += [(e["source"], e["file"], {}) for e in load_golden("corpus")]
    jobs += [(f["source"], "fuzz.mcu", {}) for f in load_golden("fuzz")]
    for src, fn, caps in jobs:
        rep = ctypes.c_void_p()
        rc = adapter.hgrd_adapter_diff_sweep(src.encode(), fn.encode(), json.dumps(caps).encode(),
                                             ctypes.byref(rep))
        assert rc == 0, (fn, caps, _take(adapter, rep))
        _take(adapter, rep)

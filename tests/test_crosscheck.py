"""Static-verdict cross-check (tests/crosscheck.py):
every race a concrete sweep observes must be in the reference static
analyzer's report at that warp size (the reference corpus runner's soundness
check, src/corpus.cpp:219-236), over input / launch-cap / warp-size lattices
far wider than the corpus manifests — on the GPU through the batched sweep,
on CPU (smaller lattice) through the restatement."""
import os

import pytest

import crosscheck
from conftest import load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _programs():
    return [{"name": e["name"], "source": e["source"], "file": e["file"]}
            for e in load_golden("corpus")]


def test_crosscheck_cpu(cpu_oracle, ref_oracle):
    caps = dict(crosscheck.WIDE_CAPS, inputSet=[-1, 0, 1, 2, 3, 4, 7, 8, 16, 33, 64],
                warpSizes=[1, 2, 4, 32])
    rep = crosscheck.crosscheck(cpu_oracle.enumerate_verdict_many, ref_oracle, _programs(),
                                caps)
    assert rep["unsound_total"] == 0, [p for p in rep["programs"] if p["unsound"]]
    assert rep["configs"] > 8000 and rep["static_races_realised"] > 100


@pytest.mark.gpu
def test_crosscheck_gpu(gpu, ref_oracle):
    rep = crosscheck.crosscheck(gpu.enumerate_verdict_many, ref_oracle, _programs())
    assert rep["unsound_total"] == 0, [p for p in rep["programs"] if p["unsound"]]
    assert rep["configs"] > 80000
    assert rep["static_races_realised"] == rep["static_races"]

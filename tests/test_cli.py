"""The GPU-backed CLI (python -m paper_2604_02106_b200): `oracle` mirrors the
reference's `hgrd oracle` output (tools/hgrd.cpp:114-137) and `corpus` runs
the oracle half of its corpus runner (src/corpus.cpp:203-216)."""
import io
import json
import os
import contextlib

import pytest

from conftest import load_golden
from paper_2604_02106_b200.__main__ import main, parse_manifest, run_corpus

REF_CORPUS = "/root/reference/proj/corpus"


@pytest.mark.skipif(not os.path.isdir(REF_CORPUS), reason="reference corpus not present")
def test_manifest_parse_matches_reference():
    """Oracle mode and caps of every bundled manifest, as the reference
    parsed them when the goldens were generated (tests/golden/corpus.json)."""
    golden = {e["name"]: e for e in load_golden("corpus")}
    n = 0
    for name in sorted(os.listdir(REF_CORPUS)):
        if name.endswith(".manifest"):
            m = parse_manifest(os.path.join(REF_CORPUS, name))
            e = golden[m["name"]]
            assert (m["oracle"], m["caps"]) == (e["oracle"], e["caps"]), name
            n += 1
    assert n == len(golden) == 29


def _write_corpus(tmp_path):
    for e in load_golden("corpus"):
        (tmp_path / f"{e['name']}.mcu").write_text(e["source"])
        lines = [f"name = {e['name']}", f"source = {e['name']}.mcu", f"oracle = {e['oracle']}"]
        caps = e["caps"]
        keys = {"gridCap": "oracle_grid_cap", "blockCap": "oracle_block_cap",
                "inputSet": "oracle_inputs", "warpSizes": "oracle_warp_sizes"}
        for k, key in keys.items():
            if k in caps:
                lines.append(f"{key} = " + " ".join(str(v) for v in caps[k]))
        if "maxThreads" in caps:
            lines.append(f"oracle_max_threads = {caps['maxThreads']}")
        (tmp_path / f"{e['name']}.manifest").write_text("\n".join(lines) + "\n")


@pytest.mark.gpu
def test_corpus_runner(gpu, tmp_path):
    _write_corpus(tmp_path)
    rows = run_corpus(str(tmp_path), gpu)
    assert len(rows) == 29 and all(r["pass"] for r in rows), [r for r in rows if not r["pass"]]
    assert sum(r["oracle"] == "racy" for r in rows) > 0


@pytest.mark.gpu
def test_oracle_cli_output(gpu, tmp_path):
    """`oracle` with default caps prints the reference's race list."""
    for e in load_golden("corpus")[:8]:
        path = tmp_path / e["file"].split("/")[-1]
        path.write_text(e["source"])
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            rc = main(["oracle", str(path)])
        got = json.loads(out.getvalue())
        want = e["sweep_default"]["races"]
        assert rc == (1 if want else 0)
        assert [(r["kind"], r["locA"]["line"], r["locB"]["line"], r["warpSize"])
                for r in got["races"]] == \
            [(r["kind"], r["locA"]["line"], r["locB"]["line"], r["warpSize"]) for r in want]

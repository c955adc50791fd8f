"""JSONL ingest, CPU side: the decimal -> binary64 conversion the GPU parser uses
(csrc/decimal.cuh) against the C library's strtod (what nlohmann's lexer calls), and the committed
golden fixtures (tests/golden/jsonl_ref.json) pinned to the reference's own parse_jsonl_records
(oracle/_ref, serde.hpp:158-170) when it is built."""
import base64
import json
import os
import subprocess
import struct

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "jsonl_ref.json")


def test_decimal_conversion_matches_strtod(tmp_path):
    exe = str(tmp_path / "decimal_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "paper_2512_09200_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "decimal_check.cpp"), "-o", exe], check=True)
    for seed in (1, 2, 3):
        r = subprocess.run([exe, "300000", str(seed)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.startswith("ok")


def test_golden_cases_cover_the_spec():
    import jsonl_cases
    g = json.load(open(GOLDEN))
    assert [c["name"] for c in g] == [n for n, _ in jsonl_cases.cases()]
    for c, (_, content) in zip(g, jsonl_cases.cases()):
        assert base64.b64decode(c["content_b64"]) == content
        assert (c["records"] is None) == (c["error"] is not None)
        assert c["name"].startswith("err_") == (c["error"] is not None), c["name"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_golden_is_the_reference():
    g = json.load(open(GOLDEN))
    for c in g:
        recs, err = oracle.ref_parse_jsonl(base64.b64decode(c["content_b64"]), c["name"] + ".jsonl")
        assert err == c["error"], c["name"]
        if recs is not None:
            for r in recs:
                r["features"] = {k: struct.pack(">d", v).hex() for k, v in r["features"].items()}
            assert recs == c["records"], c["name"]

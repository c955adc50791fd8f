"""JSONL impression ingest on the GPU (lattice_jsonl_*, csrc/jsonl.cu) against the reference's
parse_jsonl_records (serde.hpp:158-170): every committed golden case bit-exact (records, feature
values as IEEE bits, conversions) or the same error (line, kind, and nlohmann's exact text for
record-level errors); a large random file against the live reference (oracle/_ref); and the zip
path (JSONL -> columns -> Zipper kernel) against the reference's zip_dataset."""
import base64
import json
import os
import struct

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "jsonl_ref.json")))


def _bits(recs):
    for r in recs:
        r.pop("line", None)
        r["features"] = {k: struct.pack(">d", v).hex() for k, v in r["features"].items()}
    return recs


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_golden_case(case):
    import paper_2512_09200_b200 as L
    content = base64.b64decode(case["content_b64"])
    src = case["name"] + ".jsonl"
    if case["error"] is None:
        assert _bits(L.jsonl_records(content, src)) == case["records"]
        return
    with pytest.raises(L.DataError) as ei:
        L.jsonl_records(content, src)
    got, want = str(ei.value), case["error"]
    if want.startswith("exception: "):  # nlohmann out_of_range.406: not a DataError in the reference
        assert got == want[len("exception: "):]
        return
    where, msg = want.split(": ", 1)
    assert got.startswith(where + ": "), (got, want)
    if "parse_error" in msg:  # same code and line; the GPU parser words the reason its own way
        assert got[len(where) + 2:].startswith("[json.exception.parse_error.101] parse error at line 1, column ")
    else:
        assert got == want


def test_random_file_matches_reference():
    import jsonl_cases
    import paper_2512_09200_b200 as L
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    content = jsonl_cases.random_file(20000, 5)
    recs, err = oracle.ref_parse_jsonl(content, "big.jsonl")
    assert err is None
    got = L.jsonl_records(content, "big.jsonl")
    assert len(got) == len(recs) == 20000
    assert _bits(got) == _bits(recs)


def test_blank_lines_keep_line_numbers():
    import paper_2512_09200_b200 as L
    content = b'\n\n{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1}\n \n' \
              b'{"domain":"d","user_id":"v","ad_id":"a","impression_time_ms":2}'
    cols = L.jsonl_columns(content)
    assert cols["records"] == 2 and cols["lines"] == 5
    assert cols["line"].cpu().tolist() == [3, 5]


def test_zip_from_jsonl_matches_reference_zip_dataset():
    """JSONL -> columns -> task columns -> the Zipper kernel, vs the reference parsing the same
    file and running zip_dataset (datasets.hpp:199-249) on its records."""
    import torch

    import jsonl_cases
    import paper_2512_09200_b200 as L
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    tasks = ["cvr", "ctr", "atc"]
    content = jsonl_cases.random_file(30000, 9, tasks)
    cols = L.jsonl_columns(content)
    conv, pres = L.jsonl_task_columns(cols, tasks)
    dur, pr = [5_400_000, 86_400_000, 604_800_000], [0.5, 0.3, 0.2]
    n = cols["records"]
    w, lab, _ = L.zipper_assign_labels(cols["user"], cols["user_off"], cols["ad"], cols["ad_off"], cols["ts"][:n],
                                       conv, pres, dur, pr, 7)
    recs, err = oracle.ref_parse_jsonl(content)
    assert err is None
    users = [r["user_id"].encode() for r in recs]
    ads = [r["ad_id"].encode() for r in recs]
    ts = np.array([r["impression_time_ms"] for r in recs], dtype=np.int64)
    rc = np.array([[r["conversions"].get(t, 0) for t in tasks] for r in recs], dtype=np.int64)
    rp = np.array([[t in r["conversions"] for t in tasks] for r in recs], dtype=np.uint8)
    assert np.array_equal(conv.cpu().numpy(), rc) and np.array_equal(pres.cpu().numpy(), rp)
    status, rw, rl, msg = oracle.ref_zip_dataset(users, ads, ts, rc, rp, dur, pr, 7)
    assert status == 0, msg
    assert np.array_equal(w.cpu().numpy(), rw)
    assert np.array_equal(lab.cpu().numpy(), rl)
    torch.cuda.synchronize()


def test_wide_records_with_duplicates_match_reference():
    """Records with hundreds of feature keys, repeated keys (the last occurrence wins), escaped
    spellings of the same key and 17-digit values: the per-object duplicate scan at width."""
    import json
    import random

    import paper_2512_09200_b200 as L
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(11)
    lines = []
    for i in range(300):
        items = []
        for k in range(rng.randint(100, 300)):
            key = f"f{rng.randint(0, 150)}"
            if rng.random() < 0.1:
                key = key.replace("f", "\\u0066", 1)  # the same key, escaped
            items.append(f'"{key}":{rng.uniform(-1e6, 1e6)!r}')
        conv = ",".join(f'"t{rng.randint(0, 5)}":{1700000000000 + rng.randint(0, 10**9)}' for _ in range(10))
        lines.append('{"domain":"w","user_id":"u%d","ad_id":"a","impression_time_ms":%d,"features":{%s},'
                     '"conversions":{%s}}' % (i, 1700000000000 + i, ",".join(items), conv))
    content = ("\n".join(lines) + "\n").encode()
    recs, err = oracle.ref_parse_jsonl(content, "wide.jsonl")
    assert err is None, err
    assert _bits(L.jsonl_records(content, "wide.jsonl")) == _bits(recs)


"""Generates tests/golden/jsonl_ref.json from the REFERENCE itself: parse_jsonl_records
(serde.hpp:158-170) compiled in place into oracle/_ref/libref.so (oracle/Makefile), run on every
case of tests/jsonl_cases.py. Run here (where /root/reference exists):
    python tests/golden/make_jsonl_golden.py
Feature values are stored as the hex of their IEEE bits (exact)."""
import base64
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import jsonl_cases  # noqa: E402


def main():
    out = []
    for name, content in jsonl_cases.cases():
        recs, err = oracle.ref_parse_jsonl(content, name + ".jsonl")
        if recs is not None:
            for r in recs:
                r["features"] = {k: struct.pack(">d", v).hex() for k, v in r["features"].items()}
        out.append({"name": name, "content_b64": base64.b64encode(content).decode(), "records": recs,
                    "error": err})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "jsonl_ref.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, ensure_ascii=False)
    print(path, len(out))


if __name__ == "__main__":
    main()

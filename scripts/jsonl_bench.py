"""JSONL impression ingest throughput: the GPU parser (lattice_jsonl_open + extract: line split,
validation, record checks, columns) vs the reference's parse_jsonl_records (oracle/_ref, one host
thread, as the CLI runs it) on the same synthetic file. Prints one JSON line.
usage: python scripts/jsonl_bench.py [records] [ref_sample_records]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import jsonl_cases  # noqa: E402
import oracle  # noqa: E402
import paper_2512_09200_b200 as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
content = jsonl_cases.random_file(n, 3)
host = torch.frombuffer(bytearray(content), dtype=torch.uint8).pin_memory()
dev = host.cuda()
for _ in range(2):
    L.jsonl_columns(dev)
torch.cuda.synchronize()
K = 10
t0 = time.perf_counter()
for _ in range(K):
    cols = L.jsonl_columns(dev)
torch.cuda.synchronize()
t_dev = (time.perf_counter() - t0) / K
t0 = time.perf_counter()
for _ in range(K):
    d = host.cuda(non_blocking=True)
    cols = L.jsonl_columns(d)
    for k in ("user", "ad", "ts", "feature_val", "conversion_val"):
        cols[k].cpu()
torch.cuda.synchronize()
t_e2e = (time.perf_counter() - t0) / K
sample = b"\n".join(content.split(b"\n")[:ns]) + b"\n"
t0 = time.perf_counter()
recs, err = oracle.ref_parse_jsonl(sample)
t_ref = time.perf_counter() - t0
assert err is None
print(json.dumps({"metric": "JSONL impression ingest records/s", "records": cols["records"], "bytes": len(content),
                  "gpu_device_resident": {"records_per_s": cols["records"] / t_dev, "GB_per_s": len(content) / t_dev / 1e9,
                                          "ms": t_dev * 1e3},
                  "gpu_e2e_host_buffers": {"records_per_s": cols["records"] / t_e2e, "ms": t_e2e * 1e3},
                  "reference_cpu": {"records_per_s": len(recs) / t_ref, "cores": 1, "sample_records": len(recs),
                                    "kind": "reference (parse_jsonl_records, oracle/_ref)"}}))

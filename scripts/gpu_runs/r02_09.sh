#!/bin/bash
# round 2, call 9: large-n FM/LCB v2 (chunked X, deep W_L ring, 15 warps): parity first, then
# kernel timing A/B against the previous library (ab/liblattice_prev.so)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_09.jsonl
rm -f $PARITY_LOG
timeout 900 python -m pytest tests/test_fm_lcb_gpu.py tests/test_network_gpu.py -q -rf -p no:cacheprovider -k "512 or 384 or large" > gpurun_out/pytest_r02_09.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_09.log
if grep -q "pytest rc=0" gpurun_out/pytest_r02_09.log; then
  for rep in 1 2; do
    timeout 300 python scripts/fm_bench.py >> gpurun_out/fm_bench_v2.log 2>&1
    LATTICE_LIB=ab/liblattice_prev.so timeout 300 python scripts/fm_bench.py >> gpurun_out/fm_bench_v1.log 2>&1
  done
fi

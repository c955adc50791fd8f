#!/bin/bash
# round 2, call 16: large-n FM/LCB with the warp-converged MMA issuer: parity, timing A/B vs the
# previous library, wait-site trace
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fm_lcb_gpu.py tests/test_network_gpu.py -q -rf -p no:cacheprovider -k "512 or 384 or large" > gpurun_out/pytest_r02_16.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_16.log
if grep -q "pytest rc=0" gpurun_out/pytest_r02_16.log; then
  rm -f gpurun_out/fm16_*.log
  for rep in 1 2; do
    timeout 300 python scripts/fm_bench.py >> gpurun_out/fm16_new.log 2>&1
    LATTICE_LIB=ab/liblattice_v5.so timeout 300 python scripts/fm_bench.py >> gpurun_out/fm16_prev.log 2>&1
  done
  LATTICE_FM_TRACE=1 timeout 300 python scripts/fm_bench.py large > gpurun_out/fm16_trace.log 2>&1
fi

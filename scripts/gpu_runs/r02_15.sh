#!/bin/bash
# round 2, call 15: towers on the CTA-pair GEMM: parity (network, dense, portfolio, backward), then
# the mid bench with and without it on the same box
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_15.jsonl
rm -f $PARITY_LOG
timeout 1200 python -m pytest tests/test_network_gpu.py tests/test_dense_gpu.py tests/test_portfolio_gpu.py tests/test_backward_gpu.py tests/test_dropin_gpu.py -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_15.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_15.log
if grep -q "pytest rc=0" gpurun_out/pytest_r02_15.log; then
  for rep in 1 2; do
    timeout 600 python bench.py --no-micro --cpu-seconds 1 > gpurun_out/bench15_pair_$rep.json 2>/dev/null
    LATTICE_TOWER_PAIR=0 timeout 600 python bench.py --no-micro --cpu-seconds 1 > gpurun_out/bench15_single_$rep.json 2>/dev/null
  done
fi

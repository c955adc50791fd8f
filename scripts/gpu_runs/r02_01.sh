#!/bin/bash
# round 2, call 1: new parity suite (torch fp64 restatement, K2 kernel tests, full portfolio,
# large real widths) with the observed errors logged
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_01.jsonl
rm -f $PARITY_LOG
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/pytest_r02_01.log
echo "pytest rc=$?" >> gpurun_out/pytest_r02_01.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/pytest_r02_01.log

#!/bin/bash
# round 2, call 11: backward (VJP adjoint vs reference JVP, routed BCE, tower backward vs fp64,
# DP trainer), MN-major GEMM operands
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_11.jsonl
rm -f $PARITY_LOG
timeout 900 python -m pytest tests/test_backward_gpu.py tests/test_gemm_gpu.py -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_11.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_11.log

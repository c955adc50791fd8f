#!/bin/bash
# round 2, call 24: last-block MLP backward (parity vs autograd restatement, training) + backward suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/r24_parity_errors.jsonl timeout 900 python -m pytest tests/test_backward_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r24_backward.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r24_backward.log
echo done

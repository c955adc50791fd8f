#!/bin/bash
# round 2, call 17: warp-converged MMA issue in both GEMM kernels: GEMM + network parity, then the
# mid bench A/B against the previous library on the same box
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_network_gpu.py tests/test_backward_gpu.py -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_17.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_17.log
if grep -q "pytest rc=0" gpurun_out/pytest_r02_17.log; then
  for rep in 1 2; do
    timeout 600 python bench.py --no-micro --cpu-seconds 1 > gpurun_out/bench17_new_$rep.json 2>/dev/null
    LATTICE_LIB=ab/liblattice_v4.so timeout 600 python bench.py --no-micro --cpu-seconds 1 > gpurun_out/bench17_prev_$rep.json 2>/dev/null
  done
fi

#!/bin/bash
# round 2, call 47: swish GEMM row-exchange with relaxed polling + relaxed drained-TMEM arrivals:
# GEMM/network parity, then same-box A/B of the default bench line (3 reps, no micro) and the
# ncu launch list of one mid forward
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_network_gpu.py tests/test_backward_gpu.py -q -rA -p no:cacheprovider -x > gpurun_out/r47_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r47_tests.log
grep -q "tests rc=0" gpurun_out/r47_tests.log || exit 0
for rep in 1 2 3; do
  timeout 600 python bench.py --no-micro --cpu-seconds 1 >> gpurun_out/r47_new.json 2>/dev/null
  LATTICE_LIB=$GRAFT_REPO_ROOT/ab/liblattice_prev.so timeout 600 python bench.py --no-micro --cpu-seconds 1 >> gpurun_out/r47_prev.json 2>/dev/null
done
CMD="python bench.py --steps 2 --warmup 3 --no-micro --cpu-seconds 1"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"gemm2" -c 13 --csv \
    --log-file gpurun_out/r47_launches.csv $CMD > gpurun_out/r47_ncu.log 2>&1
echo done

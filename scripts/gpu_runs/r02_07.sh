#!/bin/bash
# round 2, call 7: default bench line (micro clocks, DRAM/L2 split), concurrency tests, ncu of the
# swish GEMM (cooperative launch skipped under the profiler's injection), smoke launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02_07.json 2> gpurun_out/bench_r02_07.err
echo "bench rc=$?" >> gpurun_out/bench_r02_07.err
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -s -k "two_networks" -p no:cacheprovider > gpurun_out/conc_r02_07.log 2>&1
python scripts/coop_ncu_probe.py > gpurun_out/coop_plain.log 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm \
      python scripts/coop_ncu_probe.py > gpurun_out/coop_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/coop_ncu.log

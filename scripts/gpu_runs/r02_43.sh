#!/bin/bash
# round 2, call 43: large K2 kernel with Y^T resident (LATTICE_FM_YRES=1, 3 W_L stages) vs the
# 2-deep Y^T ring (5 W_L stages): parity with the resident variant, then alternating timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
LATTICE_FM_YRES=1 timeout 600 python -m pytest tests/test_fm_lcb_gpu.py -q -rA -p no:cacheprovider -k "512 or 384 or 400" > gpurun_out/r43_fm.log 2>&1
echo "fm rc=$?" >> gpurun_out/r43_fm.log
grep -q "fm rc=0" gpurun_out/r43_fm.log || exit 0
for rep in 1 2 3; do
  LATTICE_FM_YRES=1 timeout 300 python scripts/fm_bench.py large >> gpurun_out/r43_yres.log 2>&1
  timeout 300 python scripts/fm_bench.py large >> gpurun_out/r43_ring.log 2>&1
done
LATTICE_FM_YRES=1 LATTICE_FM_TRACE=1 timeout 120 python scripts/fm_bench.py large 2>&1 | tail -14 > gpurun_out/r43_trace.log
echo done

#!/bin/bash
# round 2, call 32: large K2 kernel with L + X kept in TMEM between the LCB epilogue's two passes
# (residual read once): K2 parity, then same-box A/B against the previous library (3 reps each)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/r32_parity.jsonl timeout 600 python -m pytest tests/test_fm_lcb_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r32_fm.log 2>&1
echo "fm rc=$?" >> gpurun_out/r32_fm.log
grep -q "fm rc=0" gpurun_out/r32_fm.log || exit 0
for rep in 1 2 3; do
  timeout 300 python scripts/fm_bench.py large >> gpurun_out/r32_new.log 2>&1
  LATTICE_LIB=$GRAFT_REPO_ROOT/ab/liblattice_prev.so timeout 300 python scripts/fm_bench.py large >> gpurun_out/r32_prev.log 2>&1
done
LATTICE_FM_TRACE=1 timeout 120 python scripts/fm_bench.py large 2>&1 | tail -14 > gpurun_out/r32_trace.log
echo done

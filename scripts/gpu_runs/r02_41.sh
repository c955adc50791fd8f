#!/bin/bash
# round 2, call 41: end-of-round single-GPU record (final code): GPU suite (release + debug library), smoke, the default
# bench line, the large-n FM/LCB kernel timing, and the mid launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_41.jsonl
rm -f $PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_41.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_41.log
PARITY_LOG= LATTICE_LIB=$GRAFT_REPO_ROOT/paper_2512_09200_b200/liblattice_b200_debug.so timeout 1500 \
    python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_dropin_gpu.py > gpurun_out/pytest_debug_r02_41.log 2>&1
echo "pytest(debug lib) rc=$?" >> gpurun_out/pytest_debug_r02_41.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_41.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r02_41.log
timeout 900 python bench.py > gpurun_out/bench_r02_41.json 2> gpurun_out/bench_r02_41.err
echo "bench rc=$?" >> gpurun_out/bench_r02_41.err
timeout 300 python scripts/fm_bench.py > gpurun_out/fm_bench_r02_41.log 2>&1

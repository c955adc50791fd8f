#!/bin/bash
# round 2, call 13: the full GPU suite on the release library, then again on the debug library
# (pipeline waits time out with a report: the sanitizer substitute on this pool), and smoke()
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_13.jsonl
rm -f $PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_13.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_13.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_13.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r02_13.log
PARITY_LOG= LATTICE_LIB=$GRAFT_REPO_ROOT/paper_2512_09200_b200/liblattice_b200_debug.so timeout 1500 \
    python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_dropin_gpu.py > gpurun_out/pytest_debug_r02_13.log 2>&1
echo "pytest(debug lib) rc=$?" >> gpurun_out/pytest_debug_r02_13.log

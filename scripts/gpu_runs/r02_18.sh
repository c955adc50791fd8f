#!/bin/bash
# round 2, call 18: final single-GPU record: GPU suite (release + debug library), smoke, the default
# bench line, the large-n FM/LCB kernel timing, and the mid launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_18.jsonl
rm -f $PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_18.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_18.log
PARITY_LOG= LATTICE_LIB=$GRAFT_REPO_ROOT/paper_2512_09200_b200/liblattice_b200_debug.so timeout 1500 \
    python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_dropin_gpu.py > gpurun_out/pytest_debug_r02_18.log 2>&1
echo "pytest(debug lib) rc=$?" >> gpurun_out/pytest_debug_r02_18.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_18.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r02_18.log
timeout 900 python bench.py > gpurun_out/bench_r02_18.json 2> gpurun_out/bench_r02_18.err
echo "bench rc=$?" >> gpurun_out/bench_r02_18.err
timeout 300 python scripts/fm_bench.py > gpurun_out/fm_bench_r02_18.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-micro --cpu-seconds 1"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
$CMD > gpurun_out/plain18.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"bag_kernel|fm_lcb|gemm|bucket|tiles|heads" -c 46 --csv \
    --log-file gpurun_out/launches_mid_r02_final.csv $CMD > gpurun_out/ncu18.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu18.log

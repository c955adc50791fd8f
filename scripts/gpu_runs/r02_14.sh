#!/bin/bash
# round 2, call 14: mid-step launch list with DRAM / L2 / tensor-pipe metrics per launch, and one
# ncu --set full capture of the MLP GEMM (gemm2_kernel) and of the grouped tower GEMM
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-micro --cpu-seconds 1"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
$CMD > gpurun_out/plain14.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"bag_kernel|fm_lcb|gemm|bucket|tiles|hist|rank|scan" -c 44 --csv \
    --log-file gpurun_out/launches_mid_r02.csv $CMD > gpurun_out/ncu14a.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu14a.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel" -s 2 -c 1 \
    -o gpurun_out/gemm2_mid_r02 $CMD > gpurun_out/ncu14b.log 2>&1
echo "gemm2 rc=$?" >> gpurun_out/ncu14b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^gemm_kernel|gemm_kernel<" -s 0 -c 1 \
    -o gpurun_out/tower_mid_r02 $CMD > gpurun_out/ncu14c.log 2>&1
echo "tower rc=$?" >> gpurun_out/ncu14c.log

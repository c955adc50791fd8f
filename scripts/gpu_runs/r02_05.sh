#!/bin/bash
# round 2, call 5: L2 probe, the new default bench line (mid + micro bf16/f32 + Zipper + CPU
# baselines at 1 and all threads), and ncu DRAM/L2 bytes per launch for traffic.json
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
./scripts/l2_probe > gpurun_out/l2_probe.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02_05.json 2> gpurun_out/bench_r02_05.err
echo "bench rc=$?" >> gpurun_out/bench_r02_05.err
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum
CMD="python bench.py --steps 2 --warmup 3 --no-micro --cpu-seconds 1"
$CMD > gpurun_out/plain_mid.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"bag_kernel|fm_lcb|gemm" -c 18 --csv \
    --log-file gpurun_out/traffic_mid.csv $CMD > gpurun_out/ncu_mid.log 2>&1
for dt in bf16 f32; do
  CMD="python bench.py --workload micro --dtype $dt --steps 2 --warmup 3 --cpu-seconds 1"
  $CMD > gpurun_out/plain_micro_$dt.log 2>&1 && \
    timeout 600 ncu --metrics $M --clock-control none -k regex:"bag_kernel" -c 1 --csv \
      --log-file gpurun_out/traffic_micro_$dt.csv $CMD > gpurun_out/ncu_micro_$dt.log 2>&1
done
echo done

B="python bench.py --steps 2 --warmup 3 --cpu-seconds 1"
timeout 300 $B > gpurun_out/plain_mid.json 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag_l2 $B > gpurun_out/ncu_bag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 1 -o gpurun_out/prof_tower $B > gpurun_out/ncu_tower.log 2>&1
ls -la gpurun_out/*.ncu-rep

# round-1 profile set (current kernels), mid workload, 1 GPU; every ncu after the plain run exits 0
B="python bench.py --steps 2 --warmup 3 --cpu-seconds 1"
timeout 300 $B > gpurun_out/plain_mid.json 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 0 -c 3 -o gpurun_out/prof_gemm_mlp $B > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fm_lcb -s 4 -c 1 -o gpurun_out/prof_fm $B > gpurun_out/ncu_fm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag $B > gpurun_out/ncu_bag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 1 -o gpurun_out/prof_tower $B > gpurun_out/ncu_tower.log 2>&1
ls -la gpurun_out/*.ncu-rep

# detailed captures of the mid bag kernel and the tower GEMM (memory workload / stall reasons)
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:bag_kernel -c 1 -o gpurun_out/prof_bag_mid python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_bag.log 2>&1; echo rc=$?
timeout 900 $NCU -k regex:'^gemm_kernel' -c 1 -o gpurun_out/prof_tower_mid python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_tower.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_bag.log gpurun_out/ncu_tower.log
ls -la gpurun_out

# final full ncu captures of the bag kernel, the tower GEMM and the middle (2048x2048 swish) MLP GEMM
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:bag_kernel -c 1 -o gpurun_out/prof_bag_final python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > /dev/null 2>&1; echo bag rc=$?
timeout 900 $NCU -k regex:'^gemm_kernel' -c 1 -o gpurun_out/prof_tower_final python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > /dev/null 2>&1; echo tower rc=$?
timeout 900 $NCU -k regex:gemm2_kernel -s 1 -c 1 -o gpurun_out/prof_gemm_mid_final python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > /dev/null 2>&1; echo gemm rc=$?

# FM/LCB (mid) and the large-n variant: full ncu captures with source for stall attribution
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:fm_lcb_kernel -c 1 -o gpurun_out/prof_fm_mid python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_fm.log 2>&1; echo rc=$?

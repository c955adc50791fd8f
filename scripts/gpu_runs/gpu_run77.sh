# end-of-session record, 1 GPU: full GPU suite, smoke, drop-in, default bench + reference arm,
# full workload, launch list of the default bench, full ncu capture of the new FM/LCB kernel
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 300 tests/cpp/test_dropin > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; tail -1 gpurun_out/dropin.log
timeout 400 python bench.py > gpurun_out/n1.json 2>gpurun_out/n1.err; echo bench rc=$?; tail -c 300 gpurun_out/n1.json
timeout 400 python bench.py --impl reference > gpurun_out/ref.json 2>gpurun_out/ref.err; echo ref rc=$?
timeout 400 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/full_n1.json 2>gpurun_out/full_n1.err; echo full rc=$?
timeout 400 python bench.py --workload micro > gpurun_out/micro_bf16.json 2>/dev/null; echo micro rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_mid_r01end.csv python bench.py --steps 2 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fm_lcb_kernel -c 1 -o gpurun_out/prof_fm_r01end python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_fm.log 2>&1; echo ncu_fm rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_last_r01end python bench.py --steps 1 --warmup 3 --no-graph --cpu-seconds 0.1 > gpurun_out/ncu_gemm.log 2>&1; echo ncu_gemm rc=$?

# tower split-K after the exchange-phase fix: short timeouts first
timeout 240 python -m pytest tests/test_network_gpu.py -x -q -k "routing or mid_config_matches or forward_matches" > gpurun_out/pytest_ks_quick.log 2>&1; echo quick rc=$?; tail -3 gpurun_out/pytest_ks_quick.log

timeout 900 python scripts/bag_sweep.py l2 > gpurun_out/bag_l2.log 2>&1; cat gpurun_out/bag_l2.log

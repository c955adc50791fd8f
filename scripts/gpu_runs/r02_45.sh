#!/bin/bash
# round 2, call 45 (4 GPUs): final code -- multi-GPU tests, mid / large / full bench at N=4, reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
N=4
timeout 900 python -m pytest tests/test_multi_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r45_mgpu_pytest_n$N.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r45_mgpu_pytest_n$N.log
P=29931
for wl in mid large full; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      bench.py --gpus $N --workload $wl > gpurun_out/r45_bench_${wl}_n$N.json 2> gpurun_out/r45_bench_${wl}_n$N.err
  echo "bench $wl rc=$?" >> gpurun_out/r45_bench_${wl}_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29939 \
    bench.py --gpus $N --impl reference > gpurun_out/r45_bench_ref_n$N.json 2> gpurun_out/r45_bench_ref_n$N.err
echo done

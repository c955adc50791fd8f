#!/bin/bash
# round 2, call 23 (4 GPUs): mid / large / full bench at N=4 after the split-L-M-tile FM/LCB kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
N=4
P=29901
for wl in mid large full; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      bench.py --gpus $N --workload $wl > gpurun_out/r23_bench_${wl}_n$N.json 2> gpurun_out/r23_bench_${wl}_n$N.err
  echo "bench $wl rc=$?" >> gpurun_out/r23_bench_${wl}_n$N.err
done
echo done

#!/bin/bash
# round 2, call 6: L2 probe (.cg loads), ncu on the cooperative swish GEMM (COOP=1 vs 0)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
./scripts/l2_probe > gpurun_out/l2_probe_cg.log 2>&1
for c in 0 1; do
  LATTICE_GEMM_COOP=$c python scripts/coop_ncu_probe.py > gpurun_out/coop_plain_$c.log 2>&1 && \
  LATTICE_GEMM_COOP=$c timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm \
      python scripts/coop_ncu_probe.py > gpurun_out/coop_ncu_$c.log 2>&1
  echo "coop=$c rc=$?" >> gpurun_out/coop_ncu_$c.log
done

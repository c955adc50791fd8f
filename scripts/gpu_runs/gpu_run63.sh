# overlap feasibility: bag kernel on a second stream beside the dense stage, bag blocks/SM capped
for c in 0 1 2 3; do
  LATTICE_BAG_BLOCKS_PER_SM=$c timeout 240 python scripts/overlap_probe.py 2>&1 | tail -4
done | tee gpurun_out/overlap_probe.log

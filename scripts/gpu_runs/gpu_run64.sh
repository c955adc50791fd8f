for p in net rand ident; do
  PROBE_POS=$p timeout 240 python scripts/overlap_probe.py 2>&1 | tail -5
done | tee gpurun_out/overlap_probe2.log
for c in 1 2 3; do
  LATTICE_BAG_BLOCKS_PER_SM=$c timeout 240 python scripts/overlap_probe.py 2>&1 | tail -5
done | tee -a gpurun_out/overlap_probe2.log

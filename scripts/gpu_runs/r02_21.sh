#!/bin/bash
# round 2, call 21: bag kernel A/B: L2::256B prefetch-size hint on the row loads (ab/liblattice_pf256.so)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f gpurun_out/bagab_*.json
for rep in 1 2; do
  for lib in paper_2512_09200_b200/liblattice_b200.so ab/liblattice_pf256.so; do
    tag=$(basename $lib .so)
    LATTICE_LIB=$GRAFT_REPO_ROOT/$lib timeout 600 python bench.py --workload micro --dtype bf16 --steps 200 --cpu-seconds 1 >> gpurun_out/bagab_micro_$tag.json 2>/dev/null
    LATTICE_LIB=$GRAFT_REPO_ROOT/$lib timeout 600 python bench.py --no-micro --cpu-seconds 1 >> gpurun_out/bagab_mid_$tag.json 2>/dev/null
  done
done

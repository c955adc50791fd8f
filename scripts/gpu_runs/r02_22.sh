#!/bin/bash
# round 2, call 22: bag kernel A/B (micro bf16 + f32, 3 reps interleaved): L2::256B prefetch hint
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f gpurun_out/bagab2_*.json
for rep in 1 2 3; do
  for lib in paper_2512_09200_b200/liblattice_b200.so ab/liblattice_pf256.so; do
    tag=$(basename $lib .so)
    for dt in bf16 f32; do
      LATTICE_LIB=$GRAFT_REPO_ROOT/$lib timeout 600 python bench.py --workload micro --dtype $dt --steps 300 --cpu-seconds 1 >> gpurun_out/bagab2_${dt}_$tag.json 2>/dev/null
    done
  done
done

#!/bin/bash
# round 2, call 10: ncu --set full of the v2 large-n FM/LCB kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python scripts/fm_bench.py large > gpurun_out/fm_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fm_lcb_large -s 2 -c 1 \
    -o gpurun_out/fm_large_v2 python scripts/fm_bench.py large > gpurun_out/fm_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/fm_ncu.log

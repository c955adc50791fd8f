B="python bench.py --steps 10 --warmup 3 --cpu-seconds 1"
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', d['value'], d['stages']['embedding'], d['clocks'])"; }
timeout 300 $B > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
LATTICE_PEER_ORDER=1 timeout 300 $B --exchange peer1 > gpurun_out/n1p1.json 2>gpurun_out/n1p1.err; summ gpurun_out/n1p1.json
LATTICE_PEER_ORDER=2 timeout 300 $B --exchange peer1 > gpurun_out/n1p2.json 2>/dev/null; summ gpurun_out/n1p2.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag_n1 $B > /dev/null 2>&1
LATTICE_PEER_ORDER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag_peer1 $B --exchange peer1 > /dev/null 2>&1
ls gpurun_out

B="python bench.py --steps 10 --warmup 3 --cpu-seconds 1"
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), d['roofline']['frac'], d.get('stages',{}).get('embedding'), d['clocks'])"; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 $B > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
timeout 300 $B --exchange peer1 > gpurun_out/n1p.json 2>gpurun_out/n1p.err; summ gpurun_out/n1p.json
LATTICE_BAG_VARIANT=2 timeout 300 $B --exchange peer1 > gpurun_out/n1p2.json 2>/dev/null; summ gpurun_out/n1p2.json
timeout 300 python bench.py --workload micro --dtype bf16 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mb.json 2>/dev/null; summ gpurun_out/mb.json
timeout 300 python bench.py --workload micro --dtype f32 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mf.json 2>/dev/null; summ gpurun_out/mf.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag_n1 $B > gpurun_out/ncu1.log 2>&1; tail -2 gpurun_out/ncu1.log

summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 1 > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 1 --graph > gpurun_out/n1g.json 2>gpurun_out/n1g.err; summ gpurun_out/n1g.json; tail -2 gpurun_out/n1g.err
done

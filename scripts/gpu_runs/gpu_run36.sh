summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['roofline'], d['clocks'])"; }
timeout 600 python -m pytest tests/test_objective_gpu.py -x -q > gpurun_out/pytest_obj.log 2>&1; tail -3 gpurun_out/pytest_obj.log
timeout 300 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/full_n1.json 2>gpurun_out/full_n1.err; summ gpurun_out/full_n1.json; tail -3 gpurun_out/full_n1.err
timeout 300 python bench.py > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json

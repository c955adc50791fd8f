summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), d['ms_per_step'], st.get('embedding',{}).get('ms'), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; }
timeout 900 python -m pytest tests/test_embedding_bag_gpu.py tests/test_network_gpu.py tests/test_dense_gpu.py -x -q > gpurun_out/pytest_bag.log 2>&1; tail -2 gpurun_out/pytest_bag.log
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
timeout 300 python bench.py --workload micro --dtype bf16 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/mb.json 2>/dev/null; summ gpurun_out/mb.json
timeout 300 python bench.py --workload micro --dtype f32 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/mf.json 2>/dev/null; summ gpurun_out/mf.json
timeout 900 ncu --set full --clock-control none -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag_v5 python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > /dev/null 2>&1

summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), d['ms_per_step'], st.get('mlp',{}).get('ms_per_block'), st.get('tower',{}).get('ms'), d['clocks']['sm_mhz'])"; }
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$?; tail -15 gpurun_out/pytest_gemm.log
timeout 300 python -m pytest tests/test_network_gpu.py tests/test_dense_gpu.py -x -q > gpurun_out/pytest_net.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_net.log
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
LATTICE_GEMM_2CTA=0 timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1_off.json 2>/dev/null; summ gpurun_out/n1_off.json

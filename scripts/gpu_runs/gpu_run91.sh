# tower split-K: parity (network tests, full workload towers), then A/B LATTICE_TOWER_KSPLIT=1 vs 3
timeout 400 python -m pytest tests/test_network_gpu.py tests/test_gemm_gpu.py tests/test_dense_gpu.py tests/test_objective_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_ksplit.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ksplit.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d['stages']
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], 'tower', round(st['tower']['ms'],3), d['clocks']['sm_mhz'])"; }
for v in 1 3 1 3; do
  LATTICE_TOWER_KSPLIT=$v timeout 200 python bench.py --steps 40 --warmup 5 --cpu-seconds 0.1 > gpurun_out/mid_ks$v.json 2>/dev/null; summ gpurun_out/mid_ks$v.json
done | tee gpurun_out/ksplit_ab.log
LATTICE_TOWER_KSPLIT=3 timeout 200 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 0.1 > gpurun_out/full_ks3.json 2>/dev/null; summ gpurun_out/full_ks3.json

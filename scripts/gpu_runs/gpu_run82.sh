# programmatic dependent launch across the dense chain: parity, then A/B (LATTICE_PDL=0 vs 1)
timeout 900 python -m pytest tests/test_network_gpu.py tests/test_gemm_gpu.py tests/test_dense_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_pdl.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_pdl.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d['stages']
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], 'dense', round(st['dense_total']['ms'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do
for v in 0 1; do
  LATTICE_PDL=$v timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 0.1 > gpurun_out/mid_pdl$v.json 2>/dev/null; summ gpurun_out/mid_pdl$v.json
done; done | tee gpurun_out/pdl_ab.log

# 32-byte (LDG/STG .256) epilogue accesses in the GEMM and FM/LCB kernels: parity, then A/B vs
# the previous build (ab/base.so) on one box
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_network_gpu.py tests/test_dense_gpu.py -x -q > gpurun_out/pytest_st256.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_st256.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d['stages']
print('$1', round(d['value']), d['ms_per_step'], 'fm', round(st['fm_lcb']['ms_per_block'],3), 'mlp', round(st['mlp']['ms_per_block'],3), 'tower', round(st['tower']['ms'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do
for v in base new; do
  if [ $v = base ]; then export LATTICE_LIB=$PWD/ab/base.so; else unset LATTICE_LIB; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 0.1 > gpurun_out/mid_$v.json 2>/dev/null; summ gpurun_out/mid_$v.json
done; done | tee gpurun_out/st256_ab.log

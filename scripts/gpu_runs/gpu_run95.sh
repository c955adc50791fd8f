# direct bag kernel: 8-bag work claims (half the counter atomics) vs 4, same box
timeout 300 python -m pytest tests/test_embedding_bag_gpu.py -x -q > gpurun_out/pytest_chunk.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_chunk.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$2', round(d['value']), d['ms_per_step'], 'emb', round(d['stages']['embedding']['ms'],3), d['clocks']['sm_mhz'])"; }
for v in base new base new; do
  if [ $v = base ]; then export LATTICE_LIB=$PWD/ab/base.so; else unset LATTICE_LIB; fi
  timeout 200 python bench.py --steps 40 --warmup 5 --cpu-seconds 0.1 > gpurun_out/chunk_$v.json 2>/dev/null; summ gpurun_out/chunk_$v.json $v
done | tee gpurun_out/chunk_ab.log

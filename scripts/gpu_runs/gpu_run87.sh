# N=4 e2e check: PDL on/off, twice
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for v in 1 0 1 0; do
LATTICE_PDL=$v timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$v bench.py --gpus 4 --cpu-seconds 0.1 > gpurun_out/n4_pdl$v.json 2>/dev/null; summ gpurun_out/n4_pdl$v.json
done
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1

summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), d['ms_per_step'], d.get('stages',{}).get('embedding',{}).get('peer_split_ms'), d['clocks']['sm_mhz'])"; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for kv in "1 0" "0 0" "1 2" "0 2" "1 0"; do set -- $kv
LATTICE_BAG_V3=$1 LATTICE_BAG_VARIANT=$2 timeout 400 $TR --master-port 2954$1 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/n4_k$1v$2.json 2> /dev/null; summ gpurun_out/n4_k$1v$2.json
done

TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for dbg in reads stores reads,stores; do
LATTICE_PEER_ORDER=1 LATTICE_PEER_DEBUG=$dbg timeout 400 $TR --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/dbg.json 2> gpurun_out/dbg.err; echo rc=$?
python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/dbg.json') if l.startswith('{')][-1])
print('$dbg', d['value'], d['stages']['embedding']['peer_split_ms'])"
done

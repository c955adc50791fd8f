TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29517 tests/dist_sharded_check.py > gpurun_out/dist2.log 2>&1; echo rc=$?; grep bit-identical gpurun_out/dist2.log
for o in 2 1; do
LATTICE_PEER_ORDER=$o timeout 400 $TR --master-port 2952$o bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_peer_o$o.json 2> gpurun_out/bench_n2_peer_o$o.err; echo rc=$?
python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/bench_n2_peer_o$o.json') if l.startswith('{')][-1])
print('order $o', d['value'], d['ms_per_step'], d['e2e']['value'], d['stages']['embedding'], d['clocks'])"
done

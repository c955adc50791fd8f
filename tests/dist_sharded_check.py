"""Multi-GPU check (torchrun, NCCL): the table-wise sharded embedding path + network forward
must give bit-identical logits to the single-GPU fused path on the same rank-local batch.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/dist_sharded_check.py
Run by tests/test_multi_gpu.py when >= 2 GPUs are visible. Exit code 0 = pass.
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_09200_b200 as L  # noqa: E402
from paper_2512_09200_b200.sharded import ShardedBags  # noqa: E402

CFG = dict(n=64, d=128, blocks=2, nF=32, nL=32, k=16, mlp=[1024, 512, 4096], domains=3, heads=4,
           tower_hidden=256)
ROWS, B = 4000, 600


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, d = CFG["n"], CFG["d"]
    net = L.Network(**CFG, max_batch=B, weight_seed=0x1A79)
    full = torch.empty((n, ROWS, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(full, 0x1A77)
    sb = ShardedBags(n, B, d, world, rank)
    own = full[sb.owned()[0]: sb.owned()[-1] + 1].contiguous()
    # the owned shard generated independently with the global feature index
    own2 = torch.empty_like(own)
    L.fill_tables(own2, 0x1A77, feature_base=sb.owned()[0], rows_total=ROWS)
    assert torch.equal(own, own2)
    off, ids = L.synth_bags(n, B, 40, ROWS, 0x1A78 + rank)
    dom = L.synth_domains(B, CFG["domains"], 0x1A78 + rank)
    fptrs = torch.tensor([t.data_ptr() for t in full.unbind(0)], dtype=torch.int64, device="cuda")
    frows = torch.full((n,), ROWS, dtype=torch.int64, device="cuda")
    ref = net.forward(dom, off, ids, fptrs, frows, torch.bfloat16).clone()
    optrs = torch.tensor([t.data_ptr() for t in own.unbind(0)], dtype=torch.int64, device="cuda")
    orows = torch.full((sb.Fl,), ROWS, dtype=torch.int64, device="cuda")
    pooled = sb.forward_embeddings(off, ids, list(own.unbind(0)), optrs, orows)
    got = net.forward(dom, pooled=pooled, shards=world).clone()
    # static-capacity (sync-free) exchange gives the same result
    cnt, _ = sb.slice_counts(off)
    cap = cnt.max().reshape(1)
    dist.all_reduce(cap, op=dist.ReduceOp.MAX)
    sb.capacity = int(cap.item())
    pooled2 = sb.forward_embeddings(off, ids, list(own.unbind(0)), optrs, orows)
    got2 = net.forward(dom, pooled=pooled2, shards=world)
    torch.cuda.synchronize()
    sb.check_overflow()
    # peer-memory path (IPC over NVLink, one owner kernel, in-kernel barrier flags): the
    # owners write straight into this rank's X0 -> same logits
    from paper_2512_09200_b200.peer import PeerBags
    pb = PeerBags(net, n, B, d, world, rank)
    pb.register(0, off, ids)
    got3 = pb.forward(0, dom, list(own.unbind(0)), optrs, orows).clone()
    # a second batch buffer pair (the e2e double buffer) and repeated steps keep the barrier
    # epochs in lock step
    off_b, ids_b = off.clone(), ids.clone()
    pb.register(1, off_b, ids_b)
    for i in range(3):
        got4 = pb.forward(i % 2, dom, list(own.unbind(0)), optrs, orows)
    torch.cuda.synchronize()
    pb.check()
    ok3 = torch.equal(got3, ref) and torch.equal(got4, ref)
    if not ok3:
        print(f"rank {rank}: peer path mismatch, max |diff| = {(got3 - ref).abs().max().item()}")
    pb.close()
    ok = torch.equal(got, ref) and torch.equal(got2, ref) and ok3
    t = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(f"sharded W={world}: logits bit-identical to the single-GPU path on every rank: {t.item() == 0}")
    dist.destroy_process_group()
    sys.exit(int(t.item() != 0))


if __name__ == "__main__":
    main()

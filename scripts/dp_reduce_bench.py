"""Gradient reduction + SGD of a data-parallel step, two ways, on N GPUs (torchrun):
  nccl: torch.distributed.all_reduce (NCCL over NVLink) of the flat fp32 bucket, divide, then SGD
        and the weight refresh as torch elementwise ops (the library's SGD kernel does the same
        two passes in one);
  peer: barrier -> lattice_peer_reduce_sgd (each rank reduces its 1/N shard from every rank's HBM,
        applies SGD to its master shard and writes the bf16 weight into every rank) -> barrier.
Bucket = the mid config's trained head (towers 4 x 512 x 32768 + heads + the last block's MLP
8192x2048 + 2048x2048 + 2048x16384): 113 M fp32 gradients. Device time per step, max over ranks.
Prints one JSON line on rank 0."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    import paper_2512_09200_b200 as L
    from paper_2512_09200_b200.train import PeerReducer
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    sizes = [4 * 512 * 32768, 4 * 6 * 512, 8192 * 2048, 2048 * 2048, 2048 * 16384]
    n = sum(sizes) + 1
    g = torch.Generator(device="cuda").manual_seed(rank)
    bucket = torch.randn(n, generator=g, device="cuda") * 1e-3
    master = torch.randn(n, generator=torch.Generator(device="cuda").manual_seed(99), device="cuda")
    weights = [torch.empty(k, dtype=torch.bfloat16 if i != 1 else torch.float32, device="cuda")
               for i, k in enumerate(sizes)]

    class Tr:  # the parts of TowerTrainer PeerReducer reads
        pass
    tr = Tr()
    tr.bucket, tr.master = bucket, master
    offs, o = [], 0
    for k in sizes:
        offs.append(o)
        o += k
    tr.segments = lambda: [(offs[i], sizes[i], weights[i].data_ptr(), i != 1) for i in range(len(sizes))]
    peer = PeerReducer(tr, rank, world)

    def nccl_step():
        dist.all_reduce(bucket)
        bucket.div_(world)
        for i, k in enumerate(sizes):  # SGD + weight refresh (torch elementwise, no network here)
            m = master[offs[i]:offs[i] + k]
            m.sub_(bucket[offs[i]:offs[i] + k], alpha=0.01)
            weights[i].copy_(m)

    def peer_step():
        peer.step(0.01)

    res = {}
    for name, fn in (("nccl", nccl_step), ("peer", peer_step)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 10], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t)
    if rank == 0:
        print(json.dumps({"world": world, "gradients": n, "bucket_MB": n * 4 / 1e6, "ms_nccl_allreduce_plus_sgd": res["nccl"],
                          "ms_peer_reduce_sgd": res["peer"]}))
    peer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

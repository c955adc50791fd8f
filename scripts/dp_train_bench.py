"""Data-parallel training step at the mid config on N GPUs (torchrun): every rank runs forward +
routed BCE + backward of the towers and the last block's MLP on its own batch (B = 32768 per GPU),
then the gradient reduction + SGD -- reducer "peer" (lattice_peer_reduce_sgd over NVLink) or
"nccl" (all-reduce + SGD kernels). Device time per step, max over ranks; whole-job samples/s.
Prints one JSON line per reducer on rank 0."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    import paper_2512_09200_b200 as L
    import bench
    from paper_2512_09200_b200.train import TowerTrainer
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    c, B = bench.MID, bench.MID_B
    n, d = c["n"], c["d"]
    tab = torch.empty((n, bench.MID_ROWS, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, bench.SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rows = torch.full((n,), bench.MID_ROWS, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(n, B, bench.MID_MAXLEN, bench.MID_ROWS, bench.SEED_D + rank)
    dom = L.synth_domains(B, c["domains"], bench.SEED_D + rank)
    imp = L.synth_impressions(B, 2, 7 + rank)
    win, lab, _ = L.zipper_assign_labels(*imp, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    for reducer in ("peer", "nccl"):
        net = L.Network(**c, max_batch=B, weight_seed=bench.SEED_W)
        tr = TowerTrainer(net, lr=0.05, train_mlp=True, reducer=reducer)

        def step():
            net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits)
            return tr.step(logits, win, lab, 2, 3)

        losses = [float(step()) for _ in range(2)]
        torch.cuda.synchronize()
        dist.barrier()
        steps = 6
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            loss = step()
            ev[i + 1].record()
        torch.cuda.synchronize()
        per = [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(steps)]
        t = torch.tensor([ev[0].elapsed_time(ev[steps]) / steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        losses.append(float(loss))
        if rank == 0:
            ms = float(t)
            print(json.dumps({"reducer": reducer, "world": world, "ms_per_step": ms, "rank0_steps_ms": per,
                              "training_samples_per_s": world * B / (ms / 1e3), "loss_first_last": [losses[0], losses[-1]]}))
        if tr._peer is not None:
            tr._peer.close()
        del tr, net
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

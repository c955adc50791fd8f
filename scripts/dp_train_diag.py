"""Diagnose the peer reducer inside the training step (N GPUs, torchrun): per-stage device times
(forward, backward, barrier 1, reduce kernel, barrier 2) on every rank. Prints one JSON line per
rank."""
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
    net = L.Network(**c, max_batch=B, weight_seed=bench.SEED_W)
    tr = TowerTrainer(net, lr=0.05, train_mlp=True, reducer="peer")
    pr = tr._peer
    dX = torch.empty((B, n * d), dtype=torch.float32, device="cuda")
    names = ["forward", "backward", "barrier1", "reduce", "barrier2"]
    acc = {k: [] for k in names}
    for it in range(5):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits)
        ev[1].record()
        loss, dl = L.routed_bce(logits, win, lab, 2, 3)
        net.tower_backward(dl, dW1=tr.dW1, dW2=tr.dW2, dX=dX)
        net.mlp_backward(dX, dW=tr.dW_mlp)
        tr.loss_slot.copy_(loss.reshape(1))
        ev[2].record()
        pr.barrier()
        ev[3].record()
        L.peer_reduce_sgd(pr.grad_ptrs, pr.master, pr.segs, pr.n, pr.r, pr.W, 0.05)
        ev[4].record()
        pr.barrier()
        ev[5].record()
        torch.cuda.synchronize()
        if it >= 2:
            for i, k in enumerate(names):
                acc[k].append(round(ev[i].elapsed_time(ev[i + 1]), 3))
    print(json.dumps({"rank": rank, "world": world, **acc, "status": int(pr.status.item())}))
    pr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

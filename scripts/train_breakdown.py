"""Per-stage device times of one mid training step (bench.train_timing's step): forward, routed
BCE, tower backward (with dX), last-block MLP backward, SGD. Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_09200_b200 as L
    import bench
    from paper_2512_09200_b200.train import TowerTrainer
    c, B = bench.MID, bench.MID_B
    n, d = c["n"], c["d"]
    net = L.Network(**c, max_batch=B, weight_seed=bench.SEED_W)
    tab = torch.empty((n, bench.MID_ROWS, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, bench.SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rows = torch.full((n,), bench.MID_ROWS, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(n, B, bench.MID_MAXLEN, bench.MID_ROWS, bench.SEED_D)
    dom = L.synth_domains(B, c["domains"], bench.SEED_D)
    imp = L.synth_impressions(B, 2, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    tr = TowerTrainer(net, lr=0.05, train_mlp=True)
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    dX = torch.empty((B, n * d), dtype=torch.float32, device="cuda")
    names = ["forward", "routed_bce", "tower_backward", "mlp_backward", "sgd"]
    tot = {k: 0.0 for k in names}
    reps = 4
    for rep in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits)
        ev[1].record()
        loss, dl = L.routed_bce(logits, win, lab, 2, 3)
        ev[2].record()
        net.tower_backward(dl, dW1=tr.dW1, dW2=tr.dW2, dX=dX)
        ev[3].record()
        net.mlp_backward(dX, dW=tr.dW_mlp)
        ev[4].record()
        net.tower_sgd(0.05, tr.dW1, tr.dW2, tr.W1, tr.W2)
        for i, (g, w) in enumerate(zip(tr.dW_mlp, tr.mlp)):
            net.weight_sgd(c["blocks"] - 1, 3, i, 0.05, g, w)
        ev[5].record()
        torch.cuda.synchronize()
        if rep:
            for i, k in enumerate(names):
                tot[k] += ev[i].elapsed_time(ev[i + 1]) / reps
    print(json.dumps({k: round(v, 3) for k, v in tot.items()}))


if __name__ == "__main__":
    main()

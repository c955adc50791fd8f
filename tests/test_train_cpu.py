"""Host logic of the data-parallel tower training step (paper_2512_09200_b200/train.py) on the CPU
with gloo at world sizes 2 and 4: the library calls (routed BCE, tower backward, SGD) are replaced
by torch stand-ins with the same contracts. Checks: one collective over the flat gradient bucket,
gradients and loss averaged over ranks, every rank applying the identical update (replicas stay
bit-identical), and world size 1 skipping the collective."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_09200_b200.train import TowerTrainer


class FakeNet:
    def __init__(self, G=3, th=8, n=2, d=4, heads=2):
        self.cfg = dict(domains=G, tower_hidden=th, n=n, d=d, heads=heads, blocks=2, mlp=[6, 10, 8])

    def mlp_masters(self):
        g = torch.Generator().manual_seed(1)
        w = self.cfg["mlp"]
        return [torch.randn((w[i + 1], w[i]), generator=g) for i in range(len(w) - 1)]

    def tower_masters(self):
        c = self.cfg
        g = torch.Generator().manual_seed(0)  # every rank starts from the same weights
        return (torch.randn((c["domains"], c["tower_hidden"], c["n"] * c["d"]), generator=g),
                torch.randn((c["domains"], c["heads"], c["tower_hidden"]), generator=g))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, train_mlp):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    net = FakeNet()
    W1_0, W2_0 = net.tower_masters()
    M_0 = net.mlp_masters()

    def allreduce(t):
        calls.append(t.numel())
        dist.all_reduce(t)

    def loss_fn(logits, window, labels, tasks, windows):
        return torch.tensor(float(rank + 1), dtype=torch.float64), logits * 0 + rank

    def backward(dlogits, dW1, dW2, *dW_mlp):  # rank-dependent gradients
        dW1.fill_(float(rank))
        dW2.fill_(float(2 * rank))
        for i, g in enumerate(dW_mlp):
            g.fill_(float((3 + i) * rank))

    def mlp_sgd(lr, i, g, W):
        W.sub_(lr * g)

    def sgd(lr, dW1, dW2, W1, W2):
        W1.sub_(lr * dW1)
        W2.sub_(lr * dW2)

    tr = TowerTrainer(net, lr=0.5, allreduce=allreduce, backward=backward, sgd=sgd, loss_fn=loss_fn,
                      train_mlp=train_mlp, mlp_sgd=mlp_sgd)
    logits = torch.zeros((4, 2))
    loss = tr.step(logits, None, None, 1, 2)
    mean_rank = (world - 1) / 2
    ok = (len(calls) == 1 and calls[0] == tr.bucket.numel()
          and abs(float(loss) - (mean_rank + 1)) < 1e-6
          and torch.allclose(tr.W1, W1_0 - 0.5 * mean_rank)
          and torch.allclose(tr.W2, W2_0 - 0.5 * 2 * mean_rank)
          and len(tr.mlp) == (2 if train_mlp else 0)
          and all(torch.allclose(w, M_0[i] - 0.5 * (3 + i) * mean_rank) for i, w in enumerate(tr.mlp)))
    # replicas identical: compare a checksum of the updated masters across ranks
    cs = torch.tensor([float(tr.W1.double().sum()), float(tr.W2.double().sum())] +
                      [float(w.double().sum()) for w in tr.mlp], dtype=torch.float64)
    allcs = [torch.zeros_like(cs) for _ in range(world)]
    dist.all_gather(allcs, cs)
    ok = ok and all(torch.equal(c, allcs[0]) for c in allcs)
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,train_mlp", [(2, False), (4, False), (2, True)])
def test_dp_tower_step_gloo(world, train_mlp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, train_mlp)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_single_process_skips_collective():
    calls = []
    net = FakeNet()
    W1_0, _ = net.tower_masters()
    tr = TowerTrainer(net, lr=1.0, allreduce=lambda t: calls.append(1),
                      backward=lambda dl, a, b: (a.fill_(1.0), b.fill_(0.0)),
                      sgd=lambda lr, a, b, W1, W2: (W1.sub_(lr * a), W2.sub_(lr * b)),
                      loss_fn=lambda *a: (torch.tensor(0.25, dtype=torch.float64), torch.zeros((2, 2))))
    loss = tr.step(torch.zeros((2, 2)), None, None, 1, 2)
    assert not calls and float(loss) == 0.25 and torch.allclose(tr.W1, W1_0 - 1.0)

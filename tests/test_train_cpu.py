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


MAPPED = 1 << 40


class FakePeerOps:
    """IPC / barrier / reduce kernel stand-ins recording the calls (the real ones run in
    tests/dist_train_check.py on >= 2 GPUs)."""
    BF16, F32 = 1, 0

    def __init__(self, rank):
        self.rank, self.log = rank, []

    def ipc_handle(self, ptr):
        return (int(ptr).to_bytes(8, "little") + bytes([self.rank]) * 56, 0)

    def ipc_open(self, h, off):
        assert h[8] != self.rank
        return int.from_bytes(h[:8], "little") + off + MAPPED

    def ipc_close(self, p):
        pass

    def peer_barrier(self, flags, rank, world, status, timeout_s, stream=None):
        self.log.append(("barrier",))

    def peer_reduce_sgd(self, grads, masters, segs, n, rank, world, lr, stream=None):
        self.log.append(("reduce", grads.tolist(), masters.data_ptr(),
                         [(o, c, m, dt, d.tolist()) for o, c, m, dt, d in segs], n, rank, world, lr))


class FakeWeightNet(FakeNet):
    def __init__(self, rank):
        super().__init__()
        self.cfg["dtype"] = "bf16"
        self.rank = rank

    def weight_ptr(self, block, kind, index=0):
        return 10_000 * (self.rank + 1) + 100 * kind + 10 * block + index


def _peer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ops = FakePeerOps(rank)
    net = FakeWeightNet(rank)
    tr = TowerTrainer(net, lr=0.25, backward=lambda *a: None, loss_fn=lambda *a: (torch.tensor(0.5), torch.zeros(2)),
                      train_mlp=True, reducer="peer", peer_ops=ops)
    tr.step(torch.zeros((2, 2)), None, None, 1, 2)
    kinds = [e[0] for e in ops.log]
    _, grads, masters, segs, n, r, w, lr = ops.log[1]
    sizes = [tr.W1.numel(), tr.W2.numel()] + [m.numel() for m in tr.mlp]

    def own_at_rank(ptrs, base):  # own pointer unmapped, peers' mapped
        return ptrs[rank] == base and all(p >= MAPPED for i, p in enumerate(ptrs) if i != rank)

    ok = (kinds == ["barrier", "reduce", "barrier"] and n == tr.bucket.numel() and (r, w, lr) == (rank, world, 0.25)
          and own_at_rank(grads, tr.bucket.data_ptr()) and masters == tr.master.data_ptr()
          and [s[1] for s in segs] == sizes + [1]
          and [s[0] for s in segs] == tr.offsets + [n - 1]
          and [s[2] for s in segs] == [0] * len(sizes) + [1]                 # sgd ..., loss: mean
          and [s[3] for s in segs] == [1, 0, 1, 1, 0]                        # bf16 W1, fp32 W2, bf16 MLP, fp32 loss
          and own_at_rank(segs[0][4], net.weight_ptr(0, 4)) and own_at_rank(segs[2][4], net.weight_ptr(1, 3, 0))
          and torch.equal(tr.W1, net.tower_masters()[0]) and torch.equal(tr.mlp[1], net.mlp_masters()[1]))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_reducer_host_logic(world):
    """TowerTrainer(reducer="peer"): exports bucket / every trained weight / loss (masters stay local), one
    barrier -> lattice_peer_reduce_sgd -> barrier per step, segments in bucket order (sgd for the
    weights in their storage dtype, mean for the loss)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res

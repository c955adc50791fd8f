"""Data-parallel training step of the untied per-domain towers -- and optionally the last DWFB
block's MLP -- (SURVEY.md 8f rank 4).

The reference defines no training step; its only pinned piece of a backward
pass is the activation derivative (swish_rn_jvp, numerics.hpp:113-136). This module composes the
library's backward entries into one step of the consolidated model's trainable head, run
data-parallel (one process per GPU):

  1. forward (lattice_net_forward) -> logits [B, O*W]
  2. window-routed BCE (lattice_routed_bce): each sample trains only its Zipper-assigned window's
     head per objective -> loss, dlogits
  3. lattice_net_tower_backward -> dW1 [G, th, n*d], dW2 [G, heads, th], written straight into one
     flat fp32 bucket
  4. gradient all-reduce over the data-parallel group: ONE collective on the bucket (NCCL over
     NVLink on GPUs), averaged; the loss is averaged too
  5. lattice_net_tower_sgd: fp32 masters -= lr * grad, the network's bf16 copies refreshed

With train_mlp=True the towers' backward also returns dX_L, lattice_net_mlp_backward carries it
through the last block's residual rms_norm_d and MLP, the MLP gradients join the
same bucket (still one collective) and lattice_net_weight_sgd updates those weights too.

With reducer="peer" steps 4-5 become ONE kernel over peer memory (lattice_peer_reduce_sgd,
PeerReducer below): rank r owns 1/W of the flat gradient bucket, sums every rank's gradients for
it in rank order straight from their HBM over NVLink, applies SGD to its shard of the fp32
masters (ZeRO-1: tr.master is current on the owned shard only) and writes the new weight into
every rank's network -- reduce-scatter, optimizer and all-gather fused, between two device-side
barriers, with no NCCL call and no host synchronisation.

Gradients are deterministic (fixed-order reductions in the library), so replicas that start equal
stay bit-identical. `allreduce` is injectable so the host logic is tested with gloo on the CPU
(tests/test_train_cpu.py).
"""
import torch
import torch.distributed as dist


class TowerTrainer:
    def __init__(self, net, lr, group=None, allreduce=None, backward=None, sgd=None, loss_fn=None,
                 train_mlp=False, mlp_sgd=None, reducer="auto", peer_ops=None):
        """net: paper_2512_09200_b200.Network (or a stand-in exposing cfg / tower_masters /
        mlp_masters). allreduce(tensor) sums in place across the group (default:
        torch.distributed.all_reduce when initialised with world > 1); backward(dlogits, dW1, dW2,
        *dW_mlp) / sgd(lr, dW1, dW2, W1, W2) / mlp_sgd(lr, layer, dW, W) / loss_fn replace the
        library calls (CPU tests of the host logic). reducer: "peer" (the fused peer-memory
        kernel), "nccl" (all-reduce + SGD kernel) or "auto" (peer when every rank's GPU is on this
        node and no allreduce is injected, else nccl)."""
        self.net, self.lr, self.group = net, lr, group
        c = net.cfg
        self.G, self.th, self.nd, self.heads = c["domains"], c["tower_hidden"], c["n"] * c["d"], c["heads"]
        W1, W2 = net.tower_masters()
        self.train_mlp = train_mlp
        mlp = net.mlp_masters() if train_mlp else []
        dev = W1.device
        shapes = [W1.shape, W2.shape] + [w.shape for w in mlp]
        sizes = [W1.numel(), W2.numel()] + [w.numel() for w in mlp]
        n = sum(sizes)
        # one flat bucket (the backward writes every gradient into it, one collective reduces all)
        # and one flat fp32 master buffer with the same layout; the last slot carries the loss
        self.bucket = torch.empty(n + 1, dtype=torch.float32, device=dev)
        self.master = torch.zeros(n + 1, dtype=torch.float32, device=dev)
        grads, masters, self.offsets, o = [], [], [], 0
        for shp, k, init in zip(shapes, sizes, [W1, W2] + mlp):
            grads.append(self.bucket[o:o + k].view(shp))
            masters.append(self.master[o:o + k].view(shp))
            masters[-1].copy_(init)
            self.offsets.append(o)
            o += k
        self.dW1, self.dW2, self.dW_mlp = grads[0], grads[1], grads[2:]
        self.W1, self.W2, self.mlp = masters[0], masters[1], masters[2:]
        self.loss_slot = self.bucket[o:]
        self._dX = None
        self._allreduce = allreduce
        self._backward = backward
        self._sgd = sgd
        self._mlp_sgd = mlp_sgd
        self._loss_fn = loss_fn
        self._peer = None
        if reducer not in ("nccl", "peer", "auto"):
            raise ValueError("reducer must be 'nccl', 'peer' or 'auto'")
        if reducer == "auto":
            single_node = (torch.cuda.is_available() and dev.type == "cuda" and
                           self.world() <= torch.cuda.device_count())
            reducer = "peer" if single_node and allreduce is None and backward is None else "nccl"
        if reducer == "peer" and self.world() > 1:
            self._peer = PeerReducer(self, dist.get_rank(group), self.world(), group=group, ops=peer_ops)

    def segments(self):
        """(offset, count, weight pointer, bf16) of every trained weight in the flat buffers."""
        c = self.net.cfg
        bf16 = c.get("dtype", "bf16") not in ("f32", "fp32", "float32")
        segs = [(self.offsets[0], self.W1.numel(), self.net.weight_ptr(0, 4, 0), bf16),
                (self.offsets[1], self.W2.numel(), self.net.weight_ptr(0, 5, 0), False)]
        for i, w in enumerate(self.mlp):
            segs.append((self.offsets[2 + i], w.numel(), self.net.weight_ptr(c["blocks"] - 1, 3, i), bf16))
        return segs

    def world(self):
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def reduce(self, world):
        if world == 1:
            return
        if self._allreduce is not None:
            self._allreduce(self.bucket)
        else:
            dist.all_reduce(self.bucket, op=dist.ReduceOp.SUM, group=self.group)
        self.bucket.div_(world)

    def step(self, logits, window, labels, tasks, windows, stream=None):
        """One optimizer step after a forward that produced `logits` [B, tasks*windows]; returns the
        data-parallel mean loss (a device fp32 scalar, no host synchronisation)."""
        if self._loss_fn is not None:
            loss, dlogits = self._loss_fn(logits, window, labels, tasks, windows)
        else:
            import paper_2512_09200_b200 as L
            loss, dlogits = L.routed_bce(logits, window, labels, tasks, windows, stream=stream)
        if self._backward is not None:
            self._backward(dlogits, self.dW1, self.dW2, *self.dW_mlp)
        elif self.train_mlp:
            B = dlogits.shape[0]
            if self._dX is None or self._dX.shape[0] < B:
                self._dX = torch.empty((B, self.nd), dtype=torch.float32, device=dlogits.device)
            dX = self._dX[:B]
            self.net.tower_backward(dlogits, dW1=self.dW1, dW2=self.dW2, dX=dX, stream=stream)
            self.net.mlp_backward(dX, dW=self.dW_mlp, stream=stream)
        else:
            self.net.tower_backward(dlogits, dW1=self.dW1, dW2=self.dW2, stream=stream)
        self.loss_slot.copy_(loss.reshape(1))
        if self._peer is not None:  # reduce-scatter + SGD + all-gather in one peer-memory kernel
            return self._peer.step(self.lr, stream=stream)
        self.reduce(self.world())
        if self._sgd is not None:
            self._sgd(self.lr, self.dW1, self.dW2, self.W1, self.W2)
        else:
            self.net.tower_sgd(self.lr, self.dW1, self.dW2, self.W1, self.W2, stream=stream)
        for i, (g, w) in enumerate(zip(self.dW_mlp, self.mlp)):
            if self._mlp_sgd is not None:
                self._mlp_sgd(self.lr, i, g, w)
            else:
                self.net.weight_sgd(self.net.cfg["blocks"] - 1, 3, i, self.lr, g, w, stream=stream)
        return self.loss_slot[0]


class PeerReducer:
    """Data-parallel reduction + SGD over peer memory for a TowerTrainer (module docstring). At
    setup every rank exports, through CUDA IPC, its gradient bucket, every trained weight buffer
    of its network, a loss output and a barrier flag array; a step is barrier ->
    lattice_peer_reduce_sgd -> barrier, all stream-ordered."""

    def __init__(self, tr, rank, world, group=None, timeout_s=30.0, ops=None):
        if ops is None:
            import paper_2512_09200_b200 as ops
        self.ops, self.r, self.W, self.group, self.timeout_s = ops, rank, world, group, timeout_s
        self._opened = []
        dev = tr.bucket.device
        self.flags = torch.zeros(world + 1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.loss_out = torch.zeros(1, dtype=torch.float32, device=dev)
        self.flag_ptrs = self.share(self.flags.data_ptr(), dev)
        self.grad_ptrs = self.share(tr.bucket.data_ptr(), dev)
        self.master = tr.master
        self.n = tr.bucket.numel()
        self.segs = [(off, cnt, 0, ops.BF16 if bf16 else ops.F32, self.share(ptr, dev))
                     for off, cnt, ptr, bf16 in tr.segments()]
        self.segs.append((self.n - 1, 1, 1, ops.F32, self.share(self.loss_out.data_ptr(), dev)))

    def share(self, ptr, dev):
        """Collective: int64 tensor [W] of every rank's pointer (peers' mapped through IPC)."""
        mine = self.ops.ipc_handle(ptr)
        allh = [None] * self.W
        dist.all_gather_object(allh, mine, group=self.group)
        ptrs = []
        for q, (h, off) in enumerate(allh):
            if q == self.r:
                ptrs.append(int(ptr))
            else:
                p = self.ops.ipc_open(h, off)
                self._opened.append(p)
                ptrs.append(int(p))
        return torch.tensor(ptrs, dtype=torch.int64, device=dev)

    def barrier(self, stream=None):
        self.ops.peer_barrier(self.flag_ptrs, self.r, self.W, self.status, self.timeout_s, stream=stream)

    def step(self, lr, stream=None):
        """Every rank's gradients published -> reduce + SGD of this rank's shard into every rank
        -> all copies written. Returns the mean loss (device scalar)."""
        self.barrier(stream)
        self.ops.peer_reduce_sgd(self.grad_ptrs, self.master, self.segs, self.n, self.r, self.W, lr,
                                 stream=stream)
        self.barrier(stream)
        return self.loss_out[0]

    def close(self):
        for p in self._opened:
            try:
                self.ops.ipc_close(p)
            except Exception:
                pass
        self._opened = []

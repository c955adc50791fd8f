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

Gradients are deterministic (fixed-order reductions in the library), so replicas that start equal
stay bit-identical. `allreduce` is injectable so the host logic is tested with gloo on the CPU
(tests/test_train_cpu.py).
"""
import torch
import torch.distributed as dist


class TowerTrainer:
    def __init__(self, net, lr, group=None, allreduce=None, backward=None, sgd=None, loss_fn=None,
                 train_mlp=False, mlp_sgd=None):
        """net: paper_2512_09200_b200.Network (or a stand-in exposing cfg / tower_masters /
        mlp_masters). allreduce(tensor) sums in place across the group (default:
        torch.distributed.all_reduce when initialised with world > 1); backward(dlogits, dW1, dW2,
        *dW_mlp) / sgd(lr, dW1, dW2, W1, W2) / mlp_sgd(lr, layer, dW, W) / loss_fn replace the
        library calls (CPU tests of the host logic)."""
        self.net, self.lr, self.group = net, lr, group
        c = net.cfg
        self.G, self.th, self.nd, self.heads = c["domains"], c["tower_hidden"], c["n"] * c["d"], c["heads"]
        self.W1, self.W2 = net.tower_masters()
        self.train_mlp = train_mlp
        self.mlp = net.mlp_masters() if train_mlp else []  # fp32 masters [out, in] of the last block
        dev = self.W1.device
        n1, n2 = self.W1.numel(), self.W2.numel()
        nm = sum(w.numel() for w in self.mlp)
        # one flat bucket: the backward writes every gradient into it, one collective reduces all
        self.bucket = torch.empty(n1 + n2 + nm + 1, dtype=torch.float32, device=dev)
        self.dW1 = self.bucket[:n1].view(self.G, self.th, self.nd)
        self.dW2 = self.bucket[n1:n1 + n2].view(self.G, self.heads, self.th)
        self.dW_mlp, o = [], n1 + n2
        for w in self.mlp:
            self.dW_mlp.append(self.bucket[o:o + w.numel()].view(w.shape))
            o += w.numel()
        self.loss_slot = self.bucket[o:]
        self._dX = None
        self._allreduce = allreduce
        self._backward = backward
        self._sgd = sgd
        self._mlp_sgd = mlp_sgd
        self._loss_fn = loss_fn

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

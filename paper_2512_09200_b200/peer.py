"""Table-wise sharded embedding stage over peer memory (NVLink / NVSwitch), one kernel per
owner and no NCCL call on the data path (the "stretch" design: "K1 writes
pooled rows straight into peers' receive buffers through P2P-mapped memory").

Rank o owns the contiguous feature block [o*F/W, (o+1)*F/W) (as in sharded.py). At setup every
rank exports, through CUDA IPC, the buffers its peers touch:

  * its network's X0 ([B][n][d], domain-sorted rows) and sample_pos ([B]) -- written / read
    by every owner;
  * the CSR offsets / ids of each input batch buffer it will use -- read by every owner;
  * a flags array of W+1 words for the cross-GPU barrier.

One step on rank r (everything stream-ordered, no host synchronisation):

  1. lattice_net_bucket: sample_pos of r's batch;
  2. barrier: r's offsets / ids / sample_pos are published and r's X0 is free;
  3. lattice_peer_embedding_bag: for every source s, pool r's tables over s's bags (offsets and
     ids read from s's HBM over NVLink, rows from local HBM) and store the normalised rows
     into s's X0 at sample_pos[s][b] (NVLink stores);
  4. barrier: every owner has finished writing r's X0;
  5. the dense forward in place (lattice_net_forward, pooled_layout 2).

Compared with sharded.py's ids all-to-all -> pool -> pooled all-to-all -> shard gather, this
removes the lengths exchange and scan, the ids pack, the pooled staging write and read, and
the X0 scatter pass; the only NVLink traffic is the ids read and the pooled-row stores, and it
overlaps the local HBM gathers inside one kernel.

`ops` is injectable so the handle-exchange logic runs under gloo on CPU
(tests/test_peer_cpu.py); on GPUs it is this package's ctypes binding.
"""

import torch
import torch.distributed as dist


class PeerBags:
    def __init__(self, net, n_features, batch, dim, world, rank, group=None, timeout_s=30.0, ops=None,
                 device="cuda", row_stride=None):
        """n_features: table-pooled embeddings (sharded); row_stride: elements per X0 row
        (n * d when the network also has dense embeddings after the pooled ones)."""
        if n_features % world:
            raise ValueError("table-wise sharding needs the feature count divisible by the world size")
        if ops is None:
            import paper_2512_09200_b200 as ops
        self.ops = ops
        self.net = net
        self.F, self.B, self.D, self.W, self.r = n_features, batch, dim, world, rank
        self.Fl = n_features // world
        self.row_stride = row_stride or n_features * dim
        self.group = group
        self.timeout_s = timeout_s
        self.device = device
        self._opened = []
        self.flags = torch.zeros(world + 1, dtype=torch.int32, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.flag_ptrs = self.share(self.flags.data_ptr())
        self.out_ptrs = self.share(net.buffer(0))
        self.pos_ptrs = self.share(net.buffer(1))
        self.batches = {}

    def owned(self):
        return range(self.r * self.Fl, (self.r + 1) * self.Fl)

    def share(self, ptr):
        """Collective: every rank exports `ptr`; returns an int64 tensor [W] of device pointers
        (own pointer at [rank], peers' mapped through IPC)."""
        if self.W == 1:  # single rank: nothing to map
            return torch.tensor([int(ptr)], dtype=torch.int64, device=self.device)
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
        return torch.tensor(ptrs, dtype=torch.int64, device=self.device)

    def register(self, key, offsets, ids):
        """Collective: publish an input batch buffer pair (feature-major CSR over all n
        features of this rank's batch) under `key`; the tensors must stay alive."""
        self.batches[key] = (self.share(offsets.data_ptr()), self.share(ids.data_ptr()), offsets, ids)

    def barrier(self, stream=None):
        self.ops.peer_barrier(self.flag_ptrs, self.r, self.W, self.status, self.timeout_s, stream=stream)

    def pool(self, key, tables, table_ptrs, rows, stream=None):
        off_ptrs, ids_ptrs, _, _ = self.batches[key]
        pos_ptrs, out_ptrs = self.pos_ptrs, self.out_ptrs
        self.ops.peer_embedding_bag(self.r, self.W, tables, table_ptrs, rows, self.r * self.Fl, self.B,
                                    off_ptrs, ids_ptrs, pos_ptrs, out_ptrs, self.row_stride,
                                    normalize=True, stream=stream)

    def forward(self, key, domain, tables, table_ptrs, rows, logits=None, stream=None, dense=None):
        """Steps 1-5 of the module docstring: logits of this rank's batch."""
        self.net.bucket(domain, stream=stream)
        self.barrier(stream)
        self.pool(key, tables, table_ptrs, rows, stream)
        self.barrier(stream)
        return self.net.forward_in_place(domain, logits=logits, stream=stream, dense=dense)

    def forward_embeddings(self, key, domain, tables, table_ptrs, rows, stream=None, timed=False):
        """Steps 1-4 only (the embedding stage). timed: CUDA events between the sub-steps,
        read with stage_ms() -> [bucket, barrier 1, owner kernel, barrier 2] in ms."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timed else None
        s = stream if stream is not None else torch.cuda.current_stream()
        mark = (lambda i: ev[i].record(s)) if timed else (lambda i: None)
        mark(0)
        self.net.bucket(domain, stream=stream)
        mark(1)
        self.barrier(stream)
        mark(2)
        self.pool(key, tables, table_ptrs, rows, stream)
        mark(3)
        self.barrier(stream)
        mark(4)
        self._ev = ev

    def stage_ms(self):
        ev = self._ev
        ev[-1].synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)]

    def check(self):
        """Raise if a barrier timed out (a peer never arrived). Synchronises."""
        if int(self.status.item()) != 0:
            raise RuntimeError("peer barrier timed out: a rank did not arrive")

    def close(self):
        for p in self._opened:
            try:
                self.ops.ipc_close(p)
            except Exception:
                pass
        self._opened = []

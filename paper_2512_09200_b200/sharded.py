"""Table-wise sharded embedding bags across ranks ("TorchRec ...
embedding table sharding").

Rank o owns the contiguous feature block [o*F/W, (o+1)*F/W). One step:

  1. ids all-to-all (input dist): every rank sends owner o the CSR slice of o's features over
     its local batch -- bag lengths (fixed F/W*B per peer) and the ids they cover.
  2. owners pool: lattice_embedding_bag with sources = W over bags laid out [src][f_local][b],
     rms-normalised, bf16, written as [W*B][F/W][D] = the send buffer of step 3.
  3. pooled all-to-all (output dist): rank r receives [W][B][F/W][D] -> lattice_net_forward with
     pooled_layout = 1 scatters it into the network's domain-sorted X0.

With a static `capacity` (ids per source->owner slice; the paper's "pre-allocated static GPU
storage") the ids exchange is sync-free: lattice_pack_slices copies each
slice into a fixed [W][capacity] buffer with sizes read on the device, the buffers are
exchanged with equal splits, and the owner's bag kernel reads the received slices in place
(slice_cap), rebasing the global CSR offsets per source. Without a capacity the split sizes
are read back to the host each step.

The dense part is replicated (forward only: the reference has no backward, so there is no
gradient allreduce). `pool_fn` / `scan_fn` / `pack_fn` are injectable so the exchange logic
is tested with gloo on CPU (tests/test_sharded_cpu.py); on GPUs they are the CUDA kernels.
"""
import torch
import torch.distributed as dist


class ShardedBags:
    def __init__(self, n_features, batch, dim, world, rank, group=None, capacity=None):
        if n_features % world:
            raise ValueError("table-wise sharding needs the feature count divisible by the world size")
        self.F, self.B, self.D, self.W, self.r = n_features, batch, dim, world, rank
        self.Fl = n_features // world
        self.group = group
        self.capacity = capacity
        self._overflow = None
        self._send = None
        self._recv = None

    def owned(self):
        return range(self.r * self.Fl, (self.r + 1) * self.Fl)

    def slice_bounds(self, offsets):
        """ids [bounds[o], bounds[o+1]) of the local batch belong to owner o (device int64)."""
        return offsets[torch.arange(self.W + 1, device=offsets.device) * (self.Fl * self.B)]

    def slice_counts(self, offsets):
        b = self.slice_bounds(offsets)
        return b[1:] - b[:-1], b

    def check_overflow(self):
        if self._overflow is not None and int(self._overflow.item()) != 0:
            raise RuntimeError("sharded ids exchange: a slice exceeded the static capacity")

    def _lengths(self, offsets, scan_fn):
        W, Fl, B = self.W, self.Fl, self.B
        lengths = (offsets[1:] - offsets[:-1]).to(torch.int32)
        recv_len = torch.empty(W * Fl * B, dtype=torch.int32, device=offsets.device)
        dist.all_to_all_single(recv_len, lengths, group=self.group)
        if scan_fn is None:
            import paper_2512_09200_b200 as L
            return L.lengths_to_offsets(recv_len)
        return scan_fn(recv_len)

    # ---- 1. input dist ------------------------------------------------------------------
    def exchange_ids(self, offsets, ids, scan_fn=None, pack_fn=None):
        """-> (recv_offsets int64 [W*Fl*B+1] over bags [src][f_local][b], recv_ids int32,
        slice_cap: 0 for a compact CSR, else source r's ids start at r*slice_cap)."""
        W = self.W
        dev = offsets.device
        recv_off = self._lengths(offsets, scan_fn)
        counts, bounds = self.slice_counts(offsets)
        if self.capacity:
            cap = self.capacity
            if self._send is None or self._send.shape != (W, cap) or self._send.device != dev:
                self._send = torch.empty((W, cap), dtype=torch.int32, device=dev)
                self._recv = torch.empty((W, cap), dtype=torch.int32, device=dev)
                self._overflow = torch.zeros(1, dtype=torch.int32, device=dev)
            if pack_fn is None:
                import paper_2512_09200_b200 as L
                L.pack_slices(bounds, ids, cap, self._send, self._overflow)
            else:
                pack_fn(bounds, ids, cap, self._send, self._overflow)
            dist.all_to_all_single(self._recv.view(-1), self._send.view(-1), group=self.group)
            return recv_off, self._recv.view(-1), cap
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        sizes = torch.cat([counts, recv_counts]).tolist()  # host sync: split sizes
        sc, rc = sizes[:W], sizes[W:]
        recv_ids = torch.empty(max(sum(rc), 1), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_ids[:sum(rc)], ids[:sum(sc)], rc, sc, group=self.group)
        return recv_off, recv_ids, 0

    # ---- 2. owner pooling ---------------------------------------------------------------------
    def pool(self, recv_off, recv_ids, slice_cap=0, tables=None, table_ptrs=None, rows=None, out=None,
             pool_fn=None):
        """-> send buffer [W*B][Fl][D] bf16, rms-normalised (the fused K1 epilogue)."""
        if pool_fn is not None:
            return pool_fn(recv_off, recv_ids, slice_cap)
        import paper_2512_09200_b200 as L
        return L.embedding_bag(tables, recv_off, recv_ids, self.B, out=out, out_dtype=torch.bfloat16,
                               normalize=True, check_errors=False, table_ptrs=table_ptrs, rows=rows,
                               sources=self.W, slice_cap=slice_cap)

    # ---- 3. output dist -------------------------------------------------------------------------
    def exchange_pooled(self, send, recv=None):
        """[W*B][Fl][D] (rows r*B.. go to rank r) -> [W][B][Fl][D] (block o from owner o)."""
        if recv is None:
            recv = torch.empty_like(send)
        dist.all_to_all_single(recv.view(-1), send.view(-1), group=self.group)
        return recv

    def forward_embeddings(self, offsets, ids, tables, table_ptrs, rows, send=None, recv=None,
                           check_errors=False):
        """check_errors: synchronise after the ids exchange and raise if a slice exceeded the
        static capacity (the owners then pool only the ids that fit: truncation, never a read
        outside the slice). Unchecked (graphs, pipelines): call check_overflow() later."""
        recv_off, recv_ids, cap = self.exchange_ids(offsets, ids)
        if check_errors:
            self.check_overflow()
        send = self.pool(recv_off, recv_ids, cap, tables, table_ptrs, rows, out=send)
        return self.exchange_pooled(send, recv)

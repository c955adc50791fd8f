"""Table-wise sharded embedding bags across ranks ("TorchRec ...
embedding table sharding").

Rank o owns the contiguous feature block [o*F/W, (o+1)*F/W). One step:

  1. ids all-to-all (input dist): every rank sends owner o the CSR slice of o's features over
     its local batch -- bag lengths (fixed F/W*B per peer) and the ids they cover (variable).
  2. owners pool: lattice_embedding_bag with sources = W over bags laid out [src][f_local][b],
     rms-normalised, bf16, written as [W*B][F/W][D] = the send buffer of step 3.
  3. pooled all-to-all (output dist): rank r receives [W][B][F/W][D] -> lattice_net_forward with
     pooled_layout = 1 scatters it into the network's domain-sorted X0.

The dense part is replicated (forward only: the reference has no backward, so there is no
gradient allreduce). `pool_fn` / `scan_fn` are injectable so the exchange logic is tested
with gloo on CPU (tests/test_sharded_cpu.py); on GPUs they default to the CUDA kernels.
"""
import torch
import torch.distributed as dist


class ShardedBags:
    def __init__(self, n_features, batch, dim, world, rank, group=None, capacity=None):
        """capacity: ids per (source, owner) slice of the static exchange buffers. With a
        capacity the ids all-to-all needs no host synchronisation (fixed-size slices, device-side
        compaction); without one, split sizes are read back each step."""
        if n_features % world:
            raise ValueError("table-wise sharding needs the feature count divisible by the world size")
        self.F, self.B, self.D, self.W, self.r = n_features, batch, dim, world, rank
        self.Fl = n_features // world
        self.group = group
        self.capacity = capacity
        self.overflow = None

    def owned(self):
        return range(self.r * self.Fl, (self.r + 1) * self.Fl)

    def slice_counts(self, offsets):
        """ids this rank sends to each owner (device int64 [W])."""
        W, Fl, B = self.W, self.Fl, self.B
        bounds = offsets[torch.arange(W + 1, device=offsets.device) * (Fl * B)]
        return bounds[1:] - bounds[:-1], bounds

    def check_overflow(self):
        if self.overflow is not None and bool(self.overflow.item()):
            raise RuntimeError("sharded ids exchange: a slice exceeded the static capacity")

    # ---- 1. input dist ------------------------------------------------------------------
    def exchange_ids(self, offsets, ids, scan_fn=None):
        """offsets int64 [F*B+1] (local batch, feature-major), ids int32 -> (recv_offsets int64
        [W*Fl*B+1] over bags [src][f_local][b], recv_ids int32)."""
        if self.capacity:
            return self._exchange_ids_static(offsets, ids, scan_fn)
        W, Fl, B = self.W, self.Fl, self.B
        dev = offsets.device
        lengths = (offsets[1:] - offsets[:-1]).to(torch.int32)
        recv_len = torch.empty(W * Fl * B, dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_len, lengths, group=self.group)
        bounds = offsets[torch.arange(W + 1, device=dev) * (Fl * B)]
        send_counts = (bounds[1:] - bounds[:-1]).to(torch.int64)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        counts = torch.cat([send_counts, recv_counts]).tolist()  # one host sync: split sizes
        sc, rc = counts[:W], counts[W:]
        recv_ids = torch.empty(max(sum(rc), 1), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_ids[:sum(rc)], ids[:sum(sc)], rc, sc, group=self.group)
        if scan_fn is None:
            import paper_2512_09200_b200 as L
            recv_off = L.lengths_to_offsets(recv_len)
        else:
            recv_off = scan_fn(recv_len)
        return recv_off, recv_ids

    def _exchange_ids_static(self, offsets, ids, scan_fn=None):
        W, Fl, B, cap = self.W, self.Fl, self.B, self.capacity
        dev = offsets.device
        lengths = (offsets[1:] - offsets[:-1]).to(torch.int32)
        recv_len = torch.empty(W * Fl * B, dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_len, lengths, group=self.group)
        counts, bounds = self.slice_counts(offsets)
        ovf = (counts > cap).any()
        self.overflow = ovf if self.overflow is None else (self.overflow | ovf)
        # pack: slice o of the local ids -> row o of a [W][cap] buffer
        j = torch.arange(cap, device=dev)
        src = (bounds[:-1, None] + j[None, :]).clamp_(max=max(ids.numel() - 1, 0))
        send = torch.where(j[None, :] < counts[:, None], ids[src], torch.zeros((), dtype=ids.dtype, device=dev))
        recv = torch.empty((W, cap), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv.view(-1), send.reshape(-1).contiguous(), group=self.group)
        # receiver: offsets over [src][f_local][b] and compaction of the padded slices
        if scan_fn is None:
            import paper_2512_09200_b200 as L
            recv_off = L.lengths_to_offsets(recv_len)
        else:
            recv_off = scan_fn(recv_len)
        seg = recv_off[torch.arange(W + 1, device=dev) * (Fl * B)]
        rcount = (seg[1:] - seg[:-1])
        dest = torch.where(j[None, :] < rcount[:, None], seg[:-1, None] + j[None, :],
                           torch.full((), W * cap, dtype=torch.int64, device=dev))
        recv_ids = torch.empty(W * cap + 1, dtype=torch.int32, device=dev)
        recv_ids.scatter_(0, dest.reshape(-1), recv.reshape(-1))
        return recv_off, recv_ids

    # ---- 2. owner pooling ---------------------------------------------------------------------
    def pool(self, recv_off, recv_ids, tables=None, table_ptrs=None, rows=None, out=None, pool_fn=None):
        """-> send buffer [W*B][Fl][D] bf16, rms-normalised (the fused K1 epilogue)."""
        if pool_fn is not None:
            return pool_fn(recv_off, recv_ids)
        import paper_2512_09200_b200 as L
        return L.embedding_bag(tables, recv_off, recv_ids, self.B, out=out, out_dtype=torch.bfloat16,
                               normalize=True, check_errors=False, table_ptrs=table_ptrs, rows=rows,
                               sources=self.W)

    # ---- 3. output dist -------------------------------------------------------------------------
    def exchange_pooled(self, send, recv=None):
        """[W*B][Fl][D] (rows r*B.. go to rank r) -> [W][B][Fl][D] (block o from owner o)."""
        if recv is None:
            recv = torch.empty_like(send)
        dist.all_to_all_single(recv.view(-1), send.view(-1), group=self.group)
        return recv

    def forward_embeddings(self, offsets, ids, tables, table_ptrs, rows, send=None, recv=None):
        recv_off, recv_ids = self.exchange_ids(offsets, ids)
        send = self.pool(recv_off, recv_ids, tables, table_ptrs, rows, out=send)
        return self.exchange_pooled(send, recv)

"""World-size-2/3/8 gloo test (CPU) of the peer-memory sharded embedding host logic
(paper_2512_09200_b200/peer.py): every shared buffer is exported once per rank, the pointer
table a rank hands to the owner kernel holds its own pointer at its own index and the peers'
IPC-mapped pointers elsewhere, and one step issues bucket -> barrier -> owner kernel ->
barrier -> in-place forward with the owned feature block. The IPC / barrier / kernel calls are
injected fakes here; the real ones run in tests/dist_sharded_check.py on >= 2 GPUs."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAPPED = 1 << 40  # fake peer mappings live at handle-ptr + MAPPED


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeOps:
    def __init__(self, rank):
        self.rank = rank
        self.log = []

    def ipc_handle(self, ptr):
        return (int(ptr).to_bytes(8, "little") + bytes([self.rank]) * 56, 0)

    def ipc_open(self, h, off):
        assert len(h) == 64 and h[8] != self.rank  # never map our own allocation
        return int.from_bytes(h[:8], "little") + off + MAPPED

    def ipc_close(self, p):
        self.log.append(("close", p))

    def peer_barrier(self, flags, rank, world, status, timeout_s, stream=None):
        self.log.append(("barrier", rank, world))

    def peer_embedding_bag(self, rank, world, tables, table_ptrs, rows, feature_base, batch, off_ptrs,
                           ids_ptrs, pos_ptrs, out_ptrs, stride, normalize=True, stream=None):
        self.log.append(("bag", rank, world, len(tables), feature_base, batch, stride,
                         off_ptrs.tolist(), ids_ptrs.tolist(), pos_ptrs.tolist(), out_ptrs.tolist()))


class FakeNet:
    def __init__(self, rank, log):
        self.rank, self.log = rank, log

    def buffer(self, which):
        return 1000 * (self.rank + 1) + which  # distinct per rank and buffer

    def bucket(self, domain, stream=None):
        self.log.append(("bucket",))

    def forward_in_place(self, domain, logits=None, stream=None, dense=None):
        self.log.append(("forward",))
        return logits


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from paper_2512_09200_b200.peer import PeerBags
        ops = FakeOps(rank)
        net = FakeNet(rank, ops.log)
        F, B, D = 6 * world, 5, 16
        pb = PeerBags(net, F, B, D, world, rank, ops=ops, device="cpu")
        off = torch.zeros(F * B + 1, dtype=torch.int64)
        ids = torch.zeros(10, dtype=torch.int32)
        pb.register("k", off, ids)
        tables = [torch.zeros(3, D) for _ in range(pb.Fl)]
        pb.forward("k", torch.zeros(B, dtype=torch.int32), tables, None, None)
        pb.close()
        # collect what the owner kernel was handed
        bag = [e for e in ops.log if e[0] == "bag"][0]
        seq = [e[0] for e in ops.log if e[0] != "close"]
        q.put((rank, bag, seq, off.data_ptr(), ids.data_ptr(), sum(e[0] == "close" for e in ops.log)))
    except Exception as e:  # surface worker failures instead of a queue timeout
        q.put((rank, "error", repr(e), 0, 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_peer_exchange_pointer_tables(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, bag, seq, offp, idsp, closes = q.get(timeout=120)
        assert bag != "error", seq
        res[r] = (bag, seq, offp, idsp, closes)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    F, B, D = 6 * world, 5, 16
    for r in range(world):
        bag, seq, offp, idsp, closes = res[r]
        assert seq == ["bucket", "barrier", "bag", "barrier", "forward"]
        _, rank, w, n_tab, fbase, batch, stride, offs, idss, poss, outs = bag
        assert (rank, w, n_tab, fbase, batch, stride) == (r, world, F // world, r * (F // world), B, F * D)
        for q_ in range(world):
            own = q_ == r
            # X0 (buffer 0) and sample_pos (buffer 1) of rank q_
            assert outs[q_] == 1000 * (q_ + 1) + (0 if own else MAPPED)
            assert poss[q_] == 1000 * (q_ + 1) + 1 + (0 if own else MAPPED)
            assert offs[q_] == res[q_][2] + (0 if own else MAPPED)
            assert idss[q_] == res[q_][3] + (0 if own else MAPPED)
        # flags, X0, pos, offsets, ids: one mapping per peer each, all closed
        assert closes == 5 * (world - 1)

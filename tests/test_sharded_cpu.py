"""World-size-2 gloo test (CPU) of the table-wise sharding exchange logic
(paper_2512_09200_b200/sharded.py): ids all-to-all, owner pooling over [src][f][b] bags,
pooled all-to-all. Pooling is done by the CPU oracle here (injected), so this checks the
layouts and split sizes; the CUDA pooling itself is covered by tests/test_embedding_bag_gpu.py
and the 2-GPU check tests/dist_sharded_check.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

F, ROWS, D, B, MAXLEN = 6, 500, 16, 7, 9
SEED_T = 0x1A77


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_pool(Fl, owned0, W, B):
    """pool_fn stand-in: [src][f_local][b] bags -> [W*B][Fl][D] normalised (fp32 here)."""
    def fn(recv_off, recv_ids, slice_cap):
        off = recv_off.numpy()
        ids = recv_ids.numpy()
        out = np.zeros((W * B, Fl, D), np.float32)
        for r in range(W):
            shift = r * slice_cap - off[r * Fl * B] if slice_cap else 0
            for fl in range(Fl):
                for b in range(B):
                    bag = (r * Fl + fl) * B + b
                    for j in range(off[bag] + shift, off[bag + 1] + shift):
                        for c in range(D):
                            out[r * B + b, fl, c] += oracle.load_oracle().lo_table_value(
                                SEED_T, owned0 + fl, int(ids[j]), D, ROWS, c)
        n = out / np.sqrt((out.astype(np.float64) ** 2).mean(-1, keepdims=True) + 1e-6)
        return torch.from_numpy(n.astype(np.float32))
    return fn


def _worker(rank, world, port, q, capacity):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2512_09200_b200.sharded import ShardedBags  # noqa: E402  (no CUDA needed)
        sb = ShardedBags(F, B, D, world, rank, capacity=capacity)
        off, ids = oracle.synth_bags(F, B, MAXLEN, ROWS, 0x1A78 + rank)
        def pack(bounds, ids_, cap, out, overflow):  # CPU stand-in for lattice_pack_slices
            for o in range(world):
                n = int(bounds[o + 1] - bounds[o])
                overflow |= int(n > cap)
                out[o, :min(n, cap)] = ids_[int(bounds[o]): int(bounds[o]) + min(n, cap)]

        recv_off, recv_ids, cap = sb.exchange_ids(
            torch.from_numpy(off), torch.from_numpy(ids.astype(np.int32)),
            scan_fn=lambda l: torch.cat([torch.zeros(1, dtype=torch.int64), torch.cumsum(l.to(torch.int64), 0)]),
            pack_fn=pack)
        send = sb.pool(recv_off, recv_ids, cap, pool_fn=_oracle_pool(sb.Fl, sb.owned()[0], world, B))
        sb.check_overflow()
        recv = sb.exchange_pooled(send)
        # expected: oracle pooling of this rank's own batch over all F features, normalised
        full, _ = oracle.embedding_bag_synth(SEED_T, F, ROWS, D, B, off, ids)
        full = full / np.sqrt((full.astype(np.float64) ** 2).mean(-1, keepdims=True) + 1e-6)
        got = recv.numpy().reshape(world, B, sb.Fl, D).transpose(1, 0, 2, 3).reshape(B, F, D)
        q.put((rank, float(np.abs(got - full).max())))
    except Exception as e:  # surface failures to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("capacity", [None, 101, 160])
def test_two_rank_exchange_matches_oracle(capacity):
    """capacity None: split sizes read back each step; 101 (= the largest slice of this batch,
    exactly full) and 160 (padded): static slices, device-side compaction, no host sync."""
    if not dist.is_gloo_available():
        pytest.skip("gloo unavailable")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, capacity)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert not isinstance(err, str), err
        assert err < 1e-5, (rank, err)

"""Static-slice overflow of the sharded ids exchange (slice_cap): a source that sent an owner more
ids than the slice holds has its slice truncated by the sender (lattice_pack_slices sets the
overflow flag); the owner's bag kernel must pool only the ids inside the slice -- never the next
source's ids and never past the receive buffer. Run as a script so LATTICE_BAG_KERNEL can select
the direct (0) or the staged (1) kernel for the whole process (tests/test_embedding_bag_gpu.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_09200_b200 as L
    F, rows, D, B, R = 3, 2000, 128, 301, 3
    tab = torch.empty((F, rows, D), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, 0x1A77)
    parts = [L.synth_bags(F, B, 40, rows, 0x1A78 + r) for r in range(R)]
    n = [int(o[-1]) for o, _ in parts]
    cap = min(n) - 500  # every source overflows its slice by > 500 ids
    lens = torch.cat([o[1:] - o[:-1] for o, _ in parts])
    off = torch.zeros(R * F * B + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lens, 0)
    # the receive buffer exactly [R][cap]; what pack_slices delivers: the first cap ids of each
    recv = torch.cat([i[:cap] for _, i in parts]).contiguous()
    got = L.embedding_bag(list(tab.unbind(0)), off, recv, B, sources=R, slice_cap=cap, check_errors=False)
    # expected: each source's bags with their CSR clamped to the slice
    want = torch.cat([L.embedding_bag(list(tab.unbind(0)), o.clamp(max=cap), i[:cap].contiguous(), B)
                      for o, i in parts])
    torch.cuda.synchronize()
    assert torch.equal(got, want), "truncated slices pooled wrongly"
    print("ok", os.environ.get("LATTICE_BAG_KERNEL", "default"))


if __name__ == "__main__":
    main()

"""Logits of a G=16, 12-head network through whichever tower path LATTICE_TOWER_PAIR selects (the
CTA-pair swish GEMM + heads kernel by default, the round-1 single-CTA grouped kernel with the heads
in its epilogue when 0), saved to argv[1] (.npy). tests/test_network_gpu.py compares the two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import paper_2512_09200_b200 as L
    cfg = dict(n=64, d=128, blocks=2, nF=32, nL=32, k=16, mlp=[1024, 512, 4096], domains=16, heads=12,
               tower_hidden=256)
    B, rows = 3000, 3000
    net = L.Network(**cfg, max_batch=B, weight_seed=0x1A79)
    tab = torch.empty((cfg["n"], rows, cfg["d"]), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, 0x1A77)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rws = torch.full((cfg["n"],), rows, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(cfg["n"], B, 40, rows, 0x1A78)
    dom = L.synth_domains(B, cfg["domains"], 0x1A78)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    np.save(sys.argv[1], logits.cpu().numpy())


if __name__ == "__main__":
    main()

"""Two lattice_nets forwarding concurrently on two CUDA streams: the CTA-pair
swish GEMMs of both run persistent grids that each want the whole GPU, and their row-statistics
exchange needs every pair of a grid resident. With cooperative launches (default) both nets must
produce their single-stream logits bit for bit and lattice_device_check must report nothing; with
LATTICE_GEMM_COOP=0 a lost co-residency must surface as a reported timeout, never a hang.
Run as a script (the env var is read once per process) by tests/test_gemm_gpu.py under a timeout.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_09200_b200 as L
    cfg = dict(n=64, d=128, blocks=2, nF=32, nL=32, k=16, mlp=[1024, 2048, 2048, 4096], domains=3, heads=4,
               tower_hidden=256)
    B, rows = 16384, 5000
    nets = [L.Network(**cfg, max_batch=B, weight_seed=0x1A79 + i) for i in range(2)]
    tab = torch.empty((cfg["n"], rows, cfg["d"]), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, 0x1A77)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rws = torch.full((cfg["n"],), rows, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(cfg["n"], B, 40, rows, 0x1A78)
    dom = L.synth_domains(B, cfg["domains"], 0x1A78)
    want = [n.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16).clone() for n in nets]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in nets]
    outs = [torch.empty_like(w) for w in want]
    for _ in range(20):
        for n, s, o in zip(nets, streams, outs):
            with torch.cuda.stream(s):
                n.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16, logits=o, stream=s)
    torch.cuda.synchronize()
    status = "ok"
    try:
        L.device_check()
    except L.CudaError as e:
        status = "timeout reported: " + str(e)
    same = all(torch.equal(o, w) for o, w in zip(outs, want))
    print(json.dumps({"coop": os.environ.get("LATTICE_GEMM_COOP", "1"), "status": status, "bit_identical": same}))


if __name__ == "__main__":
    main()

"""K2 (lattice_fm_lcb) timing at the mid and large block shapes on one GPU, with the per-launch
kernel time from CUDA events (the entry's small Y^T / W_L pad copies included) and the HBM
fraction of its algorithmic bytes. Prints one JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_09200_b200 as L
    shapes = [("mid", 256, 32, 128, 32768), ("large", 512, 32, 256, 65536)]
    if len(sys.argv) > 1:
        shapes = [s for s in shapes if s[0] in sys.argv[1:]]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6446.3
    for name, n, k, nF, B in shapes:
        d, nL = 128, n - nF
        g = torch.Generator(device="cuda").manual_seed(1)
        X = (torch.randn((B, n, d), generator=g, device="cuda") * 0.3).to(torch.bfloat16)
        YT = (torch.randn((k, n), generator=g, device="cuda") * 0.05).to(torch.bfloat16)
        WL = (torch.randn((nL, n), generator=g, device="cuda") * 0.05).to(torch.bfloat16)
        Fin = torch.empty((B, n * k), dtype=torch.bfloat16, device="cuda")
        Xout = torch.empty_like(X)
        for _ in range(3):
            L.fm_lcb(X, YT, WL, nF, Fin, Xout)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        for i in range(10):
            ev[i].record()
            L.fm_lcb(X, YT, WL, nF, Fin, Xout)
        ev[10].record()
        torch.cuda.synchronize()
        ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
        alg = B * (n * d * 2 + n * k * 2 + nL * d * 2)
        med = ms[5]
        print(json.dumps({"shape": name, "n": n, "k": k, "nL": nL, "B": B, "ms_median": med, "ms_min": ms[0],
                          "GB/s": alg / (med / 1e3) / 1e9, "frac_hbm": alg / (med / 1e3) / 1e9 / peak,
                          "us_per_sample_per_sm": med * 1e3 / (B / 148)}))
        del X, Xout, Fin


if __name__ == "__main__":
    main()

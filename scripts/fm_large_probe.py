"""Times the large-n FM/LCB kernel (n = 512, nL = 256, d = 128, k = 32, B = 65536: the large
config's backbone) on ONE GPU, without the 196 GB of tables: the network is fed pooled rows
(pooled_layout 0) and its stage timer reports ms per FM/LCB launch and per MLP block.
usage: python scripts/fm_large_probe.py [reps]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_09200_b200 as L  # noqa: E402

LARGE = dict(n=512, d=128, blocks=4, nF=256, nL=256, k=32, mlp=[16384, 2048, 2048, 32768], domains=16, heads=12,
             tower_hidden=512)
B = 65536
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
torch.cuda.set_device(0)
net = L.Network(**LARGE, max_batch=B, weight_seed=0x1A79)
pooled = (torch.randn((B, LARGE["n"], LARGE["d"]), device="cuda") * 0.1).to(torch.bfloat16)
dom = L.synth_domains(B, LARGE["domains"], 0x1A78)
logits = torch.empty((B, LARGE["heads"]), device="cuda")
net.set_timing(True)
fm, mlp = [], []
for r in range(reps + 1):
    net.forward(dom, pooled=pooled, logits=logits)
    st = net.stage_times()  # [bucket, bag, (fm, mlp) x blocks, tower]
    if r:
        fm += st[2:2 + 2 * LARGE["blocks"]:2]
        mlp += st[3:3 + 2 * LARGE["blocks"]:2]
fm_bytes = B * (512 * 128 * 2 + 512 * 32 * 2 + 256 * 128 * 2)
print("fm_lcb large ms/block: median %.3f  min %.3f  (%.0f GB/s algorithmic)  mlp ms/block %.3f"
      % (statistics.median(fm), min(fm), fm_bytes / statistics.median(fm) / 1e6, statistics.median(mlp)))

"""Does ncu profile the cooperative CTA-pair swish GEMM? (one lattice_gemm swish launch)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_09200_b200 as L
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randn((1024, 512), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
B = (torch.randn((2048, 512), generator=g, device="cuda") / 512 ** 0.5).to(torch.bfloat16)
C = L.gemm(A, B, epilogue=L.EPI_SWISH)
torch.cuda.synchronize()
L.device_check()
print("ok", os.environ.get("LATTICE_GEMM_COOP", "1"), float(C.float().abs().sum()))

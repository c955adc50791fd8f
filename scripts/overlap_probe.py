"""Feasibility probe: does the embedding-bag kernel (HBM-bound) overlap with the dense stage
(tensor-bound) when they run on two streams? Mid shapes. Prints ms per iteration for each alone
and both together. LATTICE_BAG_BLOCKS_PER_SM controls how many bag blocks share an SM."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_09200_b200 as L

MID = dict(n=256, d=128, blocks=4, nF=128, nL=128, k=32, mlp=[8192, 2048, 2048, 16384], domains=4, heads=6,
           tower_hidden=512)
B, ROWS, K = 32768, 100000, 10
torch.cuda.set_device(0)
net = L.Network(**MID, max_batch=B, weight_seed=0x1A79)
n, d = MID["n"], MID["d"]
tab = torch.empty((n, ROWS, d), dtype=torch.bfloat16, device="cuda")
L.fill_tables(tab, 0x1A77)
tables = list(tab.unbind(0))
ptrs = torch.tensor([t.data_ptr() for t in tables], dtype=torch.int64, device="cuda")
rows = torch.full((n,), ROWS, dtype=torch.int64, device="cuda")
off, ids = L.synth_bags(n, B, 40, ROWS, 0x1A78)
dom = L.synth_domains(B, 4, 0x1A78)
E = torch.empty((B, n, d), dtype=torch.bfloat16, device="cuda")
logits = torch.empty((B, 6), device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
net.forward(dom, off, ids, ptrs, rows, torch.bfloat16, logits=logits)  # X0 valid
net.bucket(dom)
import ctypes
POS = os.environ.get("PROBE_POS", "net")
if POS == "rand":
    pos = torch.randperm(B, device="cuda").to(torch.int32)
elif POS == "ident":
    pos = torch.arange(B, device="cuda", dtype=torch.int32)
else:
    order = torch.argsort(dom.long(), stable=True)  # the network's domain-sorted rows (K6)
    pos = torch.empty(B, dtype=torch.int32, device="cuda")
    pos[order] = torch.arange(B, dtype=torch.int32, device="cuda")


def dense(k):
    with torch.cuda.stream(s1):
        for _ in range(k):
            net.forward_in_place(dom, logits=logits, stream=s1)


def emb(k):
    with torch.cuda.stream(s2):
        for _ in range(k):
            L.embedding_bag(tables, off, ids, B, out=E, sample_pos=pos, normalize=True, check_errors=False,
                            table_ptrs=ptrs, rows=rows, stream=s2)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for _ in range(2):
    dense(2), emb(2)
print("pos", POS, "blocks/SM cap", os.environ.get("LATTICE_BAG_BLOCKS_PER_SM", "default"))
print("dense alone  %.2f ms" % timed(lambda: dense(K)))
print("bag alone    %.2f ms" % timed(lambda: emb(K)))
def full(k):
    for _ in range(k):
        net.forward(dom, off, ids, ptrs, rows, torch.bfloat16, logits=logits)


print("net forward  %.2f ms" % timed(lambda: full(K)))
print("both         %.2f ms" % timed(lambda: (dense(K), emb(K))))

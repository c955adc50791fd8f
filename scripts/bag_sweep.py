"""Embedding-bag variant sweep: kernel ms for micro (fp32/bf16) and mid-shaped bags."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def one(F, R, D, B, dt, variant, net_like=False, keep=0):
    code = f"""
import os, sys, torch, json
sys.path.insert(0, {ROOT!r})
import paper_2512_09200_b200 as L
dt = torch.{dt}
tab = torch.empty(({F}, {R}, {D}), dtype=dt, device='cuda'); L.fill_tables(tab, 0x1A77)
tables = list(tab.unbind(0))
ptrs = torch.tensor([t.data_ptr() for t in tables], dtype=torch.int64, device='cuda')
rows = torch.full(({F},), {R}, dtype=torch.int64, device='cuda')
off, ids = L.synth_bags({F}, {B}, 40, {R}, 0x1A78)
out = torch.empty(({B}, {F}, {D}), dtype=dt, device='cuda')
pos = torch.randperm({B}, device='cuda').to(torch.int32) if {net_like} else None
for _ in range(3): L.embedding_bag(tables, off, ids, {B}, out=out, check_errors=False, table_ptrs=ptrs, rows=rows, sample_pos=pos, normalize={net_like})
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): L.embedding_bag(tables, off, ids, {B}, out=out, check_errors=False, table_ptrs=ptrs, rows=rows, sample_pos=pos, normalize={net_like})
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
n = int(off[-1]); s = tab.element_size()
by = n*{D}*s + n*4 + ({F}*{B}+1)*8 + {F}*{B}*{D}*s
print(json.dumps(dict(ms=ms, GBs=by/ms/1e6)))
"""
    env = dict(os.environ, LATTICE_BAG_VARIANT=str(variant), LATTICE_BAG_L2KEEP=str(keep))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    return r.stdout.strip() or r.stderr[-300:]

if len(sys.argv) > 1 and sys.argv[1] == "l2":
    # LATTICE_BAG_L2KEEP bit 0: rows evict_last, bit 1: pooled-row stores evict_first
    for rows in (100000, 1000000):
        for keep in (0, 1, 2, 3):
            print("mid_bf16 rows", rows, "keep", keep,
                  one(256, rows, 128, 32768, "bfloat16", 0, True, keep), flush=True)
    sys.exit(0)
for name, cfg in [("micro_f32", (64, 1000000, 128, 16384, "float32")),
                  ("micro_bf16", (64, 1000000, 128, 16384, "bfloat16")),
                  ("mid_bf16", (256, 100000, 128, 32768, "bfloat16"))]:
    for v in (0, 1, 2):
        print(name, "variant", v, one(*cfg, v), flush=True)
for v in (0, 1, 2):
    print("mid_bf16 normalize+pos variant", v, one(256, 100000, 128, 32768, "bfloat16", v, True), flush=True)

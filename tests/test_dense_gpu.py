"""Dense features of consolidated domains on the GPU: the merge_domains
value gather (bit-exact vs the oracle, itself pinned to the reference in tests/test_oracle.py)
and the network's dense processor feeding the last embeddings of X0, against the
fp64 oracle with the same bf16 rounding points.

Tolerance: merge bit-exact; logits |gpu - oracle| <= 2e-2 + 2e-2 |oracle| (bf16, as
tests/test_network_gpu.py)."""
import numpy as np
import pytest

import oracle
from test_network_gpu import SEED_D, SEED_T, SEED_W, assert_logits_close

pytestmark = pytest.mark.gpu

DENSE = dict(n=24, d=128, blocks=2, nF=12, nL=12, k=16, mlp=[384, 512, 1536], domains=3, heads=4,
             tower_hidden=128, dense_features=4, dense_in=40, dense_hidden=256)


def make_dense(B, G, seed=5):
    """Three domains declaring overlapping dense feature sets, merged under the union schema."""
    import paper_2512_09200_b200 as L
    rng = np.random.default_rng(seed)
    declared = [[f"f{i}" for i in rng.choice(40, size=k, replace=False)] for k in (10, 17, 23)][:G]
    union, src = L.union_schema(declared)
    md = max(len(x) for x in declared)
    dom = rng.integers(0, G, B).astype(np.int32)
    vals = np.zeros((B, md), np.float32)
    for b in range(B):
        k = len(declared[dom[b]])
        vals[b, :k] = rng.normal(size=k).astype(np.float32)
    return declared, union, src, dom, vals


def test_merge_dense_bit_exact():
    import torch
    import paper_2512_09200_b200 as L
    B, G = 5000, 3
    declared, union, src, dom, vals = make_dense(B, G)
    width = 48  # the union (<= 40 names) padded to a GEMM-friendly width
    src_w = np.full((G, width), -1, np.int32)
    src_w[:, : len(union)] = src
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for odt, bf in ((torch.float32, False), (torch.bfloat16, True)):
        got = L.merge_dense(d(dom), d(vals), d(src_w), width, out_dtype=odt)
        bad, want = oracle.merge_dense(dom, vals, src_w, bf16=bf)
        assert bad == -1 and np.array_equal(got.float().cpu().numpy(), want)
    # fp64 in / out (the C++ drop-in's merge_domains): exact
    v64 = vals.astype(np.float64) + 1e-9  # not fp32-representable
    got = L.merge_dense(d(dom), d(v64), d(src_w), width, out_dtype=torch.float64).cpu().numpy()
    for b in (0, 1, 4999):
        for c in range(width):
            j = src_w[dom[b], c]
            assert got[b, c] == (v64[b, j] if j >= 0 else 0.0)
    dom2 = dom.copy()
    dom2[77] = G
    with pytest.raises(L.DataError):
        L.merge_dense(d(dom2), d(vals), d(src_w), width)


def test_network_with_dense_features_matches_oracle():
    import torch
    import paper_2512_09200_b200 as L
    cfg = DENSE
    B, rows = 600, 3000
    n, d, nd = cfg["n"], cfg["d"], cfg["dense_features"]
    nc = n - nd
    net = L.Network(**cfg, max_batch=B, weight_seed=SEED_W)
    tab = torch.empty((nc, rows, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rws = torch.full((nc,), rows, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(nc, B, 40, rows, SEED_D)
    dom = L.synth_domains(B, cfg["domains"], SEED_D)
    declared, union, src, ddom, vals = make_dense(B, 3)
    src_w = np.full((3, cfg["dense_in"]), -1, np.int32)
    src_w[:, : len(union)] = src
    dense = L.merge_dense(torch.from_numpy(ddom).cuda(), torch.from_numpy(vals).cuda(),
                          torch.from_numpy(src_w).cuda(), cfg["dense_in"])
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16, dense=dense).cpu().numpy()
    with pytest.raises(L.UsageError):  # the dense input is required
        net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    # oracle: pooled sparse rows + the dense processor's rows, then lo_net_forward
    samples = list(range(0, B, 25)) + [B - 1]
    o_cpu = offsets.cpu().numpy()
    i_cpu = ids.cpu().numpy()[: o_cpu[-1]]
    w = net.weights()
    pooled = np.zeros((len(samples), n, d), np.float32)
    for j, s in enumerate(samples):
        pooled[j, :nc] = oracle.embedding_bag_synth(SEED_T, nc, rows, d, B, o_cpu, i_cpu, s, s + 1)[0][0]
    c = oracle.LoNetCfg()
    c.n, c.d, c.blocks, c.nF, c.nL, c.k = n, d, cfg["blocks"], cfg["nF"], cfg["nL"], cfg["k"]
    c.n_mlp = len(cfg["mlp"]) - 1
    for i, v in enumerate(cfg["mlp"]):
        c.mlp[i] = v
    c.G, c.heads, c.tower_hidden, c.hard, c.bf16 = cfg["domains"], cfg["heads"], cfg["tower_hidden"], 0, 1
    dense_cpu = dense.float().cpu().numpy()[samples]
    oracle.dense_processor(c, nd, cfg["dense_in"], cfg["dense_hidden"], w["D1"], w["D2"], dense_cpu, pooled)
    keep = [np.ascontiguousarray(a, dtype=np.float32) for a in w["YT"] + w["WL"] + w["mlp"]]
    nb = cfg["blocks"]
    P = oracle.ctypes.c_void_p
    yt = (P * nb)(*[a.ctypes.data for a in keep[:nb]])
    wl = (P * nb)(*[a.ctypes.data for a in keep[nb:2 * nb]])
    ml = (P * len(w["mlp"]))(*[a.ctypes.data for a in keep[2 * nb:]])
    T1 = np.ascontiguousarray(w["T1"], dtype=np.float32)
    T2 = np.ascontiguousarray(w["T2"], dtype=np.float32)
    ws = oracle.LoNetWeights(oracle.ctypes.cast(yt, P), oracle.ctypes.cast(wl, P), oracle.ctypes.cast(ml, P),
                             P(T1.ctypes.data), P(T2.ctypes.data))
    dcpu = np.ascontiguousarray(dom.cpu().numpy()[samples], dtype=np.int32)
    want = np.zeros((len(samples), cfg["heads"]), np.float32)
    oracle.load_oracle().lo_net_forward(oracle.ctypes.byref(c), oracle.ctypes.byref(ws), len(samples),
                                        oracle.ptr(pooled), oracle.ptr(dcpu), oracle.ptr(want), 0)
    # weights come from the shared counter-based generator
    lib = oracle.load_oracle()
    assert w["D1"][3, 5] == lib.lo_weight_value(SEED_W, lib.lo_weight_tag(0, 6, 0), 3, 5, cfg["dense_in"])
    assert w["D2"][100, 7] == lib.lo_weight_value(SEED_W, lib.lo_weight_tag(0, 7, 0), 100, 7, cfg["dense_hidden"])
    assert_logits_close(logits[samples], want)
    # zeroing the dense input changes the logits (the dense rows are live)
    zero = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16, dense=torch.zeros_like(dense)).cpu().numpy()
    assert not np.array_equal(zero, logits)

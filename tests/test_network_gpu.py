"""Lattice Network forward (K6 -> K1 -> [K2 -> K3 x n_mlp] x blocks -> K4) on the GPU vs the
fp64 CPU oracle (oracle/lattice_oracle.c lo_net_forward) on identical synthetic inputs and the
network's own bf16 weights. The oracle rounds to bf16 at every point the GPU stores bf16.

Tolerance (bf16 configs, stated per SURVEY.md 8d): |gpu - oracle| <= 2e-2 + 2e-2 * |oracle| on
every logit. Order/permutation properties are checked bit-exactly."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
SEED_T, SEED_D, SEED_W = 0x1A77, 0x1A78, 0x1A79

TINY = dict(n=8, d=64, blocks=2, nF=4, nL=4, k=4, mlp=[32, 64, 256], domains=2, heads=2,
            tower_hidden=64)
MID = dict(n=256, d=128, blocks=4, nF=128, nL=128, k=32, mlp=[8192, 2048, 2048, 16384],
           domains=4, heads=6, tower_hidden=512)
SMALL = dict(n=64, d=128, blocks=2, nF=32, nL=32, k=16, mlp=[1024, 512, 4096], domains=3,
             heads=4, tower_hidden=256)


def build(cfg, B, rows, max_len=40, hard=False, dtype="bf16"):
    import torch
    import paper_2512_09200_b200 as L
    net = L.Network(**cfg, hard=hard, max_batch=B, weight_seed=SEED_W, dtype=dtype)
    n, d = cfg["n"], cfg["d"]
    tab = torch.empty((n, rows, d), dtype=torch.float32 if dtype == "f32" else torch.bfloat16, device="cuda")
    L.fill_tables(tab, SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rws = torch.full((n,), rows, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(n, B, max_len, rows, SEED_D)
    dom = L.synth_domains(B, cfg["domains"], SEED_D)
    return net, tab, ptrs, rws, offsets, ids, dom


def oracle_logits(net, cfg, rows, offsets, ids, dom, samples, hard=False, bf16=True):
    n, d = cfg["n"], cfg["d"]
    B = dom.shape[0]
    o_cpu = offsets.cpu().numpy()
    i_cpu = ids.cpu().numpy()[: o_cpu[-1]]
    pooled = np.concatenate([oracle.embedding_bag_synth(SEED_T, n, rows, d, B, o_cpu, i_cpu, s, s + 1)[0]
                             for s in samples])
    w = net.weights()
    lib = oracle.load_oracle()
    c = oracle.LoNetCfg()
    c.n, c.d, c.blocks, c.nF, c.nL, c.k = n, d, cfg["blocks"], cfg["nF"], cfg["nL"], cfg["k"]
    c.n_mlp = len(cfg["mlp"]) - 1
    for i, v in enumerate(cfg["mlp"]):
        c.mlp[i] = v
    c.G, c.heads, c.tower_hidden, c.hard = cfg["domains"], cfg["heads"], cfg["tower_hidden"], int(hard)
    c.bf16 = 1 if bf16 else 0
    keep = [np.ascontiguousarray(a, dtype=np.float32) for a in w["YT"] + w["WL"] + w["mlp"]]
    nb = cfg["blocks"]
    P = oracle.ctypes.c_void_p
    yt = (P * nb)(*[a.ctypes.data for a in keep[:nb]])
    wl = (P * nb)(*[a.ctypes.data for a in keep[nb:2 * nb]])
    ml = (P * len(w["mlp"]))(*[a.ctypes.data for a in keep[2 * nb:]])
    T1 = np.ascontiguousarray(w["T1"], dtype=np.float32)
    T2 = np.ascontiguousarray(w["T2"], dtype=np.float32)
    ws = oracle.LoNetWeights(oracle.ctypes.cast(yt, P), oracle.ctypes.cast(wl, P),
                             oracle.ctypes.cast(ml, P), P(T1.ctypes.data), P(T2.ctypes.data))
    d_cpu = np.ascontiguousarray(dom.cpu().numpy()[samples], dtype=np.int32)
    out = np.zeros((len(samples), cfg["heads"]), np.float32)
    lib.lo_net_forward(oracle.ctypes.byref(c), oracle.ctypes.byref(ws), len(samples),
                       oracle.ptr(pooled), oracle.ptr(d_cpu), oracle.ptr(out), 0)
    return out, w


def check_weights_against_generator(w, cfg):
    lib = oracle.load_oracle()
    rng = np.random.default_rng(0)
    for blk in range(cfg["blocks"]):
        for _ in range(20):
            o, i = int(rng.integers(0, cfg["k"])), int(rng.integers(0, cfg["n"]))
            assert w["YT"][blk][o, i] == lib.lo_weight_value(SEED_W, lib.lo_weight_tag(blk, 1, 0), o, i, cfg["n"])
            li = int(rng.integers(0, len(cfg["mlp"]) - 1))
            W = w["mlp"][blk * (len(cfg["mlp"]) - 1) + li]
            o, i = int(rng.integers(0, W.shape[0])), int(rng.integers(0, W.shape[1]))
            assert W[o, i] == lib.lo_weight_value(SEED_W, lib.lo_weight_tag(blk, 3, li), o, i, W.shape[1])
    g = cfg["domains"] - 1
    assert w["T2"][g, 1, 3] == lib.lo_weight_value(SEED_W, lib.lo_weight_tag(g, 5, 0), 1, 3, cfg["tower_hidden"])


def assert_logits_close(got, want):
    err = np.abs(got - want)
    bound = 2e-2 + 2e-2 * np.abs(want)
    assert (err <= bound).all(), f"max err {err.max():.4g} (worst ratio {(err / bound).max():.3g}); rms {np.sqrt((want ** 2).mean()):.3g}"


@pytest.mark.parametrize("name,cfg,B,rows,hard", [("tiny", TINY, 512, 10000, False),
                                                  ("small", SMALL, 1000, 5000, False),
                                                  ("small_hard", SMALL, 700, 5000, True)])
def test_forward_matches_oracle(name, cfg, B, rows, hard):
    import torch
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows, hard=hard)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    torch.cuda.synchronize()
    samples = list(range(0, B, max(1, B // 48)))[:48] + [B - 1]
    want, w = oracle_logits(net, cfg, rows, offsets, ids, dom, samples, hard)
    check_weights_against_generator(w, cfg)
    got = logits.cpu().numpy()[samples]
    assert np.isfinite(got).all()
    assert_logits_close(got, want)


def test_tiny_config_fp32_tf32_matches_oracle():
    """BASELINE configs[0] in its stated dtype: fp32 storage, kind::tf32 tensor cores, against
    the fp64 oracle with fp32 storage rounding. Tolerance (TF32, 10-bit mantissa products):
    |gpu - oracle| <= 5e-3 + 5e-3 * |oracle|."""
    import torch
    B, rows = 512, 10000
    net, tab, ptrs, rws, offsets, ids, dom = build(TINY, B, rows, dtype="f32")
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.float32)
    torch.cuda.synchronize()
    samples = list(range(0, B, 16)) + [B - 1]
    want, w = oracle_logits(net, TINY, rows, offsets, ids, dom, samples, bf16=False)
    check_weights_against_generator(w, TINY)
    got = logits.cpu().numpy()[samples]
    err = np.abs(got - want)
    bound = 5e-3 + 5e-3 * np.abs(want)
    assert (err <= bound).all(), f"max err {err.max():.4g}; rms logit {np.sqrt((want ** 2).mean()):.3g}"


LARGE_N = dict(n=512, d=128, blocks=1, nF=256, nL=256, k=32, mlp=[16384, 256, 32768], domains=2,
               heads=3, tower_hidden=256)


LARGE_N_384 = dict(n=384, d=128, blocks=2, nF=256, nL=128, k=16, mlp=[6144, 256, 32768], domains=2,
                   heads=3, tower_hidden=256)


@pytest.mark.parametrize("cfg", [LARGE_N, LARGE_N_384], ids=["n512_nL256", "n384_nL128"])
def test_large_n_streamed_matches_oracle(cfg):
    """n > 256 (the large config's backbone width) runs the large FM/LCB variant (X_b resident,
    W_L streamed through a TMA ring of panels), n = 384 with zero-padded rows; widths of the
    MLP/tower shrunk so the fp64 oracle stays fast."""
    import torch
    B, rows = 300, 4000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    torch.cuda.synchronize()
    samples = [0, 1, 150, 299]
    want, w = oracle_logits(net, cfg, rows, offsets, ids, dom, samples)
    check_weights_against_generator(w, cfg)
    assert_logits_close(logits.cpu().numpy()[samples], want)


def test_mid_config_matches_oracle():
    import torch
    B, rows = 2048, 20000
    net, tab, ptrs, rws, offsets, ids, dom = build(MID, B, rows)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    torch.cuda.synchronize()
    samples = [0, 1, 2, 777, 1500, 2047]
    want, _ = oracle_logits(net, MID, rows, offsets, ids, dom, samples)
    assert_logits_close(logits.cpu().numpy()[samples], want)


def test_permutation_invariance_and_pooled_path():
    import torch
    import paper_2512_09200_b200 as L
    cfg, B, rows = SMALL, 777, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    base = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16).clone()
    # same samples, reversed order, through the pooled-input entry
    pooled = L.embedding_bag(list(tab.unbind(0)), offsets, ids, B, out_dtype=torch.float32)
    rev = torch.arange(B - 1, -1, -1, device="cuda")
    out = net.forward(dom[rev].contiguous(), pooled=pooled[rev].contiguous())
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy()[::-1], base.cpu().numpy(), rtol=2e-2, atol=2e-2)
    # reordering the batch through the sparse path is bit-exact per sample: rows are independent
    lens = (offsets[1:] - offsets[:-1]).view(cfg["n"], B)
    perm = torch.randperm(B, device="cuda")
    lens_p = lens[:, perm]
    off_p = torch.zeros(cfg["n"] * B + 1, dtype=torch.int64, device="cuda")
    off_p[1:] = torch.cumsum(lens_p.reshape(-1), 0)
    ids_p = torch.cat([ids[offsets[f * B + b]: offsets[f * B + b + 1]]
                       for f in range(cfg["n"]) for b in perm.tolist()]).to(torch.int32)
    out_p = net.forward(dom[perm].contiguous(), off_p, ids_p, ptrs, rws, torch.bfloat16)
    assert torch.equal(out_p, base[perm])


def test_domain_routing_uses_untied_towers():
    import torch
    cfg, B, rows = SMALL, 256, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    a = net.forward(torch.zeros_like(dom), offsets, ids, ptrs, rws, torch.bfloat16).clone()
    b = net.forward(torch.full_like(dom, 2), offsets, ids, ptrs, rws, torch.bfloat16).clone()
    mixed = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    assert not torch.equal(a, b)
    d = dom.cpu().numpy()
    assert torch.equal(mixed[torch.from_numpy(d == 0).cuda()], a[torch.from_numpy(d == 0).cuda()])
    assert torch.equal(mixed[torch.from_numpy(d == 2).cuda()], b[torch.from_numpy(d == 2).cuda()])


def test_out_of_range_id_reported_when_checked():
    """An id outside its table (or a domain outside [0, domains)): with check_errors the forward
    raises DataError naming the first offender (the oracle's semantics, lattice_embedding_bag's
    message); unchecked (graph / pipelined use) the bag pools a zero row / the sample takes
    domain 0, and the logits stay finite."""
    import torch
    import paper_2512_09200_b200 as L
    cfg, B, rows = SMALL, 256, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    bad = ids.clone()
    nz = torch.nonzero(offsets[1:] > offsets[:-1]).flatten()
    pos = int(offsets[int(nz[len(nz) // 2])])  # the first id of some non-empty bag
    bad[pos] = rows + 5
    last = int(offsets[-1]) - 1
    if last > pos:
        bad[last] = -1  # a later offender: the error still names the first
    with pytest.raises(L.DataError) as e:
        net.forward(dom, offsets, bad, ptrs, rws, torch.bfloat16, check_errors=True)
    assert e.value.index == pos and f"position {pos} " in str(e.value)
    out = net.forward(dom, offsets, bad, ptrs, rws, torch.bfloat16)
    assert torch.isfinite(out).all()
    ok = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16, check_errors=True)
    assert torch.isfinite(ok).all()
    # a domain outside [0, domains): DataError naming the first such sample when checked
    bad_dom = dom.clone()
    bad_dom[7] = cfg["domains"]
    bad_dom[100] = -1
    with pytest.raises(L.DataError) as e:
        net.forward(bad_dom, offsets, ids, ptrs, rws, torch.bfloat16, check_errors=True)
    assert e.value.index == 7 and "sample 7 " in str(e.value)
    assert torch.isfinite(net.forward(bad_dom, offsets, ids, ptrs, rws, torch.bfloat16)).all()


def test_config_contract():
    import paper_2512_09200_b200 as L
    bad = dict(SMALL)
    bad["nL"] = 31  # nF + nL != n
    with pytest.raises(L.UsageError):
        L.Network(**bad, max_batch=16)
    bad = dict(SMALL)
    bad["mlp"] = [1024, 4096, 4096]  # last width != nF*d
    with pytest.raises(L.UsageError):
        L.Network(**bad, max_batch=16)


def test_mid_config_full_batch_sampled_logits():
    """BASELINE configs[2] at its full size (256 features x 100k rows, l = 4, MLP 8192-2048-2048-
    16384, B = 32768): three sampled logits against the fp64 oracle (same tolerance), plus the
    size-independent property that the per-domain towers see every sample exactly once (a
    permutation of the batch changes no sample's logits, bit for bit)."""
    import torch
    import paper_2512_09200_b200 as L
    B, rows = 32768, 100000
    net, tab, ptrs, rws, offsets, ids, dom = build(MID, B, rows)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16).clone()
    torch.cuda.synchronize()
    samples = [3, 16000, 32767]
    want, w = oracle_logits(net, MID, rows, offsets, ids, dom, samples)
    assert_logits_close(logits.cpu().numpy()[samples], want)
    # permuted batch: reverse the samples (bags and domains), logits must follow exactly
    n = MID["n"]
    lens = (offsets[1:] - offsets[:-1]).view(n, B)
    starts = offsets[:-1].view(n, B)
    rlens = lens.flip(1).reshape(-1)
    roff = torch.zeros(n * B + 1, dtype=torch.int64, device="cuda")
    roff[1:] = torch.cumsum(rlens, 0)
    src = torch.repeat_interleave(starts.flip(1).reshape(-1), rlens) + (
        torch.arange(int(roff[-1]), device="cuda") - torch.repeat_interleave(roff[:-1], rlens))
    rids = ids[src]
    rl = net.forward(dom.flip(0).contiguous(), roff, rids, ptrs, rws, torch.bfloat16)
    assert torch.equal(rl.flip(0), logits)

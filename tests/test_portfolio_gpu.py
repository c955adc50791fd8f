"""The full consolidated portfolio step (BASELINE configs[4], bench.py --workload full) composed
exactly as bench.py runs it, checked end to end against the oracle composition:

  Zipper (K5)           window + labels [B, 4 tasks, 3 windows]     bit-exact vs oracle zip_columns
  merge_domains values  union-schema dense matrix                   bit-exact vs oracle merge_dense
  KTAP student inputs   [merged || clipped teacher emb or 0] bf16   bit-exact vs oracle student_inputs
  network               16 domains x 12 heads, dense processor (16 embeddings) + 240 sparse
                        features, mid-width backbone                every logit vs torch fp64,
                                                                     16 vs the C oracle (netcheck
                                                                     calibrated bound), stage-wise
  routed objectives     routed logits, per-task correlation loss,   routed bit-exact, counts exact,
                        window summary                              loss <= 1e-12 vs the oracle on the
                                                                     same logits; vs the fp64 logits'
                                                                     loss <= 1e-3
"""
import numpy as np
import pytest

import oracle
from netcheck import calibrated, oracle_forward, record
from test_network_gpu import SEED_D, SEED_T, SEED_W, both_refs, gpu_pooled, stagewise

pytestmark = pytest.mark.gpu

TASKS, WINDOWS = 4, [5400000, 86400000, 604800000]
PROBS = [1 / 3, 1 / 3, 1 / 3]
MERGED, TEACHER, STORE, TTL = 48, 16, 1 << 16, 4 * 3600 * 1000
CFG = dict(n=256, d=128, blocks=4, nF=128, nL=128, k=32, mlp=[8192, 2048, 2048, 16384], domains=16,
           heads=TASKS * len(WINDOWS), tower_hidden=512, dense_features=16, dense_in=MERGED + TEACHER,
           dense_hidden=256)


def test_full_portfolio_composition():
    import torch
    import paper_2512_09200_b200 as L
    B, rows = 4096, 20000
    c = CFG
    nc = c["n"] - c["dense_features"]
    # --- Zipper: window assignment + labels, bit-exact
    imp = L.synth_impressions(B, TASKS, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, WINDOWS, PROBS, 7, check_errors=True)
    users, ads, ts, conv, pres = oracle.synth_impressions(B, TASKS, 7)
    ow, ol, err, _ = oracle.zip_columns(users, ads, ts, conv, pres, WINDOWS, PROBS, 7)
    assert err == -1 and np.array_equal(win.cpu().numpy(), ow) and np.array_equal(lab.cpu().numpy(), ol)
    # --- merge_domains values under the union schema (16 domains declaring subsets of 48 names)
    dom = L.synth_domains(B, c["domains"], SEED_D)
    g_dense = torch.Generator().manual_seed(0xD15E)
    declared = [[f"x{int(i)}" for i in torch.randperm(MERGED, generator=g_dense)[:8 + 2 * g]]
                for g in range(c["domains"])]
    union, src = L.union_schema(declared)
    src_col = np.full((c["domains"], MERGED), -1, np.int32)
    src_col[:, : len(union)] = np.asarray(src, np.int32)
    max_decl = max(len(x) for x in declared)
    dvals = torch.randn((B, max_decl), generator=torch.Generator(device="cuda").manual_seed(1), device="cuda")
    merged = L.merge_dense(dom, dvals, torch.from_numpy(src_col).cuda(), MERGED, out_dtype=torch.float32)
    bad, want_m = oracle.merge_dense(dom.cpu().numpy(), dvals.cpu().numpy(), src_col)
    assert bad == -1 and np.array_equal(merged.cpu().numpy(), want_m)
    # --- KTAP student inputs: [merged || clip(teacher embedding) on a valid hit, zeros otherwise]
    gk = torch.Generator(device="cuda").manual_seed(0x7EAC)
    store_emb = torch.randn((STORE, TEACHER), generator=gk, device="cuda") * 2
    store_logit = torch.randn(STORE, generator=gk, device="cuda")
    t_now = 1_700_000_000_000
    written_at = t_now - torch.randint(0, TTL * 3 // 2, (STORE,), generator=gk, device="cuda")
    slot = torch.randint(0, STORE, (B,), generator=gk, device="cuda")
    slot[torch.rand(B, generator=gk, device="cuda") < 0.25] = -1
    dense, tlogit, hit = L.student_inputs(merged, slot, store_emb, written_at, TTL, t_now, store_logit=store_logit,
                                          clip=3.0, smoothing=0.1)
    rows_o, logit_o, hit_o = oracle.student_inputs(merged.cpu().numpy(), slot.cpu().numpy(), store_emb.cpu().numpy(),
                                                   store_logit.cpu().numpy(), written_at.cpu().numpy(), TTL, t_now,
                                                   clip=3.0, smoothing=0.1, bf16=True)
    assert np.array_equal(dense.float().cpu().numpy(), rows_o) and np.array_equal(hit.cpu().numpy(), hit_o)
    assert 0.2 < hit_o.mean() < 0.7  # hits, misses and expiries all occur
    # --- the network: 240 table-pooled features + 16 dense-processor embeddings, G = 16, 12 heads
    net = L.Network(**c, max_batch=B, weight_seed=SEED_W)
    tab = torch.empty((nc, rows, c["d"]), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rws = torch.full((nc,), rows, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(nc, B, 40, rows, SEED_D)
    logits_t = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16, dense=dense)
    logits = logits_t.cpu().numpy()
    w = net.weights()
    pooled = gpu_pooled(tab, offsets, ids, B)
    dense_h = dense.float().cpu().numpy()
    want, want32 = both_refs(c, w, pooled, dom.cpu(), dense=dense_h, chunk=1024)
    samples = list(range(0, B, B // 16))
    want_o = oracle_forward(c, w, pooled[samples].cpu().numpy(), dom.cpu().numpy()[samples], dense_h[samples])
    np.testing.assert_allclose(want[samples], want_o, rtol=1e-6, atol=1e-6)
    calibrated("full_portfolio: every logit vs torch fp64", logits, want, want32)
    calibrated("full_portfolio: 16 logits vs C oracle", logits[samples], want_o, want32[samples])
    stagewise("full_portfolio", net, c, w, logits, dom, B)
    # --- routed objectives on the GPU logits vs the oracle on the same logits
    routed, corr, counts, positives = L.routed_objectives(logits_t, win, lab, TASKS, len(WINDOWS))
    rc, r_o, corr_o, cnt_o, pos_o = oracle.routed_objectives(logits, ow, ol)
    assert rc == 0
    assert np.array_equal(routed.cpu().numpy(), r_o)
    assert np.array_equal(counts.cpu().numpy(), cnt_o) and np.array_equal(positives.cpu().numpy(), pos_o)
    np.testing.assert_allclose(corr.cpu().numpy(), corr_o, rtol=0, atol=1e-12)
    # and against the loss of the fp64 restatement's logits (the end-to-end objective value)
    _, _, corr_ref, _, _ = oracle.routed_objectives(want.astype(np.float32), ow, ol)
    dc = float(np.abs(corr.cpu().numpy() - corr_ref).max())
    record("full_portfolio: correlation loss vs fp64 logits", {"max_abs": dc, "loss": corr_ref.tolist()})
    assert dc <= 1e-3

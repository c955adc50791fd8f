"""The two restatements of the network arithmetic agree (CPU, no GPU): the scalar C oracle
(oracle/lattice_oracle.c forward_one, one sample at a time) and the batched torch fp64 einsum
restatement (tests/torch_ref.py), written separately from DESIGN.md section 3 / PAPER.md:271-318.
Both apply the same bf16 (or fp32) rounding points; they differ only in fp64 summation order and
in the C oracle's fp32 logit store, so they must agree to ~1e-7 on every logit of every sample.
This is the pin of the network arithmetic where no reference code exists;
the GPU tests then check the CUDA path against the torch restatement on every logit."""
import numpy as np
import pytest
import torch

import oracle
import torch_ref
from netcheck import host_weights, oracle_forward

SEED_T, SEED_D, SEED_W = 0x1A77, 0x1A78, 0x1A79

TINY = dict(n=8, d=64, blocks=2, nF=4, nL=4, k=4, mlp=[32, 64, 256], domains=2, heads=2, tower_hidden=64)
SMALL = dict(n=64, d=128, blocks=2, nF=32, nL=32, k=16, mlp=[1024, 512, 4096], domains=3, heads=4,
             tower_hidden=256)
DENSE = dict(n=24, d=128, blocks=2, nF=12, nL=12, k=16, mlp=[384, 512, 1536], domains=3, heads=4,
             tower_hidden=128, dense_features=4, dense_in=40, dense_hidden=256)
LARGE_N = dict(n=512, d=128, blocks=1, nF=256, nL=256, k=32, mlp=[16384, 256, 32768], domains=2,
               heads=3, tower_hidden=64)
MID = dict(n=256, d=128, blocks=4, nF=128, nL=128, k=32, mlp=[8192, 2048, 2048, 16384], domains=4, heads=6,
           tower_hidden=512)


def inputs(cfg, S, rows):
    nc = cfg["n"] - cfg.get("dense_features", 0)
    o, i = oracle.synth_bags(nc, S, 40, rows, SEED_D)
    pooled, bad = oracle.embedding_bag_synth(SEED_T, nc, rows, cfg["d"], S, o, i)
    assert bad == -1
    dom = oracle.synth_domains(S, cfg["domains"], SEED_D)
    dense = None
    if cfg.get("dense_features"):
        rng = np.random.default_rng(3)
        dense = oracle.bf16_round(rng.normal(size=(S, cfg["dense_in"])).astype(np.float32))
    return pooled, dom, dense


@pytest.mark.parametrize("name,cfg,S,rows,hard,bf16", [
    ("tiny_bf16", TINY, 512, 10000, False, True),
    ("tiny_fp32", TINY, 512, 10000, False, False),
    ("small", SMALL, 96, 5000, False, True),
    ("small_hard", SMALL, 64, 5000, True, True),
    ("dense", DENSE, 96, 3000, False, True),
    ("large_n", LARGE_N, 4, 4000, False, True),
    ("mid", MID, 4, 20000, False, True),
])
def test_restatements_agree(name, cfg, S, rows, hard, bf16):
    w = host_weights(cfg, SEED_W)
    pooled, dom, dense = inputs(cfg, S, rows)
    want = oracle_forward(cfg, w, pooled, dom, dense, bf16=bf16, hard=hard)
    got = torch_ref.forward(cfg, w, pooled, dom, dense, bf16=bf16, hard=hard).numpy()
    # the C oracle stores fp32 logits: allow its rounding (and fp64 summation order)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6, err_msg=name)
    assert np.abs(want).max() > 0.05  # non-degenerate logits


def test_restatements_see_each_rounding_point():
    """Both restatements put q() at the same places: dropping bf16 rounding moves the torch
    logits by far more than the agreement bound above (so the agreement is not vacuous)."""
    cfg = SMALL
    w = host_weights(cfg, SEED_W)
    pooled, dom, _ = inputs(cfg, 32, 5000)
    a = torch_ref.forward(cfg, w, pooled, dom, bf16=True).numpy()
    b = torch_ref.forward(cfg, w, pooled, dom, bf16=False).numpy()
    assert np.abs(a - b).max() > 1e-4


def test_fm_lcb_restatement_matches_block_pieces():
    """torch_ref.fm_lcb (the K2 kernel-level reference) equals the corresponding pieces of the
    block restatement."""
    cfg = SMALL
    w = host_weights(cfg, SEED_W)
    pooled, _, _ = inputs(cfg, 8, 5000)
    X = torch_ref.q(torch_ref.rms_norm(torch.as_tensor(pooled, dtype=torch.float64)), True)
    fin, lcb = torch_ref.fm_lcb(X, torch.as_tensor(w["YT"][0], dtype=torch.float64),
                                torch.as_tensor(w["WL"][0], dtype=torch.float64), cfg["nF"])
    Xn = torch_ref.block(cfg, w, 0, X)
    assert torch.equal(Xn[:, cfg["nF"]:], lcb)
    assert fin.shape == (8, cfg["n"] * cfg["k"])

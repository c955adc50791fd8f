"""Post-tower batch reductions on the GPU through the C ABI:
correlation_loss (numerics.hpp:46-78) and window_routing_summary (datasets.hpp:256-283), and the
fused routed-objective step, against the CPU oracle (itself pinned to the reference in
tests/test_oracle.py).

Tolerances: window counts / positives and routed logits are bit-exact; the fp64 correlation
loss differs from the sequential reference only by summation order: |gpu - oracle| <= 1e-12
(absolute, the loss is in [0, 2]). The GPU result is deterministic (fixed-order partials)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_correlation_loss_known_answers_and_columns():
    import torch
    import paper_2512_09200_b200 as L
    from test_oracle import CORR_CASES
    for x, y, eps, want, tol in CORR_CASES:
        got = L.correlation_loss(torch.tensor(x, dtype=torch.float64, device="cuda"),
                                 torch.tensor(y, dtype=torch.float64, device="cuda"), eps)
        assert abs(float(got[0]) - want) <= tol
    rng = np.random.default_rng(1)
    n, cols = 100_003, 5
    x = rng.normal(size=(n, cols))
    y = 0.5 * x + rng.normal(size=(n, cols)) * np.arange(1, cols + 1)
    x[:, 4] = 3.0  # constant column -> 1.0
    got = L.correlation_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
    again = L.correlation_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
    assert np.array_equal(got, again)  # deterministic
    for c in range(cols):
        rc, want = oracle.correlation_loss(x[:, c], y[:, c])
        assert rc == 0 and abs(got[c] - want) <= 1e-12
    assert got[4] == 1.0


def test_correlation_loss_contract():
    import torch
    import paper_2512_09200_b200 as L
    one = torch.ones(1, dtype=torch.float64, device="cuda")
    two = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")
    with pytest.raises(L.UsageError):
        L.correlation_loss(one, one)
    with pytest.raises(L.UsageError):
        L.correlation_loss(two, two, eps=0.0)
    with pytest.raises(L.DataError):
        L.correlation_loss(torch.tensor([1.0, float("nan")], dtype=torch.float64, device="cuda"), two)


def test_window_summary_bit_exact_and_contract():
    import torch
    import paper_2512_09200_b200 as L
    rng = np.random.default_rng(2)
    n, T, W = 70_001, 4, 3
    window = rng.integers(0, W, n).astype(np.uint8)
    labels = (rng.random((n, T, W)) < 0.25).astype(np.uint8)
    counts, pos = L.window_summary(torch.from_numpy(window).cuda(), torch.from_numpy(labels).cuda(), W)
    rc, c0, p0 = oracle.window_summary(window, labels, W)
    assert rc == 0 and np.array_equal(counts.cpu().numpy(), c0) and np.array_equal(pos.cpu().numpy(), p0)
    window[123] = W
    with pytest.raises(L.UsageError):
        L.window_summary(torch.from_numpy(window).cuda(), torch.from_numpy(labels).cuda(), W)


def test_routed_objectives_on_zipper_output():
    """Zipper (K5) window + labels of a synthetic impression log, random tower logits."""
    import torch
    import paper_2512_09200_b200 as L
    n, T = 50_000, 4
    dur, pr = [5400000, 86400000, 604800000], [1 / 3, 1 / 3, 1 / 3]
    W = len(dur)
    imp = L.synth_impressions(n, T, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, dur, pr, 7)
    g = torch.Generator(device="cuda").manual_seed(4)
    logits = torch.randn((n, T * W), device="cuda", generator=g)
    routed, corr, counts, pos = L.routed_objectives(logits, win, lab, T, W)
    rc, r0, c0, n0, p0 = oracle.routed_objectives(logits.cpu().numpy(), win.cpu().numpy(), lab.cpu().numpy())
    assert rc == 0
    assert np.array_equal(routed.cpu().numpy(), r0)
    assert np.array_equal(counts.cpu().numpy(), n0) and np.array_equal(pos.cpu().numpy(), p0)
    assert np.abs(corr.cpu().numpy() - c0).max() <= 1e-12
    # the route_heads kernel agrees with the fused routing
    assert torch.equal(L.route_heads(logits, win, T, W), routed)

"""Backward of the network's trainable head on the GPU.

  * lattice_rownorm_vjp is the adjoint of the reference's own swish_rn_jvp (numerics.hpp:113-136,
    compiled in place: oracle/_ref): <g, J t> = <J^T g, t> to fp64 rounding, for swish_rn; rms_norm
    and swish_rn_hard against central differences of the reference's functions.
  * lattice_routed_bce against an fp64 numpy restatement (loss and every dlogit).
  * lattice_net_tower_backward (dW1, dW2, dX) against a torch fp64 restatement of the towers'
    backward on the GPU's own X_L, with the GPU's one rounding point (dz stored bf16 for the
    GEMMs) applied, under netcheck.calibrated (2x the deviation of the same restatement in fp32).
  * TowerTrainer (train.py): SGD steps on a fixed batch lower the routed loss; the network's tower
    weights equal the bf16 rounding of the fp32 masters after each step.
"""
import numpy as np
import pytest

import oracle
import torch_ref
from netcheck import calibrated, record
from test_network_gpu import SMALL, build

pytestmark = pytest.mark.gpu


def test_vjp_is_the_adjoint_of_the_reference_jvp():
    import torch
    import paper_2512_09200_b200 as L
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle.load_ref()
    rng = np.random.default_rng(11)
    for width in (1, 7, 128, 2048):
        for scale in (1e-3, 1.0, 1e4):
            x = rng.normal(size=(4, width)) * scale
            t = rng.normal(size=(4, width))
            g = rng.normal(size=(4, width))
            vjp = L.rownorm_vjp(torch.from_numpy(x).cuda(), torch.from_numpy(g).cuda(), mode=1).cpu().numpy()
            for r in range(4):
                rc, jt = oracle.swish_rn_jvp(x[r], t[r], lib=ref)
                assert rc == 0
                lhs, rhs = float(g[r] @ jt), float(vjp[r] @ t[r])
                # fp64 rounding relative to the Jacobian's scale 1/d: J cancels the component along x
                # down to eps/d^3 (all of it at width 1), on both sides alike
                d = np.sqrt(np.mean(x[r] ** 2) + 1e-6)
                tol = 1e-12 * np.linalg.norm(g[r]) * np.linalg.norm(t[r]) / d
                assert abs(lhs - rhs) <= tol, (width, scale, lhs, rhs)
    # rms_norm (mode 0) and swish_rn_hard (mode 2): central differences of the reference functions
    for mode, name in ((0, "ref_rms_norm"), (2, "ref_swish_rn_hard")):
        x = rng.normal(size=(3, 96))
        x[:, :5] = [3.5, -3.5, 2.9, -2.9, 0.1]  # hard gate: both clamps and the linear zone
        t = rng.normal(size=(3, 96))
        g = rng.normal(size=(3, 96))
        vjp = L.rownorm_vjp(torch.from_numpy(x).cuda(), torch.from_numpy(g).cuda(), mode=mode).cpu().numpy()
        h = 1e-6
        for r in range(3):
            _, fp = oracle.vec_op(ref, name, x[r] + h * t[r])
            _, fm = oracle.vec_op(ref, name, x[r] - h * t[r])
            jt = (fp - fm) / (2 * h)
            assert abs(float(g[r] @ jt) - float(vjp[r] @ t[r])) <= 1e-6 * np.linalg.norm(g[r]) * np.linalg.norm(jt)
    # fp32 path against fp64
    x = rng.normal(size=(64, 512))
    g = rng.normal(size=(64, 512))
    v64 = L.rownorm_vjp(torch.from_numpy(x).cuda(), torch.from_numpy(g).cuda(), mode=1)
    v32 = L.rownorm_vjp(torch.from_numpy(x).float().cuda(), torch.from_numpy(g).float().cuda(), mode=1)
    torch.testing.assert_close(v32.double(), v64, rtol=1e-4, atol=1e-6)


def test_routed_bce_matches_fp64():
    import torch
    import paper_2512_09200_b200 as L
    n, T, W = 3000, 4, 3
    g = torch.Generator(device="cuda").manual_seed(2)
    logits = torch.randn((n, T * W), generator=g, device="cuda") * 3
    window = torch.randint(0, W, (n,), generator=g, device="cuda").to(torch.uint8)
    labels = (torch.rand((n, T, W), generator=g, device="cuda") < 0.3).to(torch.uint8)
    loss, dl = L.routed_bce(logits, window, labels, T, W)
    z = logits.double().cpu().numpy().reshape(n, T, W)
    w = window.cpu().numpy().astype(np.int64)
    y = labels.cpu().numpy().astype(np.float64)
    zr = z[np.arange(n), :, w]           # [n, T]
    yr = y[np.arange(n), :, w]
    want = np.mean(np.log1p(np.exp(-np.abs(zr))) + np.maximum(zr, 0) - zr * yr)
    assert abs(float(loss) - want) <= 1e-6 * abs(want)
    wd = np.zeros((n, T, W))
    wd[np.arange(n), :, w] = (1 / (1 + np.exp(-zr)) - yr) / (n * T)
    np.testing.assert_allclose(dl.double().cpu().numpy().reshape(n, T, W), wd, rtol=1e-5, atol=1e-10)


def tower_backward_ref(cfg, w, X, dom, dlogits, acc, hard=False):
    """Manual backward of towers(X) in `acc` arithmetic, dz rounded to bf16 as the GPU stores it."""
    import torch
    G, th = cfg["domains"], cfg["tower_hidden"]
    X = X.to(acc)
    dlog = dlogits.to(acc)
    dW1 = torch.zeros((G, th, X.shape[1]), dtype=acc, device=X.device)
    dW2 = torch.zeros((G, cfg["heads"], th), dtype=acc, device=X.device)
    dX = torch.zeros_like(X)
    with torch_ref.accumulate(acc):
        for g in range(G):
            m = dom == g
            if not bool(m.any()):
                continue
            W1 = torch_ref._t(w["T1"][g], X.device)
            W2 = torch_ref._t(w["T2"][g], X.device)
            z = (X[m] @ W1.T).detach().requires_grad_(True)
            h = torch_ref.act(z, hard)
            dh = dlog[m] @ W2
            (dz,) = torch.autograd.grad(h, z, dh)
            dzq = dz.float().bfloat16().to(acc)
            dW2[g] = dlog[m].T @ h.detach()
            dW1[g] = dzq.T @ X[m]
            dX[m] = dzq @ W1
    return dW1, dW2, dX


def test_tower_backward_matches_restatement():
    import torch
    cfg, B, rows = SMALL, 1000, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(4)
    dlogits = torch.randn(logits.shape, generator=g, device="cuda") / B
    dW1, dW2, dX = net.tower_backward(dlogits, dx_dtype=torch.float32)
    w = net.weights()
    XL = net.activations(cfg["blocks"], B).reshape(B, -1)          # caller order
    pos = torch.as_tensor(L_view_pos(net, B), device="cuda").long()
    dX_caller = dX[pos]
    d = dom.cuda().long()
    r64 = tower_backward_ref(cfg, w, XL, d, dlogits, torch.float64)
    r32 = tower_backward_ref(cfg, w, XL, d, dlogits, torch.float32)
    for name, got, a, b in (("dW1", dW1, r64[0], r32[0]), ("dW2", dW2, r64[1], r32[1]), ("dX", dX_caller, r64[2], r32[2])):
        scale = float(a.abs().max())
        calibrated(f"tower backward {name}", got, a, b, atol=1e-3 * scale, rtol=1e-3, mean_floor=1e-5 * scale)
    # deterministic: a second backward is bit-identical
    dW1b, dW2b, _ = net.tower_backward(dlogits)
    assert torch.equal(dW1b, dW1) and torch.equal(dW2b, dW2)


def L_view_pos(net, B):
    import torch
    import paper_2512_09200_b200 as L
    return torch.as_tensor(L._CAI(net.buffer(1), (B,), "<i4"), device="cuda").clone()


def test_tower_training_lowers_routed_loss():
    import torch
    import paper_2512_09200_b200 as L
    from paper_2512_09200_b200.train import TowerTrainer
    cfg = dict(SMALL, heads=12)  # 4 objectives x 3 windows
    B, rows = 2048, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    imp = L.synth_impressions(B, 4, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    tr = TowerTrainer(net, lr=2.0)
    losses = []
    for _ in range(6):
        logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
        losses.append(float(tr.step(logits, win, lab, 4, 3)))
        W1, _ = net.tower_masters()
        assert torch.equal(W1, tr.W1.bfloat16().float())  # the net runs the bf16 rounding of the master
    record("tower training: routed BCE per step", {"losses": losses})
    assert losses[-1] < losses[0] * 0.95, losses


def mlp_backward_ref(cfg, w, Fin, Xin, dXout, acc, hard=False):
    """Autograd of <rms_norm_d(z_last + X[:nF]), dX_L[:nF]> through the last block's MLP in `acc`
    arithmetic, from the GPU's own Fin and X_{L-1} (domain-sorted rows): the hidden activations
    q()-rounded as the forward stores them, every layer's d(loss)/dz rounded to bf16 by a hook
    (the GPU's GEMM-operand rounding). Returns ([dW_i], dFin, dResid)."""
    import torch
    n, d, nF = cfg["n"], cfg["d"], cfg["nF"]
    n_mlp = len(cfg["mlp"]) - 1
    blk = cfg["blocks"] - 1
    S = Fin.shape[0]
    with torch_ref.accumulate(acc):
        a = Fin.to(acc).detach().requires_grad_(True)
        Ws = [torch_ref._t(w["mlp"][blk * n_mlp + i], Fin.device).requires_grad_(True) for i in range(n_mlp)]
        h = a
        for i in range(n_mlp):
            z = h @ Ws[i].T
            z.register_hook(lambda g: g.float().bfloat16().to(g.dtype))
            if i + 1 < n_mlp:  # straight-through q(): autograd through .bfloat16() would round the
                h = torch_ref.act(z, hard)  # gradient to bf16 too, which the GPU does not
                h = h + (torch_ref.q(h, True) - h).detach()
        Xr = Xin.to(acc).reshape(S, n, d)[:, :nF].detach().requires_grad_(True)
        out = torch_ref.rms_norm(z.reshape(S, nF, d) + Xr)
        loss = (out * dXout.to(acc).reshape(S, n, d)[:, :nF]).sum()
        grads = torch.autograd.grad(loss, Ws + [a, Xr])
    return list(grads[:n_mlp]), grads[n_mlp], grads[n_mlp + 1].reshape(S, nF * d)


@pytest.mark.parametrize("mlp,hard", [([1024, 512, 4096], False), ([1024, 384, 256, 512, 4096], True)])
def test_mlp_backward_matches_restatement(mlp, hard):
    """lattice_net_mlp_backward against autograd of the torch restatement (fp64; calibrated by the
    same in fp32). The 4-layer MLP takes the re-run path (its first hidden output is overwritten by
    the forward's ping-pong)."""
    import torch
    import paper_2512_09200_b200 as L
    cfg = dict(SMALL, mlp=mlp)
    B, rows = 1000, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows, hard=hard)
    net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
    n, d, k, nb = cfg["n"], cfg["d"], cfg["k"], cfg["blocks"]
    Fin = L._view(net.buffer(3), (B, n * k), torch.bfloat16).clone()
    Xin = L._view(net.buffer(2 if (nb - 1) & 1 else 0), (B, n * d), torch.bfloat16).clone()
    g = torch.Generator(device="cuda").manual_seed(5)
    dXout = torch.randn((B, n * d), generator=g, device="cuda") / B
    dW, dFin, dRes = net.mlp_backward(dXout, dFin=True, dResid=True)
    # the forward's buffers are untouched by the backward (the re-run is bit-identical)
    assert torch.equal(L._view(net.buffer(3), (B, n * k), torch.bfloat16), Fin)
    w = net.weights()
    r64 = mlp_backward_ref(cfg, w, Fin, Xin, dXout, torch.float64, hard)
    r32 = mlp_backward_ref(cfg, w, Fin, Xin, dXout, torch.float32, hard)
    pairs = [(f"dW{i}", dW[i], r64[0][i], r32[0][i]) for i in range(len(dW))]
    pairs += [("dFin", dFin, r64[1], r32[1]), ("dResid", dRes, r64[2], r32[2])]
    for name, got, a, b in pairs:
        scale = float(a.abs().max())
        calibrated(f"mlp backward ({len(mlp) - 1} layers, hard={hard}) {name}", got, a, b, atol=1e-3 * scale,
                   rtol=1e-3, mean_floor=1e-5 * scale)
    # deterministic
    dW2, _, _ = net.mlp_backward(dXout)
    assert all(torch.equal(x, y) for x, y in zip(dW, dW2))


def test_tower_and_mlp_training_lowers_routed_loss():
    import torch
    import paper_2512_09200_b200 as L
    from paper_2512_09200_b200.train import TowerTrainer
    cfg = dict(SMALL, heads=12)
    B, rows = 2048, 3000
    net, tab, ptrs, rws, offsets, ids, dom = build(cfg, B, rows)
    imp = L.synth_impressions(B, 4, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    tr = TowerTrainer(net, lr=2.0, train_mlp=True)
    losses = []
    for _ in range(6):
        logits = net.forward(dom, offsets, ids, ptrs, rws, torch.bfloat16)
        losses.append(float(tr.step(logits, win, lab, 4, 3)))
        for i, m in enumerate(net.mlp_masters()):
            assert torch.equal(m, tr.mlp[i].bfloat16().float())
    record("tower + last-block MLP training: routed BCE per step", {"losses": losses})
    assert losses[-1] < losses[0] * 0.95, losses

"""Second, independent restatement of the network arithmetic in torch
fp64 -- test infrastructure only, like oracle/.

oracle/lattice_oracle.c (forward_one) is a scalar, one-sample-at-a-time C loop nest; this is a
batched einsum formulation written separately from the same definition:
  X0 = q(rms_norm_d(pooled))
  per block: P = q(X^T Y); F = X P; h = q(rms_norm(flatten F))         PAPER.md:292 (FMB)
             h <- q(swish_rn(W h)) for hidden layers, z = W_last h
             X'[:nF] = q(rms_norm_d(z + X[:nF])); X'[nF:] = q(rms_norm_d(W_L X + X[nF:]))  (LCB)
  tower:     logits = W2_g . swish_rn(W1_g . flatten X), g = domain
  dense processor: rows [n - dense_features, n) of the pooled input are
             q(D2 . q(swish_rn(D1 . x_dense))) before the mixing norm.
q() = round to bf16 through fp32 (the C oracle's lo_bf16_round((float)v)), or to fp32.
rms_norm / swish_rn / swish_rn_hard follow numerics.hpp:81-107 (eps 1e-6).

The tests cross-check this against the C oracle on the CPU (two restatements agreeing is the
best pin available where no reference code exists: SURVEY.md section 0) and then use it on the
GPU (torch fp64) to check EVERY logit of a batch against the CUDA path.
"""
import contextlib

import torch

EPS = 1e-6
ACC = torch.float64  # arithmetic dtype (fp64; accumulate(torch.float32) models the GPU's fp32 sums)


@contextlib.contextmanager
def accumulate(dtype, tf32=False):
    """Run the restatement in another arithmetic dtype (same rounding points): fp32 gives the
    size of the differences fp32 accumulation alone makes against fp64 -- the error budget the
    GPU path is held to. tf32=True also runs its matmuls on TF32 tensor cores (10-bit mantissa
    operands: the budget of the network's fp32-storage / kind::tf32 mode)."""
    global ACC
    old, ACC = ACC, dtype
    old_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32
    try:
        yield
    finally:
        ACC = old
        torch.backends.cuda.matmul.allow_tf32 = old_tf32


def q(x, bf16):
    return x.float().bfloat16().to(ACC) if bf16 else x.float().to(ACC)


def rms_norm(x, dim=-1):
    return x / torch.sqrt((x * x).mean(dim=dim, keepdim=True) + EPS)


def act(x, hard):
    r = rms_norm(x)
    if hard:
        return r * ((r + 3.0) / 6.0).clamp(0.0, 1.0)
    return r * torch.sigmoid(r)


def _t(a, device):
    return torch.as_tensor(a).to(device=device, dtype=ACC)


def dense_rows(cfg, w, dense, bf16=True, hard=False, device="cpu"):
    """Dense processor output rows [S, dense_features, d] (before the mixing norm)."""
    x = _t(dense, device)
    h = q(act(x @ _t(w["D1"], device).T, hard), bf16)
    o = q(h @ _t(w["D2"], device).T, bf16)
    return o.view(x.shape[0], cfg["dense_features"], cfg["d"])


def block(cfg, w, blk, X, bf16=True, hard=False, device="cpu"):
    """One DWFB block on X [S, n, d] (fp64, already q()-rounded) -> X' [S, n, d]."""
    n, nF, nL = cfg["n"], cfg["nF"], cfg["nL"]
    n_mlp = len(cfg["mlp"]) - 1
    S = X.shape[0]
    YT = _t(w["YT"][blk], device)       # [k, n]
    P = q(torch.einsum("snc,jn->scj", X, YT), bf16)  # [S, d, k]
    F = torch.einsum("snc,scj->snj", X, P)           # [S, n, k]
    h = q(rms_norm(F.reshape(S, -1)), bf16)
    for li in range(n_mlp):
        z = h @ _t(w["mlp"][blk * n_mlp + li], device).T
        if li + 1 < n_mlp:
            h = q(act(z, hard), bf16)
    out = torch.empty_like(X)
    out[:, :nF] = q(rms_norm(z.view(S, nF, -1) + X[:, :nF]), bf16)
    if nL:
        WL = _t(w["WL"][blk], device)   # [nL, n]
        out[:, nF:] = q(rms_norm(torch.einsum("in,snc->sic", WL, X) + X[:, nF:]), bf16)
    return out


def fm_lcb(X, YT, WL, nF, bf16=True):
    """K2 alone: (Fin [S, n*k], LCB rows [S, nL, d]) from X [S, n, d] fp64."""
    S = X.shape[0]
    P = q(torch.einsum("snc,jn->scj", X, YT), bf16)
    F = torch.einsum("snc,scj->snj", X, P)
    fin = q(rms_norm(F.reshape(S, -1)), bf16)
    lcb = q(rms_norm(torch.einsum("in,snc->sic", WL, X) + X[:, nF:]), bf16)
    return fin, lcb


def forward(cfg, w, pooled, dom, dense=None, bf16=True, hard=False, device="cpu", chunk=None):
    """logits [S, heads] (fp64) for raw pooled sums [S, n - dense_features, d] and domains [S].
    chunk: samples per pass (bounds fp64 activation memory at large batches)."""
    S = pooled.shape[0]
    chunk = chunk or S
    outs = []
    for s0 in range(0, S, chunk):
        s1 = min(S, s0 + chunk)
        x = _t(pooled[s0:s1], device)
        if cfg.get("dense_features"):
            x = torch.cat([x, dense_rows(cfg, w, dense[s0:s1], bf16, hard, device)], dim=1)
        X = q(rms_norm(x), bf16)
        for blk in range(cfg["blocks"]):
            X = block(cfg, w, blk, X, bf16, hard, device)
        outs.append(towers(cfg, w, X, torch.as_tensor(dom[s0:s1]).to(device), hard, device))
    return torch.cat(outs)


def towers(cfg, w, X, dom, hard=False, device="cpu"):
    S = X.shape[0]
    Xf = X.reshape(S, -1)
    out = torch.zeros((S, cfg["heads"]), dtype=ACC, device=device)
    for g in range(cfg["domains"]):
        m = dom == g
        if not bool(m.any()):
            continue
        h = act(Xf[m] @ _t(w["T1"][g], device).T, hard)
        out[m] = h @ _t(w["T2"][g], device).T
    return out

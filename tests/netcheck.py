"""Shared helpers of the network parity tests (test infrastructure: they drive the two
restatements -- oracle/lattice_oracle.c and tests/torch_ref.py -- and record the observed
errors).

How the bf16 network is held to the fp64 restatement. The GPU accumulates
in fp32 (TMEM, epilogue registers) where the restatement accumulates in fp64; at every bf16
rounding point (P, Fin, hidden activations, X') an element whose fp64 value sits near a rounding
boundary may round the other way, and those one-ulp flips propagate through the later blocks.
The size of that effect is measured, not assumed: the same restatement run with fp32 arithmetic
(torch_ref.accumulate(torch.float32), same rounding points) deviates from the fp64 one by
`noise` on the same inputs. The CUDA path must satisfy, on EVERY logit / element,
    |gpu - ref64| <= max(atol + rtol |ref64|, 2 max(noise))
and on average
    mean |gpu - ref64| <= 2 mean(noise) + 1e-5
-- i.e. it may differ from fp64 by at most twice what fp32 accumulation alone explains. The mean
bound is the sharp one: a 1% error in one weight matrix moves the mean error 20x past it at the
small config (test_network_gpu.py test_error_is_not_vacuous). atol = rtol = 5e-3 at the logits.
Observed values are logged per config (PARITY_LOG=<file>) and committed under profiles/.
"""
import json
import os

import numpy as np

import oracle

ATOL = RTOL = 5e-3


def host_weights(cfg, seed):
    """Every weight of a Network config from the counter-based generator on the host (fp32
    arrays, bf16-exact), in the layout Network.weights() returns."""
    lib = oracle.load_oracle()

    def tensor(block, kind, index, out_f, fan_in):
        buf = np.zeros((out_f, fan_in), np.float32)
        lib.lo_fill_weights(oracle.ptr(buf), out_f, fan_in, seed, lib.lo_weight_tag(block, kind, index))
        return buf

    w = {"YT": [], "WL": [], "mlp": []}
    for blk in range(cfg["blocks"]):
        w["YT"].append(tensor(blk, 1, 0, cfg["k"], cfg["n"]))
        w["WL"].append(tensor(blk, 2, 0, cfg["nL"], cfg["n"]))
        for li in range(len(cfg["mlp"]) - 1):
            w["mlp"].append(tensor(blk, 3, li, cfg["mlp"][li + 1], cfg["mlp"][li]))
    nd = cfg["n"] * cfg["d"]
    w["T1"] = np.stack([tensor(g, 4, 0, cfg["tower_hidden"], nd) for g in range(cfg["domains"])])
    w["T2"] = np.stack([tensor(g, 5, 0, cfg["heads"], cfg["tower_hidden"]) for g in range(cfg["domains"])])
    if cfg.get("dense_features"):
        w["D1"] = tensor(0, 6, 0, cfg["dense_hidden"], cfg["dense_in"])
        w["D2"] = tensor(0, 7, 0, cfg["dense_features"] * cfg["d"], cfg["dense_hidden"])
    return w


def oracle_forward(cfg, w, pooled, dom, dense=None, bf16=True, hard=False, threads=0):
    """C oracle logits: pooled raw sums [S, n - dense_features, d] (+ the dense processor rows)."""
    S, nc, d = pooled.shape
    n = cfg["n"]
    full = np.zeros((S, n, d), np.float32)
    full[:, :nc] = pooled
    if cfg.get("dense_features"):
        c = oracle.LoNetCfg()
        c.n, c.d, c.blocks, c.nF, c.nL, c.k = n, d, cfg["blocks"], cfg["nF"], cfg["nL"], cfg["k"]
        c.n_mlp = len(cfg["mlp"]) - 1
        for i, v in enumerate(cfg["mlp"]):
            c.mlp[i] = v
        c.G, c.heads, c.tower_hidden, c.hard, c.bf16 = cfg["domains"], cfg["heads"], cfg["tower_hidden"], int(hard), int(bf16)
        oracle.dense_processor(c, cfg["dense_features"], cfg["dense_in"], cfg["dense_hidden"], w["D1"], w["D2"],
                               dense, full, threads)
    return oracle.net_forward(cfg, w, full, dom, bf16=bf16, hard=hard, threads=threads)


def stats(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want)
    return {"count": int(err.size), "max_abs": float(err.max()), "mean_abs": float(err.mean()),
            "worst_ratio": float((err / (ATOL + RTOL * np.abs(want))).max()),
            "rms_logit": float(np.sqrt((want ** 2).mean()))}


def record(name, st):
    """Append the observed errors of one check to $PARITY_LOG (JSON lines), and print them."""
    print(f"[parity] {name}: {json.dumps(st)}")
    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(dict(name=name, **st)) + "\n")


def assert_close(name, got, want, atol=ATOL, rtol=RTOL):
    st = stats(got, want)
    record(name, st)
    err = np.abs(np.asarray(got, np.float64) - np.asarray(want, np.float64))
    bound = atol + rtol * np.abs(np.asarray(want, np.float64))
    assert np.isfinite(got).all()
    assert (err <= bound).all(), f"{name}: max err {st['max_abs']:.4g} (worst ratio {(err / bound).max():.3g})"
    return st


def calibrated(name, got, ref64, ref32, atol=ATOL, rtol=RTOL, mean_floor=1e-5):
    """The calibrated bound of the module docstring; got / ref64 / ref32 numpy or torch."""
    to = lambda a: np.asarray(a.double().cpu() if hasattr(a, "double") else a, np.float64)
    got, ref64, ref32 = to(got), to(ref64), to(ref32)
    err = np.abs(got - ref64)
    noise = np.abs(ref32 - ref64)
    cap = max(2 * float(noise.max()), 0.0)
    bound = np.maximum(atol + rtol * np.abs(ref64), cap)
    st = {"count": int(err.size), "max_abs": float(err.max()), "mean_abs": float(err.mean()),
          "noise_max": float(noise.max()), "noise_mean": float(noise.mean()),
          "worst_ratio": float((err / bound).max()),
          "mean_ratio": float(err.mean() / (2 * noise.mean() + mean_floor)),
          "frac_not_identical": float((got != ref64).mean()),
          "rms_ref": float(np.sqrt((ref64 ** 2).mean()))}
    record(name, st)
    assert np.isfinite(got).all(), name
    assert (err <= bound).all(), f"{name}: {st}"
    assert st["mean_ratio"] <= 1.0, f"{name}: {st}"
    return st

"""K2 at kernel level (lattice_fm_lcb): Fin = q(rms_norm(flatten(X . q(X^T Y)))) and the LCB half
of X' = q(rms_norm_d(W_L X + X[nF:])) from fm_lcb_kernel (n <= 256, bf16 and fp32/tf32) and
fm_lcb_large_kernel (256 < n <= 512), against the torch fp64 restatement (tests/torch_ref.py
fm_lcb) on the same inputs, B >= 512.

Two input families:
  * exact-arithmetic inputs (X, Y, W_L small integers times powers of two): P = X^T Y is exact in
    bf16 and F = X P, W_L X are exact in fp32, so each output is ONE rounding of a value both
    sides compute alike up to the fp32 vs fp64 rms_norm -- every element within one ulp of the
    reference (|gpu - ref| <= 2^-7 |ref| + 1e-6 for bf16) and at most 0.1% of them off its rounding;
  * realistic inputs (rms-normalised random X, generator-scaled weights): here P's own bf16
    rounding can flip between fp32 and fp64 accumulation and the flip propagates into F, so the
    bound is netcheck.calibrated's (twice the deviation of the same restatement run in fp32).
fp32 storage on kind::tf32: the MMAs read operands with a 10-bit mantissa: 2^-9 |ref| + 1e-3."""
import numpy as np
import pytest

import torch_ref
from netcheck import calibrated, record

pytestmark = pytest.mark.gpu


def make(B, n, d, k, nL, dtype, seed=11, exact=False):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    if exact:  # |X| in {0, 1/2, 1}, Y and W_L in {-1, 0, 1} / 16: every product and sum exact
        X = (torch.randint(-2, 3, (B, n, d), generator=g, device="cuda").double() / 2).to(dtype)
        YT = (torch.randint(-1, 2, (k, n), generator=g, device="cuda").double() / 16).to(dtype)
        WL = (torch.randint(-1, 2, (nL, n), generator=g, device="cuda").double() / 16).to(dtype)
        return X, YT, WL
    raw = torch.randn((B, n, d), generator=g, device="cuda", dtype=torch.float64)
    X = torch_ref.q(torch_ref.rms_norm(raw), dtype == torch.bfloat16).to(dtype)
    scale = 2.0 ** -(7 + int(np.log2(n)) // 2)  # the generator's fan-in scaling
    YT = (torch.randint(-128, 128, (k, n), generator=g, device="cuda").double() * scale).to(dtype)
    WL = (torch.randint(-128, 128, (nL, n), generator=g, device="cuda").double() * scale).to(dtype)
    return X, YT, WL


def check_exact(name, got, want, bf16):
    got = got.double()
    err = (got - want).abs()
    ulp_rel, floor = (2.0 ** -7, 1e-6) if bf16 else (2.0 ** -9, 1e-3)
    bound = ulp_rel * want.abs() + floor
    off = (got != want).double().mean().item()
    st = {"count": int(err.numel()), "max_abs": err.max().item(), "frac_not_identical": off,
          "worst_ratio": (err / bound).max().item()}
    record(name, st)
    assert (err <= bound).all(), f"{name}: {st}"
    if bf16:
        assert off <= 1e-3, f"{name}: {st}"


CASES = [
    (256, 128, 32, 128, 1024, "bf16"),   # mid block (fm_lcb_kernel)
    (64, 128, 16, 32, 777, "bf16"),      # small, ragged batch
    (24, 64, 16, 12, 600, "bf16"),       # d = 64, n not a multiple of 16
    (8, 64, 4, 4, 512, "f32"),           # tiny config, fp32 storage on kind::tf32
    (512, 128, 32, 256, 640, "bf16"),    # large block (fm_lcb_large_kernel)
    (512, 128, 32, 256, 641, "bf16"),    # odd batch (the pair variant's last pair has one sample)
    (512, 128, 32, 288, 512, "bf16"),    # nL = 224
    (384, 128, 16, 256, 512, "bf16"),    # zero-padded n, nL = 128, k = 16
    (400, 128, 32, 200, 512, "bf16"),    # nF, nL not multiples of 32: warps with live and dead lanes
    (512, 128, 48, 256, 512, "bf16"),    # k = 48
]
PAIR_CASES = ["512-128-32-256-640-bf16", "512-128-32-256-641-bf16", "512-128-32-288-512-bf16",
              "384-128-16-256-512-bf16"]


@pytest.mark.parametrize("n,d,k,nF,B,dtype", CASES)
def test_fm_lcb_exact_inputs_one_rounding(n, d, k, nF, B, dtype):
    import torch
    import paper_2512_09200_b200 as L
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    bf16 = dt == torch.bfloat16
    X, YT, WL = make(B, n, d, k, n - nF, dt, exact=True)
    Fin, Xout = L.fm_lcb(X, YT, WL, nF)
    fin_ref, lcb_ref = torch_ref.fm_lcb(X.double(), YT.double(), WL.double(), nF, bf16=bf16)
    tag = f"K2 exact n{n} d{d} k{k} nF{nF} B{B} {dtype}"
    check_exact(tag + " Fin", Fin, fin_ref, bf16)
    check_exact(tag + " LCB rows", Xout[:, nF:], lcb_ref, bf16)
    assert torch.count_nonzero(Xout[:, :nF]) == 0  # rows [0, nF) belong to the MLP epilogue


@pytest.mark.parametrize("n,d,k,nF,B,dtype", CASES)
def test_fm_lcb_realistic_inputs_calibrated(n, d, k, nF, B, dtype):
    import torch
    import paper_2512_09200_b200 as L
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    bf16 = dt == torch.bfloat16
    X, YT, WL = make(B, n, d, k, n - nF, dt)
    Fin, Xout = L.fm_lcb(X, YT, WL, nF)
    refs = {}
    for acc in (torch.float64, torch.float32):
        with torch_ref.accumulate(acc, tf32=acc == torch.float32 and not bf16):
            refs[acc] = torch_ref.fm_lcb(X.to(acc), YT.to(acc), WL.to(acc), nF, bf16=bf16)
    tag = f"K2 n{n} d{d} k{k} nF{nF} B{B} {dtype}"
    ulp, floor = (2.0 ** -7, 1e-3) if bf16 else (2.0 ** -9, 1e-3)
    calibrated(tag + " Fin", Fin, refs[torch.float64][0], refs[torch.float32][0], atol=floor, rtol=ulp)
    calibrated(tag + " LCB rows", Xout[:, nF:], refs[torch.float64][1], refs[torch.float32][1], atol=floor,
               rtol=ulp)


def test_fm_lcb_pair_kernel():
    """The opt-in CTA-pair variant (LATTICE_FM_PAIR=1, read once per process) on its shapes, both
    input families, in a subprocess."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, LATTICE_FM_PAIR="1")
    f = os.path.join(here, "test_fm_lcb_gpu.py")
    ids = [f"{f}::{t}[{c}]" for c in PAIR_CASES
           for t in ("test_fm_lcb_exact_inputs_one_rounding", "test_fm_lcb_realistic_inputs_calibrated")]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *ids], env=env,
                       capture_output=True, text=True, timeout=600, cwd=os.path.dirname(here))
    assert r.returncode == 0 and f"{len(ids)} passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


def test_fm_lcb_contract():
    import torch
    import paper_2512_09200_b200 as L
    X, YT, WL = make(4, 64, 128, 16, 32, torch.bfloat16)
    with pytest.raises(L.UsageError):
        L.fm_lcb(X, YT, WL, 40)  # nF + nL != n
    X96 = torch.zeros((4, 64, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.UsageError):
        L.fm_lcb(X96, YT, WL, 32)  # d must be 64 or 128
    fin, xo = L.fm_lcb(X[:0], YT, WL, 32)  # empty batch: nothing launched
    assert fin.shape == (0, 64 * 16)

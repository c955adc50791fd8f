"""K5 Zipper parity on the GPU, through the C ABI, bit-exact against the oracle and the
reference itself (oracle/_ref/libref.so, the proj/include headers compiled in place) and
the committed reference fixtures (tests/golden/zipper_ref.json)."""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def to_dev(users, ads, ts, conv, pres):
    import torch
    ub, uo = oracle.pack_strings(users)
    ab, ao = oracle.pack_strings(ads)
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
    return (d(ub, np.uint8), d(uo, np.int64), d(ab, np.uint8), d(ao, np.int64), d(ts, np.int64),
            d(conv, np.int64), d(pres, np.uint8))


def run_gpu(users, ads, ts, conv, pres, dur, probs, seed, **kw):
    import paper_2512_09200_b200 as L
    cols = to_dev(users, ads, ts, conv, pres)
    w, lab, rt = L.zipper_assign_labels(*cols, dur, probs, seed, **kw)
    return w.cpu().numpy(), lab.cpu().numpy(), (rt.cpu().numpy() if rt is not None else None)


def random_records(rng, n, T, conv_lo=0):
    users = [bytes(rng.integers(0, 256, int(rng.integers(0, 70)), dtype=np.uint8)) for _ in range(n)]
    ads = [bytes(rng.integers(0, 256, int(rng.integers(0, 70)), dtype=np.uint8)) for _ in range(n)]
    ts = rng.integers(-2**50, 2**50, n)
    pres = (rng.random((n, T)) < 0.5).astype(np.uint8)
    conv = ts[:, None] + rng.integers(conv_lo, 9 * 86400000, (n, T))
    return users, ads, ts, conv, pres


def test_stable_hash_goldens_gpu():
    import torch
    import paper_2512_09200_b200 as L
    from test_oracle import XXH_GOLDENS
    for seed in {g[1] for g in XXH_GOLDENS}:
        cases = [g for g in XXH_GOLDENS if g[1] == seed]
        b, o = oracle.pack_strings([c[0] for c in cases])
        h = L.stable_hash(torch.from_numpy(b).cuda(), torch.from_numpy(o).cuda(), seed)
        got = [int(x) & (2**64 - 1) for x in h.cpu().tolist()]
        assert got == [c[2] for c in cases]


def test_reference_fixture_gpu():
    with open(os.path.join(GOLD, "zipper_ref.json")) as f:
        g = json.load(f)
    sigs = g["signatures"]
    users = [bytes.fromhex(c["user"]) for c in sigs]
    ads = [bytes.fromhex(c["ad"]) for c in sigs]
    ts = np.array([c["ts"] for c in sigs], np.int64)
    empty = np.zeros((len(sigs), 0), np.int64)
    for ci, cfg in enumerate(g["configs"]):
        w, _, _ = run_gpu(users, ads, ts, empty, empty, cfg["durations"], cfg["probs"], cfg["seed"])
        assert w.tolist() == [c["windows"][ci] for c in sigs]
    z = g["zip"]
    w, lab, _ = run_gpu([u.encode() for u in z["users"]], [a.encode() for a in z["ads"]],
                        np.array(z["ts"]), np.array(z["conv"]), np.array(z["present"]),
                        z["durations"], z["probs"], z["seed"])
    assert w.tolist() == z["window"] and lab.tolist() == z["labels"]


def test_bit_exact_vs_oracle_and_reference_fuzz():
    rng = np.random.default_rng(42)
    for trial in range(4):
        n, T, W = 20000, int(rng.integers(1, 6)), int(rng.integers(1, 9))
        users, ads, ts, conv, pres = random_records(rng, n, T)
        dur = np.cumsum(rng.integers(1, 2 * 86400000, W))
        p = rng.random(W)
        p /= p.sum()
        w, lab, rt = run_gpu(users, ads, ts, conv, pres, dur, p, 1000 + trial, routed=True)
        ow, ol, err, _ = oracle.zip_columns(users, ads, ts, conv, pres, dur, p, 1000 + trial)
        assert err == -1
        assert (w == ow).all() and (lab == ol).all()
        assert (rt == ol[np.arange(n), :, ow.astype(np.int64)]).all()  # routed = own-window label
        if oracle.ref_available() and trial < 2:
            rc, rw, rl, _ = oracle.ref_zip_dataset(users[:3000], ads[:3000], ts[:3000], conv[:3000],
                                                   pres[:3000], dur, p, 1000 + trial)
            assert rc == 0 and (rw == w[:3000]).all() and (rl == lab[:3000]).all()


def test_first_error_record_matches_reference():
    import paper_2512_09200_b200 as L
    rng = np.random.default_rng(7)
    n, T = 5000, 3
    users, ads, ts, conv, pres = random_records(rng, n, T)
    for bad in [(4321, 2), (17, 1), (4999, 0)]:
        c = conv.copy()
        p = pres.copy()
        c[bad] = ts[bad[0]] - 1
        p[bad] = 1
        c[4500, 0], p[4500, 0] = ts[4500] - 100, 1   # a later offender must not win
        with pytest.raises(L.DataError) as ei:
            run_gpu(users, ads, ts, c, p, [5400000, 86400000], [0.5, 0.5], 7)
        first = min(bad, (4500, 0))
        assert ei.value.index == first[0] * T + first[1]
        assert f"record #{first[0]}" in str(ei.value)
        _, _, err, task = oracle.zip_columns(users, ads, ts, c, p, [5400000, 86400000], [0.5, 0.5], 7)
        assert (err, task) == first


def test_acceptance_distribution_and_monotonicity():
    # SPEC.md:768-769
    n = 100_000
    users = [f"user{i}".encode() for i in range(n)]
    ads = [f"ad{(i * 7919) % 10007}".encode() for i in range(n)]
    ts = 1_700_000_000_000 + np.arange(n, dtype=np.int64)
    empty = np.zeros((n, 0), np.int64)
    w, _, _ = run_gpu(users, ads, ts, empty, empty, [1, 2, 3, 4], [0.4, 0.3, 0.2, 0.1], 2024)
    assert np.bincount(w, minlength=4).tolist() == [40017, 30003, 19839, 10141]
    rng = np.random.default_rng(3)
    users, ads, ts, conv, pres = random_records(rng, n, 2)
    w1, lab1, _ = run_gpu(users, ads, ts, conv, pres, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    w2, lab2, _ = run_gpu(users, ads, ts, conv, pres, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    assert (np.diff(lab1.astype(np.int8), axis=2) >= 0).all()   # longer window => label >= shorter
    assert (w1 == w2).all() and (lab1 == lab2).all()            # determinism


def test_empty_and_degenerate():
    import torch
    import paper_2512_09200_b200 as L
    z = torch.zeros(1, dtype=torch.int64, device="cuda")
    e8 = torch.zeros(0, dtype=torch.uint8, device="cuda")
    w, lab, _ = L.zipper_assign_labels(e8, z, e8, z, torch.zeros(0, dtype=torch.int64, device="cuda"),
                                       torch.zeros((0, 2), dtype=torch.int64, device="cuda"),
                                       torch.zeros((0, 2), dtype=torch.uint8, device="cuda"),
                                       [1, 2], [0.5, 0.5], 7)
    assert w.numel() == 0 and lab.shape == (0, 2, 2)
    with pytest.raises(L.UsageError):
        L.zipper_assign_labels(e8, z, e8, z, torch.zeros(0, dtype=torch.int64, device="cuda"),
                               torch.zeros((0, 2), dtype=torch.int64, device="cuda"),
                               torch.zeros((0, 2), dtype=torch.uint8, device="cuda"),
                               [2, 1], [0.5, 0.5], 7)
    users = [b"x"] * 1000
    ts = np.arange(1000)
    empty = np.zeros((1000, 0), np.int64)
    w, _, _ = run_gpu(users, users, ts, empty, empty, [10, 20], [1.0, 0.0], 5)
    assert (w == 0).all()


def test_synth_impressions_and_head_routing():
    """Device impression generator == oracle generator; Zipper on it == oracle; the window
    mask applied to heads picks logits[b][t*W + window[b]]."""
    import torch
    import paper_2512_09200_b200 as L
    n, T, W = 20000, 4, 3
    cols = L.synth_impressions(n, T, 7)
    users, ads, ts, conv, pres = oracle.synth_impressions(n, T, 7)
    assert cols[0].cpu().numpy().tobytes() == b"".join(users)
    assert cols[2].cpu().numpy().tobytes() == b"".join(ads)
    assert (cols[4].cpu().numpy() == ts).all() and (cols[5].cpu().numpy() == conv).all()
    assert (cols[6].cpu().numpy() == pres).all()
    dur, pr = [5400000, 86400000, 604800000], [1 / 3, 1 / 3, 1 / 3]
    w, lab, rt = L.zipper_assign_labels(*cols, dur, pr, 7, routed=True)
    ow, ol, err, _ = oracle.zip_columns(users, ads, ts, conv, pres, dur, pr, 7)
    assert err == -1 and (w.cpu().numpy() == ow).all() and (lab.cpu().numpy() == ol).all()
    logits = torch.randn((n, T * W), device="cuda")
    routed = L.route_heads(logits, w, T, W)
    idx = torch.arange(T, device="cuda")[None, :] * W + w.long()[:, None]
    assert torch.equal(routed, torch.gather(logits, 1, idx))

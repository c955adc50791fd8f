"""KTAP student-input assembly and the numerics element ops on the GPU
against the CPU oracle, which tests/test_oracle.py pins to the reference's
TeacherEmbeddingStore / student_feature_vector / clip_features / smooth_labels / swish_rn_jvp.

Tolerances: student rows, hits, logits, clip and smoothing bit-exact (fp32 / bf16 rounding of
the same fp64 values); swish_rn_jvp within 1e-13 (fp64, parallel row sums)."""
import numpy as np
import pytest

import oracle
from test_oracle import ktap_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("clip,smoothing,bf16", [(0.0, -1.0, False), (2.0, 0.1, False), (1.5, 0.0, True)])
def test_student_inputs_bit_exact(clip, smoothing, bf16):
    import torch
    import paper_2512_09200_b200 as L
    base, slot, emb, logit, written, ttl, now = ktap_case(n=5000, E=700)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    rows, lg, hit = L.student_inputs(d(base), d(slot), d(emb), d(written), ttl, now, store_logit=d(logit), clip=clip,
                                     smoothing=smoothing, out_dtype=torch.bfloat16 if bf16 else torch.float32)
    want_rows, want_lg, want_hit = oracle.student_inputs(base, slot, emb, logit, written, ttl, now, clip, smoothing,
                                                         bf16=bf16)
    assert np.array_equal(hit.cpu().numpy(), want_hit)
    assert np.array_equal(rows.float().cpu().numpy(), want_rows)
    g = lg.cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(want_lg))
    assert np.array_equal(g[~np.isnan(g)], want_lg[~np.isnan(want_lg)])


def test_student_inputs_contract():
    import torch
    import paper_2512_09200_b200 as L
    base, slot, emb, logit, written, ttl, now = ktap_case(n=10, E=5)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    with pytest.raises(L.UsageError):
        L.student_inputs(d(base), d(slot), d(emb), d(written), 0, now)  # ttl must be positive
    with pytest.raises(L.UsageError):
        L.student_inputs(d(base), d(slot), d(emb), d(written), ttl, now, smoothing=1.0)


def test_clip_smooth_jvp():
    import torch
    import paper_2512_09200_b200 as L
    lib = oracle.load_oracle()
    rng = np.random.default_rng(4)
    x = rng.normal(size=100_001) * 4
    y = (rng.random(100_001) < 0.3).astype(np.float64)
    got = L.clip_features(torch.from_numpy(x).cuda(), 2.5).cpu().numpy()
    assert np.array_equal(got, oracle.vec_op2(lib, "lo_clip_features", x, 2.5)[1])
    got = L.smooth_labels(torch.from_numpy(y).cuda(), 0.1).cpu().numpy()
    assert np.array_equal(got, oracle.vec_op2(lib, "lo_smooth_labels", y, 0.1)[1])
    with pytest.raises(L.UsageError):
        L.smooth_labels(torch.tensor([0.0, 0.5], dtype=torch.float64, device="cuda"), 0.1)
    with pytest.raises(L.UsageError):
        L.clip_features(torch.zeros(3, dtype=torch.float64, device="cuda"), 0.0)
    rows, width = 257, 300
    xs = rng.uniform(-10, 10, (rows, width))
    ts = rng.uniform(-1, 1, (rows, width))
    got = L.swish_rn_jvp(torch.from_numpy(xs).cuda(), torch.from_numpy(ts).cuda()).cpu().numpy()
    for r in (0, 100, 256):
        rc, want = oracle.swish_rn_jvp(xs[r], ts[r])
        assert rc == 0 and np.allclose(got[r], want, rtol=1e-13, atol=1e-13)
    bad = xs.copy()
    bad[3, 7] = np.nan
    with pytest.raises(L.DataError):
        L.swish_rn_jvp(torch.from_numpy(bad).cuda(), torch.from_numpy(ts).cuda())

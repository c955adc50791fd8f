"""C-ABI contract checks that need no GPU: every entry validates its arguments before touching
CUDA and reports a violation as LATTICE_USAGE (the reference's UsageError, core.hpp:20-22) with
a message naming the rule -- the same behaviour on a CPU-only host as on a B200."""
import ctypes

import pytest

import paper_2512_09200_b200 as L


def usage(rc, fragment):
    assert rc == L.USAGE, rc
    msg = L.lib.lattice_last_error().decode()
    assert fragment in msg, msg


def bag_args(**kw):
    a = L.BagArgs()
    a.features, a.batch, a.dim = 4, 8, 128
    a.table_dtype = a.out_dtype = L.BF16
    a.tables = a.rows = a.offsets = a.ids = a.out = ctypes.c_void_p(16)
    a.out_row_stride = 4 * 128
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_embedding_bag_contracts():
    usage(L.lib.lattice_embedding_bag(None, None), "null args")
    usage(L.lib.lattice_embedding_bag(ctypes.byref(bag_args(out_row_stride=3 * 128)), None),
          "out_row_stride too small")
    usage(L.lib.lattice_embedding_bag(ctypes.byref(bag_args(features=1 << 16, batch=1 << 15,
                                                            out_row_stride=(1 << 16) * 128)), None),
          "must be < 2^31")
    usage(L.lib.lattice_embedding_bag(ctypes.byref(bag_args(tables=None)), None), "null pointer")
    usage(L.lib.lattice_embedding_bag(ctypes.byref(bag_args(table_dtype=9)), None), "table dtype")


def net_config(**kw):
    kw = dict(kw)
    c = L.NetConfig()
    base = dict(n=8, d=64, blocks=2, nF=4, nL=4, k=4, n_mlp=2, domains=2, heads=2, tower_hidden=64,
                max_batch=512, dtype=L.BF16)
    mlp = kw.pop("mlp", None)
    base.update(kw)
    for k, v in base.items():
        setattr(c, k, v)
    mlp = mlp or [base["n"] * base["k"], 64, base["nF"] * base["d"]]
    for i, w in enumerate(mlp):
        c.mlp[i] = w
    return c


@pytest.mark.parametrize("kw,fragment", [
    (dict(nL=3), "nF + nL == n"),
    (dict(n=600, nF=300, nL=300), "n must be in [1, 512]"),
    (dict(k=65), "k must be in [1, 64]"),
    (dict(mlp=[31, 64, 256]), "mlp[0] must equal n*k"),
    (dict(mlp=[32, 20000, 256]), "hidden widths above 16384"),
    (dict(mlp=[32, 4096, 256], max_batch=128), "hidden widths above 2048 need bf16 and max_batch >= 256"),
    (dict(mlp=[32, 4096, 256], dtype=L.F32), "hidden widths above 2048 need bf16"),
    (dict(domains=33), "domains must be in [1, 32]"),
    (dict(heads=17), "heads must be in [1, 16]"),
    (dict(tower_hidden=12), "tower_hidden must be a multiple of 8"),
    (dict(d=96), "d must be 64 or 128"),
    (dict(dtype=L.F32, d=128), "fp32 needs d = 64"),
    (dict(dense_features=8), "dense_features must be in [0, n)"),
])
def test_network_config_contracts(kw, fragment):
    h = ctypes.c_void_p()
    usage(L.lib.lattice_net_create(ctypes.byref(net_config(**kw)), ctypes.byref(h)), fragment)
    assert not h.value


def test_bucket_rownorm_jsonl_contracts():
    p = ctypes.c_void_p(16)
    usage(L.lib.lattice_domain_bucket(10, 33, p, p, p, p, None), "domain_bucket: bad sizes")
    usage(L.lib.lattice_domain_bucket(-1, 2, p, p, p, p, None), "domain_bucket: bad sizes")
    usage(L.lib.lattice_rownorm(0, 4, 8, 0.0, p, p, 1, None), "eps must be > 0")
    usage(L.lib.lattice_rownorm(0, 4, 0, 1e-6, p, p, 1, None), "empty input")  # numerics.hpp:83
    info = L.JsonlInfo()
    h = ctypes.c_void_p()
    usage(L.lib.lattice_jsonl_open(p, 1 << 31, b"big.jsonl", ctypes.byref(h), ctypes.byref(info), None),
          "< 2 GiB")
    usage(L.lib.lattice_jsonl_open(p, 10, b"x", None, ctypes.byref(info), None), "null argument")
    usage(L.lib.lattice_jsonl_task_columns(-1, p, p, p, p, 1, p, p, p, p, None), "bad sizes")


def test_backward_contracts():
    p = ctypes.c_void_p(16)
    usage(L.lib.lattice_rownorm_vjp(3, 4, 8, 1e-6, L.F32, p, p, p, None), "mode must be 0, 1 or 2")
    usage(L.lib.lattice_rownorm_vjp(1, 4, 8, 1e-6, L.BF16, p, p, p, None), "dtype must be f32 or f64")
    usage(L.lib.lattice_routed_bce(4, 0, 3, p, p, p, p, p, None), "routed_bce: bad sizes")
    usage(L.lib.lattice_net_tower_backward(None, 4, p, p, p, None, L.F32, None), "null argument")
    usage(L.lib.lattice_net_mlp_backward(None, 4, p, p, None, None, None), "null argument")
    usage(L.lib.lattice_net_weight_sgd(None, 0, 3, 0, 0.1, p, p, None), "null argument")


def test_peer_reduce_sgd_contracts():
    p = ctypes.c_void_p(16)
    segs = (L.PeerSeg * 2)(L.PeerSeg(0, 8, 0, L.BF16, p), L.PeerSeg(4, 8, 0, L.F32, p))  # overlapping
    usage(L.lib.lattice_peer_reduce_sgd(None, p, segs, 2, 16, 0, 2, 0.1, None), "null argument")
    usage(L.lib.lattice_peer_reduce_sgd(p, p, segs, 0, 16, 0, 2, 0.1, None), "1..16 segments")
    usage(L.lib.lattice_peer_reduce_sgd(p, p, segs, 2, 16, 2, 2, 0.1, None), "bad rank/world")
    usage(L.lib.lattice_peer_reduce_sgd(p, p, segs, 2, 16, 0, 2, 0.1, None), "sorted, disjoint")
    bad = (L.PeerSeg * 1)(L.PeerSeg(0, 1, 1, L.BF16, p))  # a mean segment must be fp32
    usage(L.lib.lattice_peer_reduce_sgd(p, p, bad, 1, 16, 0, 2, 0.1, None), "dst dtype")

"""ctypes handles on the test-only checkers. TEST INFRASTRUCTURE ONLY.

`load_oracle()` -> oracle/_build/liboracle.so (the CPU restatement, lattice_oracle.c)
`load_ref()`    -> oracle/_ref/libref.so (the reference headers compiled in place, ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this
package. The product (paper_2512_09200_b200) never does.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int32
_SZ = ctypes.c_size_t
_D = ctypes.c_double


def ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class LoNetCfg(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("d", ctypes.c_int), ("blocks", ctypes.c_int),
                ("nF", ctypes.c_int), ("nL", ctypes.c_int), ("k", ctypes.c_int),
                ("n_mlp", ctypes.c_int), ("mlp", ctypes.c_int * 6), ("G", ctypes.c_int),
                ("heads", ctypes.c_int), ("tower_hidden", ctypes.c_int), ("hard", ctypes.c_int),
                ("bf16", ctypes.c_int)]


class LoNetWeights(ctypes.Structure):
    _fields_ = [("YT", _P), ("WL", _P), ("mlp", _P), ("T1", _P), ("T2", _P)]


_oracle = None
_ref = None


def load_oracle():
    global _oracle
    if _oracle is None:
        lib = ctypes.CDLL(os.path.join(_HERE, "_build", "liboracle.so"))
        lib.lo_xxh64.restype = _U64
        lib.lo_xxh64.argtypes = [_P, _SZ, _U64]
        lib.lo_gen.restype = _U64
        lib.lo_gen.argtypes = [_U64, _U64, _U64]
        lib.lo_signature.restype = _SZ
        lib.lo_signature.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p,
                                     ctypes.c_uint32, _I64, _P]
        lib.lo_assign_window.restype = ctypes.c_int
        lib.lo_assign_window.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p,
                                         ctypes.c_uint32, _I64, _U64, _P, ctypes.c_int]
        lib.lo_zip_columns.restype = _I64
        lib.lo_zip_columns.argtypes = [_I64, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P,
                                       ctypes.c_int, _P, _P, _U64, _P, _P, _P]
        for name in ("lo_rms_norm", "lo_swish_rn", "lo_swish_rn_hard"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [_P, _SZ, _D, _P]
        lib.lo_table_value.restype = ctypes.c_float
        lib.lo_table_value.argtypes = [_U64, _I64, _I64, ctypes.c_int, _I64, _I64]
        lib.lo_weight_value.restype = ctypes.c_float
        lib.lo_weight_value.argtypes = [_U64, _U64, _I64, _I64, _I64]
        lib.lo_weight_tag.restype = _U64
        lib.lo_weight_tag.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.lo_weight_shift.restype = ctypes.c_int
        lib.lo_weight_shift.argtypes = [_I64]
        lib.lo_embedding_bag_synth.restype = _I64
        lib.lo_embedding_bag_synth.argtypes = [_U64, ctypes.c_int, _I64, ctypes.c_int, _I64,
                                               _P, _P, _I64, _I64, _P, ctypes.c_int]
        lib.lo_embedding_bag.restype = _I64
        lib.lo_embedding_bag.argtypes = [ctypes.c_int, _P, ctypes.c_int, _I64, _P, _P, _P, _P]
        lib.lo_net_forward.restype = None
        lib.lo_net_forward.argtypes = [ctypes.POINTER(LoNetCfg), ctypes.POINTER(LoNetWeights),
                                       _I64, _P, _P, _P, ctypes.c_int]
        lib.lo_synth_bags.restype = None
        lib.lo_synth_bags.argtypes = [ctypes.c_int, _I64, ctypes.c_int, _I64, _U64, _P, _P]
        lib.lo_synth_domains.restype = None
        lib.lo_synth_domains.argtypes = [_I64, ctypes.c_int, _U64, _P]
        lib.lo_fill_weights.restype = None
        lib.lo_fill_weights.argtypes = [_P, _I64, _I64, _U64, _U64]
        lib.lo_synth_impressions.restype = None
        lib.lo_synth_impressions.argtypes = [_I64, ctypes.c_int, _U64, _P, _P, _P, _P, _P, _P, _P]
        lib.lo_bf16_round.restype = ctypes.c_float
        lib.lo_bf16_round.argtypes = [ctypes.c_float]
        lib.lo_correlation_loss.restype = ctypes.c_int
        lib.lo_correlation_loss.argtypes = [_P, _P, _SZ, _D, _P]
        lib.lo_window_summary.restype = ctypes.c_int
        lib.lo_window_summary.argtypes = [_I64, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P]
        lib.lo_merge_dense.restype = _I64
        lib.lo_merge_dense.argtypes = [_I64, ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P]
        lib.lo_dense_processor.restype = None
        lib.lo_dense_processor.argtypes = [ctypes.POINTER(LoNetCfg), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           _P, _P, _I64, _P, _P, ctypes.c_int]
        for name in ("lo_clip_features", "lo_smooth_labels"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [_P, _SZ, _D, _P]
        lib.lo_swish_rn_jvp.restype = ctypes.c_int
        lib.lo_swish_rn_jvp.argtypes = [_P, _P, _SZ, _D, _P]
        lib.lo_student_inputs.restype = None
        lib.lo_student_inputs.argtypes = [_I64, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _I64, _I64, _D, _D,
                                          ctypes.c_int, _P, _P, _P]
        lib.lo_routed_objectives.restype = ctypes.c_int
        lib.lo_routed_objectives.argtypes = [_I64, ctypes.c_int, ctypes.c_int, _P, _P, _P, _D, _P, _P, _P, _P]
        _oracle = lib
    return _oracle


def ref_available():
    return os.path.exists(os.path.join(_HERE, "_ref", "libref.so"))


def load_ref():
    global _ref
    if _ref is None:
        lib = ctypes.CDLL(os.path.join(_HERE, "_ref", "libref.so"))
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_stable_hash.restype = _U64
        lib.ref_stable_hash.argtypes = [_P, _SZ, _U64]
        lib.ref_signature.restype = _SZ
        lib.ref_signature.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p,
                                      ctypes.c_uint32, _I64, _P]
        lib.ref_zipper_config_check.restype = ctypes.c_int
        lib.ref_zipper_config_check.argtypes = [ctypes.c_int, _P, _P, _U64]
        lib.ref_assign_window.restype = ctypes.c_int
        lib.ref_assign_window.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p,
                                          ctypes.c_uint32, _I64, ctypes.c_int, _P, _P, _U64,
                                          ctypes.POINTER(_I64)]
        lib.ref_zip_dataset.restype = ctypes.c_int
        lib.ref_zip_dataset.argtypes = [_I64, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P,
                                        ctypes.c_int, _P, _P, _U64, _P, _P]
        for name in ("ref_rms_norm", "ref_swish_rn", "ref_swish_rn_hard"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [_P, _SZ, _D, _P]
        lib.ref_correlation_loss.restype = ctypes.c_int
        lib.ref_correlation_loss.argtypes = [_P, _P, _SZ, _D, _P]
        lib.ref_merge_domains.restype = ctypes.c_int
        lib.ref_merge_domains.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P]
        for name in ("ref_clip_features", "ref_smooth_labels"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [_P, _SZ, _D, _P]
        lib.ref_swish_rn_jvp.restype = ctypes.c_int
        lib.ref_swish_rn_jvp.argtypes = [_P, _P, _SZ, _D, _P]
        lib.ref_student_queries.restype = ctypes.c_int
        lib.ref_student_queries.argtypes = [_I64, ctypes.c_int, _P, _P, _P, _I64, _D, _I64, ctypes.c_int, _P, _P,
                                            _I64, _D, _P, _P, _P]
        lib.ref_window_summary.restype = ctypes.c_int
        lib.ref_window_summary.argtypes = [_I64, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P]
        if hasattr(lib, "ref_parse_jsonl"):
            lib.ref_parse_jsonl.restype = ctypes.c_int
            lib.ref_parse_jsonl.argtypes = [ctypes.c_char_p, _SZ, ctypes.c_char_p, ctypes.POINTER(_P),
                                            ctypes.POINTER(_SZ)]
            lib.ref_free.restype = None
            lib.ref_free.argtypes = [_P]
        _ref = lib
    return _ref


def ref_parse_jsonl(content, source="records"):
    """The reference's parse_jsonl_records (serde.hpp:158-170, via ref_shim) -> (records, None) or
    (None, error text); the text of an exception that is not a DataError (nlohmann's
    out_of_range.406 for a number literal overflowing double) is prefixed "exception: ". Records: dicts with domain / user_id / ad_id / impression_time_ms /
    features {key: float} / conversions {key: int}."""
    import json
    import struct
    lib = load_ref()
    out, n = _P(), _SZ()
    rc = lib.ref_parse_jsonl(content, len(content), source.encode(), ctypes.byref(out), ctypes.byref(n))
    if rc != 0:
        return None, ("exception: " if rc == 3 else "") + lib.ref_last_error().decode("utf-8", "replace")
    try:
        text = ctypes.string_at(out.value, n.value).decode("utf-8")
    finally:
        lib.ref_free(out)
    recs = json.loads(text)
    for r in recs:
        r["features"] = {k: struct.unpack("<d", bytes.fromhex(v)[::-1])[0] for k, v in r["features"].items()}
    return recs, None


# ---- thin numpy conveniences ---------------------------------------------------------

def xxh64(data: bytes, seed: int) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    return load_oracle().lo_xxh64(ptr(buf), len(data), seed)


def pack_strings(strs):
    """list[bytes] -> (uint8 bytes, int64 offsets[n+1])"""
    offs = np.zeros(len(strs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(s) for s in strs])
    data = np.frombuffer(b"".join(strs), dtype=np.uint8).copy() if offs[-1] else np.zeros(1, np.uint8)
    return data, offs


def zip_columns(users, ads, ts, conv, conv_present, durations, probs, seed, lib=None):
    """Oracle columnar zip. Returns (window u8[n], labels u8[n,T,W], err_record, err_task)."""
    lib = lib or load_oracle()
    n = len(users)
    T = conv.shape[1] if conv.ndim == 2 else 0
    W = len(durations)
    ub, uo = pack_strings(users)
    ab, ao = pack_strings(ads)
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    conv = np.ascontiguousarray(conv, dtype=np.int64).reshape(n, T)
    pres = np.ascontiguousarray(conv_present, dtype=np.uint8).reshape(n, T)
    dur = np.ascontiguousarray(durations, dtype=np.int64)
    pr = np.ascontiguousarray(probs, dtype=np.float64)
    win = np.zeros(max(n, 1), np.uint8)
    lab = np.zeros(max(n * T * W, 1), np.uint8)
    et = ctypes.c_int32(-1)
    err = lib.lo_zip_columns(n, ptr(ub), ptr(uo), ptr(ab), ptr(ao), ptr(ts), T, ptr(conv),
                             ptr(pres), W, ptr(dur), ptr(pr), seed, ptr(win), ptr(lab),
                             ctypes.byref(et))
    return win[:n], lab[: n * T * W].reshape(n, T, W), int(err), int(et.value)


def ref_zip_dataset(users, ads, ts, conv, conv_present, durations, probs, seed):
    """Reference zip_dataset over columns: (rc, window, labels, message)."""
    lib = load_ref()
    n = len(users)
    T = conv.shape[1]
    W = len(durations)
    ub, uo = pack_strings(users)
    ab, ao = pack_strings(ads)
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    conv = np.ascontiguousarray(conv, dtype=np.int64)
    pres = np.ascontiguousarray(conv_present, dtype=np.uint8)
    dur = np.ascontiguousarray(durations, dtype=np.int64)
    pr = np.ascontiguousarray(probs, dtype=np.float64)
    win = np.zeros(max(n, 1), np.uint8)
    lab = np.zeros(max(n * T * W, 1), np.uint8)
    rc = lib.ref_zip_dataset(n, ptr(ub), ptr(uo), ptr(ab), ptr(ao), ptr(ts), T, ptr(conv),
                             ptr(pres), W, ptr(dur), ptr(pr), seed, ptr(win), ptr(lab))
    msg = lib.ref_last_error().decode() if rc else ""
    return rc, win[:n], lab[: n * T * W].reshape(n, T, W), msg


def vec_op(lib, name, x, eps=1e-6):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(max(len(x), 1), np.float64)
    rc = getattr(lib, name)(ptr(x) if len(x) else None, len(x), eps, ptr(out))
    return rc, out[: len(x)]


def correlation_loss(x, y, eps=1e-6, lib=None):
    """-> (rc, loss): lo_correlation_loss (or ref_correlation_loss with lib=load_ref())."""
    lib = lib or load_oracle()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(1, np.float64)
    name = "ref_correlation_loss" if hasattr(lib, "ref_correlation_loss") else "lo_correlation_loss"
    rc = getattr(lib, name)(ptr(x) if len(x) else None, ptr(y) if len(y) else None, len(x), eps, ptr(out))
    return rc, float(out[0])


def window_summary(window, labels, W):
    """lo_window_summary: (rc, counts [W], positives [W, T])."""
    window = np.ascontiguousarray(window, dtype=np.uint8)
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    n, T = len(window), labels.shape[1]
    counts = np.zeros(W, np.int64)
    pos = np.zeros((W, T), np.int64)
    rc = load_oracle().lo_window_summary(n, T, W, ptr(window), ptr(labels), ptr(counts), ptr(pos))
    return rc, counts, pos


def ref_window_summary(window, labels, W):
    """The reference's window_routing_summary: (rc, counts [W], rates [W, T])."""
    window = np.ascontiguousarray(window, dtype=np.uint8)
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    n, T = len(window), labels.shape[1]
    dur = np.arange(1, W + 1, dtype=np.int64) * 1000
    pr = np.full(W, 1.0 / W)
    pr[-1] = 1.0 - pr[:-1].sum()
    counts = np.zeros(W, np.int64)
    rates = np.zeros((W, T), np.float64)
    rc = load_ref().ref_window_summary(n, T, W, ptr(window), ptr(labels), ptr(dur), ptr(pr), ptr(counts),
                                       ptr(rates))
    return rc, counts, rates


def routed_objectives(logits, window, labels, eps=1e-6):
    """lo_routed_objectives: (rc, routed [n, T], corr [T], counts [W], positives [W, T])."""
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    window = np.ascontiguousarray(window, dtype=np.uint8)
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    n, T, W = labels.shape
    routed = np.zeros((n, T), np.float32)
    corr = np.zeros(T, np.float64)
    counts = np.zeros(W, np.int64)
    pos = np.zeros((W, T), np.int64)
    rc = load_oracle().lo_routed_objectives(n, T, W, ptr(logits), ptr(window), ptr(labels), eps, ptr(routed),
                                            ptr(corr), ptr(counts), ptr(pos))
    return rc, routed, corr, counts, pos


def merge_dense(domain, values, src_col, bf16=False):
    """lo_merge_dense: (first bad record or -1, out [n, width] fp32)."""
    domain = np.ascontiguousarray(domain, dtype=np.int32)
    values = np.ascontiguousarray(values, dtype=np.float32)
    src_col = np.ascontiguousarray(src_col, dtype=np.int32)
    n, md = values.shape
    G, width = src_col.shape
    out = np.zeros((n, width), np.float32)
    bad = load_oracle().lo_merge_dense(n, G, md, ptr(domain), ptr(values), ptr(src_col), width, int(bf16), ptr(out))
    return bad, out


def ref_merge_domains(decl, n_rec, values):
    """The reference's merge_domains on integer-named features: decl int32 [G, max_decl] (-1 =
    unused), n_rec records per domain (grouped in order), values fp64 [n, max_decl]. Returns
    (rc, union feature ids, matrix [n, n_union])."""
    decl = np.ascontiguousarray(decl, dtype=np.int32)
    n_rec = np.ascontiguousarray(n_rec, dtype=np.int64)
    values = np.ascontiguousarray(values, dtype=np.float64)
    G, md = decl.shape
    n = int(n_rec.sum())
    uid = np.zeros(G * md + 1, np.int32)
    nu = ctypes.c_int32()
    out = np.zeros(max(n * G * md, 1), np.float64)
    rc = load_ref().ref_merge_domains(G, md, ptr(decl), ptr(n_rec), ptr(values), ptr(uid), ctypes.byref(nu),
                                      ptr(out))
    k = nu.value
    return rc, uid[:k], out[: n * k].reshape(n, k)


def dense_processor(cfg, n_dense, dense_in, dense_hidden, D1, D2, dense, pooled, threads=0):
    """lo_dense_processor: fills rows [n - n_dense, n) of pooled [count, n, d] in place."""
    D1 = np.ascontiguousarray(D1, dtype=np.float32)
    D2 = np.ascontiguousarray(D2, dtype=np.float32)
    dense = np.ascontiguousarray(dense, dtype=np.float32)
    assert pooled.flags.c_contiguous and pooled.dtype == np.float32
    load_oracle().lo_dense_processor(ctypes.byref(cfg), n_dense, dense_in, dense_hidden, ptr(D1), ptr(D2),
                                     dense.shape[0], ptr(dense), ptr(pooled), threads)
    return pooled


def vec_op2(lib, name, x, arg):
    """(rc, out) of an element op (x, n, scalar, out): clip_features / smooth_labels."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(max(len(x), 1), np.float64)
    rc = getattr(lib, name)(ptr(x) if len(x) else None, len(x), arg, ptr(out))
    return rc, out[: len(x)]


def swish_rn_jvp(x, t, eps=1e-6, lib=None):
    lib = lib or load_oracle()
    x = np.ascontiguousarray(x, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    out = np.zeros(max(len(x), 1), np.float64)
    name = "ref_swish_rn_jvp" if hasattr(lib, "ref_swish_rn_jvp") else "lo_swish_rn_jvp"
    rc = getattr(lib, name)(ptr(x) if len(x) else None, ptr(t) if len(t) else None, len(x), eps, ptr(out))
    return rc, out[: len(x)]


def student_inputs(base, slot, store_emb, store_logit, written_at, ttl, now, clip=0.0, smoothing=-1.0, bf16=False):
    """lo_student_inputs: (rows [n, base_dim+dim], logit [n], hit [n])."""
    base = np.ascontiguousarray(base, dtype=np.float32)
    slot = np.ascontiguousarray(slot, dtype=np.int64)
    store_emb = np.ascontiguousarray(store_emb, dtype=np.float32)
    store_logit = np.ascontiguousarray(store_logit, dtype=np.float32)
    written_at = np.ascontiguousarray(written_at, dtype=np.int64)
    n, bd = base.shape
    dim = store_emb.shape[1]
    out = np.zeros((n, bd + dim), np.float32)
    logit = np.zeros(n, np.float32)
    hit = np.zeros(n, np.uint8)
    load_oracle().lo_student_inputs(n, bd, dim, ptr(base), ptr(slot), ptr(store_emb), ptr(store_logit),
                                    ptr(written_at), ttl, now, clip, smoothing, int(bf16), ptr(out), ptr(logit),
                                    ptr(hit))
    return out, logit, hit


def ref_student_queries(base, slot, store_emb, store_logit, written_at, ttl, now, clip=0.0, smoothing=-1.0):
    """The reference's TeacherEmbeddingStore + student_feature_vector (+ clip_features):
    (rc, rows fp64, logits fp64 (NaN on miss), hit)."""
    base = np.ascontiguousarray(base, dtype=np.float64)
    slot = np.ascontiguousarray(slot, dtype=np.int64)
    emb = np.ascontiguousarray(store_emb, dtype=np.float64)
    lg = np.ascontiguousarray(store_logit, dtype=np.float64)
    wa = np.ascontiguousarray(written_at, dtype=np.int64)
    n, bd = base.shape
    E, dim = emb.shape
    rows = np.zeros((n, bd + dim), np.float64)
    logits = np.zeros(n, np.float64)
    hit = np.zeros(n, np.uint8)
    rc = load_ref().ref_student_queries(E, dim, ptr(emb), ptr(lg), ptr(wa), ttl, smoothing, n, bd, ptr(base),
                                        ptr(slot), now, clip, ptr(rows), ptr(logits), ptr(hit))
    return rc, rows, logits, hit


def net_forward(cfg, w, pooled, dom, bf16=True, hard=False, threads=0):
    """lo_net_forward for a Network config dict and its weights() (host fp32 arrays):
    pooled [count, n, d] raw sums, dom [count] -> logits [count, heads]."""
    c = LoNetCfg()
    c.n, c.d, c.blocks, c.nF, c.nL, c.k = cfg["n"], cfg["d"], cfg["blocks"], cfg["nF"], cfg["nL"], cfg["k"]
    c.n_mlp = len(cfg["mlp"]) - 1
    for i, v in enumerate(cfg["mlp"]):
        c.mlp[i] = v
    c.G, c.heads, c.tower_hidden, c.hard, c.bf16 = cfg["domains"], cfg["heads"], cfg["tower_hidden"], int(hard), int(bf16)
    keep = [np.ascontiguousarray(a, dtype=np.float32) for a in w["YT"] + w["WL"] + w["mlp"]]
    nb = cfg["blocks"]
    yt = (_P * nb)(*[a.ctypes.data for a in keep[:nb]])
    wl = (_P * nb)(*[a.ctypes.data for a in keep[nb:2 * nb]])
    ml = (_P * len(w["mlp"]))(*[a.ctypes.data for a in keep[2 * nb:]])
    T1 = np.ascontiguousarray(w["T1"], dtype=np.float32)
    T2 = np.ascontiguousarray(w["T2"], dtype=np.float32)
    ws = LoNetWeights(ctypes.cast(yt, _P), ctypes.cast(wl, _P), ctypes.cast(ml, _P), _P(T1.ctypes.data),
                      _P(T2.ctypes.data))
    pooled = np.ascontiguousarray(pooled, dtype=np.float32)
    d = np.ascontiguousarray(dom, dtype=np.int32)
    out = np.zeros((len(d), cfg["heads"]), np.float32)
    load_oracle().lo_net_forward(ctypes.byref(c), ctypes.byref(ws), len(d), ptr(pooled), ptr(d), ptr(out), threads)
    return out


def synth_bags(F, B, max_len, rows, seed):
    lib = load_oracle()
    offsets = np.zeros(F * B + 1, np.int64)
    ids = np.zeros(max(F * B * max_len, 1), np.int32)
    lib.lo_synth_bags(F, B, max_len, rows, seed, ptr(offsets), ptr(ids))
    return offsets, ids[: offsets[-1]]


def synth_domains(B, G, seed):
    dom = np.zeros(B, np.int32)
    load_oracle().lo_synth_domains(B, G, seed, ptr(dom))
    return dom


def embedding_bag_synth(seed, F, rows, D, B, offsets, ids, b_lo=0, b_hi=None, threads=0):
    """Exact fp32 pooled sums of samples [b_lo, b_hi) over the synthetic tables."""
    b_hi = B if b_hi is None else b_hi
    out = np.zeros((b_hi - b_lo, F, D), np.float32)
    bad = load_oracle().lo_embedding_bag_synth(seed, F, rows, D, B, ptr(offsets), ptr(ids), b_lo,
                                               b_hi, ptr(out), threads)
    return out, int(bad)


def bf16_round(x):
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (vectorised)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def synth_impressions(n, T, seed):
    """Host copy of lattice_synth_impressions: (users list[bytes], ads list[bytes], ts, conv, present)."""
    ub = np.zeros(9 * n, np.uint8)
    ab = np.zeros(7 * n, np.uint8)
    uo = np.zeros(n + 1, np.int64)
    ao = np.zeros(n + 1, np.int64)
    ts = np.zeros(n, np.int64)
    conv = np.zeros((n, T), np.int64)
    pres = np.zeros((n, T), np.uint8)
    load_oracle().lo_synth_impressions(n, T, seed, ptr(ub), ptr(uo), ptr(ab), ptr(ao), ptr(ts),
                                       ptr(conv), ptr(pres))
    users = [ub[9 * i: 9 * i + 9].tobytes() for i in range(n)]
    ads = [ab[7 * i: 7 * i + 7].tobytes() for i in range(n)]
    return users, ads, ts, conv, pres

"""Host-side (Python) mirror of the Lattice hot-path interface over liblattice_b200.so.

The product is the C ABI in include/lattice_b200.h (sm_100a CUDA kernels); this module is a
thin ctypes binding used by the tests and bench.py. torch is used only as the device-memory
and stream plumbing: every array argument is a CUDA tensor whose data_ptr() is handed to the
library. There is no CPU fallback -- if the shared library is missing, importing this module
raises.

Errors map to the reference's exception types (proj/include/lattice/core.hpp:20-27):
LATTICE_USAGE -> UsageError(ValueError), LATTICE_DATA -> DataError(RuntimeError).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LATTICE_LIB: load another build of the library (A/B runs of two builds on one box)
LIB_PATH = os.environ.get("LATTICE_LIB") or os.path.join(_HERE, "liblattice_b200.so")

OK, USAGE, DATA, CUDA, NCCL = 0, 1, 2, 3, 4
F32, BF16, F64 = 0, 1, 2


class LatticeError(Exception):
    pass


class UsageError(LatticeError, ValueError):
    """core.hpp:20 -- caller broke an API contract."""


class DataError(LatticeError, RuntimeError):
    """core.hpp:25 -- input data is malformed."""

    def __init__(self, msg, index=-1):
        super().__init__(msg)
        self.index = index


class CudaError(LatticeError, RuntimeError):
    pass


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64


class ZipArgs(ctypes.Structure):
    _fields_ = [("n", _I64), ("user_bytes", _P), ("user_off", _P), ("ad_bytes", _P),
                ("ad_off", _P), ("ts", _P), ("tasks", _I32), ("conv", _P),
                ("conv_present", _P), ("windows", _I32), ("durations_host", _P),
                ("probabilities_host", _P), ("seed", _U64), ("window", _P), ("labels", _P),
                ("routed", _P), ("check", _I32)]


class BagArgs(ctypes.Structure):
    _fields_ = [("features", _I32), ("batch", _I64), ("dim", _I32), ("table_dtype", _I32),
                ("tables", _P), ("rows", _P), ("offsets", _P), ("ids", _P), ("out_dtype", _I32),
                ("out", _P), ("out_row_stride", _I64), ("out_feature_offset", _I32),
                ("sample_pos", _P), ("normalize", _I32), ("check", _I32), ("sources", _I32),
                ("slice_cap", _I64)]


class PeerSeg(ctypes.Structure):
    _fields_ = [("offset", _I64), ("count", _I64), ("mode", _I32), ("dst_dtype", _I32), ("dst", _P)]


class PeerBagArgs(ctypes.Structure):
    _fields_ = [("rank", _I32), ("world", _I32), ("features_local", _I32), ("feature_base", _I32),
                ("batch", _I64), ("dim", _I32), ("table_dtype", _I32), ("tables", _P), ("rows", _P),
                ("offsets", _P), ("ids", _P), ("sample_pos", _P), ("out", _P), ("out_dtype", _I32),
                ("out_row_stride", _I64), ("normalize", _I32), ("check", _I32)]


class JsonlInfo(ctypes.Structure):
    _fields_ = [(k, _I64) for k in ("lines", "records", "domain_bytes", "user_bytes", "ad_bytes",
                                    "feature_entries", "feature_key_bytes", "conversion_entries",
                                    "conversion_key_bytes", "error_line", "error_kind")]


class JsonlColumns(ctypes.Structure):
    _fields_ = [(k, _P) for k in ("domain", "domain_off", "user", "user_off", "ad", "ad_off", "ts", "line",
                                  "feature_off", "feature_key", "feature_key_off", "feature_val",
                                  "conversion_off", "conversion_key", "conversion_key_off",
                                  "conversion_val")]


class ObjectiveArgs(ctypes.Structure):
    _fields_ = [("n", _I64), ("tasks", _I32), ("windows", _I32), ("logits", _P), ("window", _P),
                ("labels", _P), ("eps", ctypes.c_double), ("routed", _P), ("corr", _P), ("counts", _P),
                ("positives", _P), ("check", _I32)]


class StudentArgs(ctypes.Structure):
    _fields_ = [("n", _I64), ("base_dim", _I32), ("dim", _I32), ("base", _P), ("slot", _P), ("store_emb", _P),
                ("store_logit", _P), ("written_at", _P), ("ttl_ms", _I64), ("now", _I64), ("clip", ctypes.c_double),
                ("smoothing", ctypes.c_double), ("out_dtype", _I32), ("out", _P), ("teacher_logit", _P),
                ("hit", _P)]


class GemmArgs(ctypes.Structure):
    _fields_ = [("M", _I64), ("N", _I64), ("K", _I64), ("A", _P), ("lda", _I64), ("B", _P),
                ("ldb", _I64), ("C", _P), ("ldc", _I64), ("out_dtype", _I32), ("epilogue", _I32),
                ("resid", _P), ("ldr", _I64), ("group", _I32), ("in_dtype", _I32), ("a_major", _I32),
                ("b_major", _I32)]


class FmLcbArgs(ctypes.Structure):
    _fields_ = [("batch", _I64), ("n", _I32), ("d", _I32), ("k", _I32), ("nF", _I32), ("nL", _I32),
                ("dtype", _I32), ("X", _P), ("YT", _P), ("WL", _P), ("Fin", _P), ("Xout", _P)]


class NetConfig(ctypes.Structure):
    _fields_ = [("n", _I32), ("d", _I32), ("blocks", _I32), ("nF", _I32), ("nL", _I32),
                ("k", _I32), ("n_mlp", _I32), ("mlp", _I32 * 6), ("domains", _I32),
                ("heads", _I32), ("tower_hidden", _I32), ("hard", _I32), ("max_batch", _I64),
                ("weight_seed", _U64), ("dtype", _I32), ("dense_features", _I32), ("dense_in", _I32),
                ("dense_hidden", _I32)]


class Batch(ctypes.Structure):
    _fields_ = [("batch", _I64), ("domain", _P), ("table_dtype", _I32), ("tables", _P),
                ("rows", _P), ("offsets", _P), ("ids", _P), ("pooled", _P),
                ("pooled_layout", _I32), ("shards", _I32), ("dense", _P), ("check", _I32)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("lattice_last_error", ctypes.c_char_p, [])
_sig("lattice_last_error_index", _I64, [])
_sig("lattice_abi_version", ctypes.c_int, [])
_sig("lattice_stable_hash", ctypes.c_int, [_I64, _P, _P, _U64, _P, _P])
_sig("lattice_zipper_validate", ctypes.c_int, [_I32, _P, _P])
_sig("lattice_zipper_assign_labels", ctypes.c_int, [ctypes.POINTER(ZipArgs), _P])
_sig("lattice_embedding_bag", ctypes.c_int, [ctypes.POINTER(BagArgs), _P])
_sig("lattice_rownorm", ctypes.c_int, [_I32, _I64, _I64, ctypes.c_double, _P, _P, _I32, _P])
_sig("lattice_rownorm_f64", ctypes.c_int, [_I32, _I64, _I64, ctypes.c_double, _P, _P, _I32, _P])
_sig("lattice_fill_tables", ctypes.c_int, [_P, _I32, _I32, _I64, _I32, _U64, _I32, _I64, _P])
_sig("lattice_fill_weights", ctypes.c_int, [_P, _I32, _I64, _I64, _U64, _U64, _P])
_sig("lattice_synth_bags", ctypes.c_int, [_I32, _I64, _I32, _I64, _U64, _P, _P, _P])
_sig("lattice_synth_domains", ctypes.c_int, [_I64, _I32, _U64, _P, _P])
_sig("lattice_domain_bucket", ctypes.c_int, [_I64, _I32, _P, _P, _P, _P, _P])
_sig("lattice_lengths_to_offsets", ctypes.c_int, [_I64, _P, _P, _P])
_sig("lattice_pack_slices", ctypes.c_int, [_I32, _P, _P, _I64, _P, _P, _P])
_sig("lattice_synth_impressions", ctypes.c_int, [_I64, _I32, _U64, _P, _P, _P, _P, _P, _P, _P, _P])
_sig("lattice_route_heads", ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _P])
_sig("lattice_peer_embedding_bag", ctypes.c_int, [ctypes.POINTER(PeerBagArgs), _P])
_sig("lattice_ipc_handle", ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)])
_sig("lattice_ipc_open", ctypes.c_int, [_P, _I64, ctypes.POINTER(_P)])
_sig("lattice_ipc_close", ctypes.c_int, [_P])
_sig("lattice_peer_barrier", ctypes.c_int, [_P, _I32, _I32, ctypes.c_double, _P, _P])
_sig("lattice_peer_reduce_sgd", ctypes.c_int, [_P, _P, _P, _I32, _I64, _I32, _I32, ctypes.c_float, _P])
_sig("lattice_net_bucket", ctypes.c_int, [_P, _I64, _P, _P])
_sig("lattice_net_buffer", _P, [_P, _I32])
_sig("lattice_correlation_loss", ctypes.c_int, [_I64, _I32, _P, _I64, _P, _I64, ctypes.c_double, _P, _I32, _P])
_sig("lattice_window_summary", ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _P, _I32, _P])
_sig("lattice_routed_objectives", ctypes.c_int, [ctypes.POINTER(ObjectiveArgs), _P])
_sig("lattice_merge_dense", ctypes.c_int, [_I64, _I32, _I32, _P, _P, _I32, _P, _I32, _I32, _P, _I32, _P])
_sig("lattice_student_inputs", ctypes.c_int, [ctypes.POINTER(StudentArgs), _P])
_sig("lattice_clip_features", ctypes.c_int, [_I64, _P, ctypes.c_double, _P, _P])
_sig("lattice_smooth_labels", ctypes.c_int, [_I64, _P, ctypes.c_double, _P, _I32, _P])
_sig("lattice_swish_rn_jvp", ctypes.c_int, [_I64, _I64, ctypes.c_double, _P, _P, _P, _I32, _P])
_sig("lattice_gemm", ctypes.c_int, [ctypes.POINTER(GemmArgs), _P])
_sig("lattice_device_check", ctypes.c_int, [_P])
_sig("lattice_rownorm_vjp", ctypes.c_int, [_I32, _I64, _I64, ctypes.c_double, _I32, _P, _P, _P, _P])
_sig("lattice_routed_bce", ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _P, _P, _P])
_sig("lattice_net_tower_backward", ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _I32, _P])
_sig("lattice_net_tower_sgd", ctypes.c_int, [_P, ctypes.c_float, _P, _P, _P, _P, _P])
_sig("lattice_net_mlp_backward", ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P])
_sig("lattice_net_weight_sgd", ctypes.c_int, [_P, _I32, _I32, _I32, ctypes.c_float, _P, _P, _P])
_sig("lattice_net_create", ctypes.c_int, [ctypes.POINTER(NetConfig), ctypes.POINTER(_P)])
_sig("lattice_net_destroy", None, [_P])
_sig("lattice_net_weight", _P, [_P, _I32, _I32, _I32])
_sig("lattice_net_set_weight", ctypes.c_int, [_P, _I32, _I32, _I32, _P, _I32, _P])
_sig("lattice_fm_lcb", ctypes.c_int, [ctypes.POINTER(FmLcbArgs), _P])
_sig("lattice_net_forward", ctypes.c_int, [_P, ctypes.POINTER(Batch), _P, _P])
_sig("lattice_net_set_timing", ctypes.c_int, [_P, _I32])
_sig("lattice_net_stage_times", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_float), _I32,
                                               ctypes.POINTER(_I32)])

_sig("lattice_jsonl_open", ctypes.c_int, [_P, _I64, ctypes.c_char_p, ctypes.POINTER(_P),
                                          ctypes.POINTER(JsonlInfo), _P])
_sig("lattice_jsonl_extract", ctypes.c_int, [_P, ctypes.POINTER(JsonlColumns), _P])
_sig("lattice_jsonl_task_columns", ctypes.c_int, [_I64, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P])
_sig("lattice_jsonl_close", None, [_P])

EXPORTS = ["lattice_last_error", "lattice_last_error_index", "lattice_abi_version",
           "lattice_stable_hash", "lattice_zipper_validate", "lattice_zipper_assign_labels",
           "lattice_embedding_bag", "lattice_rownorm", "lattice_fill_tables",
           "lattice_fill_weights", "lattice_synth_bags", "lattice_synth_domains",
           "lattice_domain_bucket", "lattice_lengths_to_offsets", "lattice_pack_slices",
           "lattice_synth_impressions", "lattice_route_heads", "lattice_gemm",
           "lattice_net_create", "lattice_net_destroy",
           "lattice_net_weight", "lattice_net_forward", "lattice_net_set_timing",
           "lattice_net_stage_times", "lattice_peer_embedding_bag", "lattice_ipc_handle",
           "lattice_ipc_open", "lattice_ipc_close", "lattice_peer_barrier", "lattice_net_bucket",
           "lattice_net_buffer", "lattice_correlation_loss", "lattice_window_summary",
           "lattice_routed_objectives", "lattice_merge_dense", "lattice_student_inputs",
           "lattice_clip_features", "lattice_smooth_labels", "lattice_swish_rn_jvp",
           "lattice_jsonl_open", "lattice_jsonl_extract", "lattice_jsonl_task_columns",
           "lattice_jsonl_close", "lattice_net_set_weight", "lattice_fm_lcb",
           "lattice_rownorm_f64", "lattice_device_check", "lattice_rownorm_vjp", "lattice_routed_bce",
           "lattice_net_tower_backward", "lattice_net_tower_sgd", "lattice_net_mlp_backward",
           "lattice_net_weight_sgd", "lattice_peer_reduce_sgd"]

lib = _lib


def check(rc):
    if rc == OK:
        return
    msg = _lib.lattice_last_error().decode()
    if rc == USAGE:
        raise UsageError(msg)
    if rc == DATA:
        raise DataError(msg, int(_lib.lattice_last_error_index()))
    raise CudaError(msg)


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


# ---- Zipper ---------------------------------------------------------------------------------

def zipper_assign_labels(user_bytes, user_off, ad_bytes, ad_off, ts, conv, conv_present,
                         durations, probabilities, seed, routed=False, check_errors=True,
                         stream=None):
    """Columnar lattice::zip_dataset core (datasets.hpp:199-249) on the GPU.

    Device tensors: user_bytes/ad_bytes uint8, *_off int64 [n+1], ts int64 [n],
    conv int64 [n,T], conv_present uint8 [n,T]. durations/probabilities are host sequences.
    Returns (window uint8 [n], labels uint8 [n,T,W], routed uint8 [n,T] or None)."""
    import numpy as np
    import torch
    n = ts.shape[0]
    T = conv.shape[1] if conv.dim() == 2 else 0
    W = len(durations)
    dur = np.ascontiguousarray(durations, dtype=np.int64)
    pr = np.ascontiguousarray(probabilities, dtype=np.float64)
    dev = ts.device
    win = torch.empty(n, dtype=torch.uint8, device=dev)
    lab = torch.empty((n, T, W), dtype=torch.uint8, device=dev)
    rt = torch.empty((n, T), dtype=torch.uint8, device=dev) if routed else None
    a = ZipArgs(n, _p(user_bytes), _p(user_off), _p(ad_bytes), _p(ad_off), _p(ts), T, _p(conv),
                _p(conv_present), W, ctypes.c_void_p(dur.ctypes.data),
                ctypes.c_void_p(pr.ctypes.data), seed, _p(win), _p(lab), _p(rt),
                1 if check_errors else 0)
    check(_lib.lattice_zipper_assign_labels(ctypes.byref(a), _stream(stream)))
    return win, lab, rt


def synth_impressions(n, tasks, seed, device="cuda", stream=None):
    """Synthetic impression log columns (device): (user_bytes, user_off, ad_bytes, ad_off, ts,
    conv [n,T], present [n,T])."""
    import torch
    kw = dict(device=device)
    ub = torch.empty(9 * n, dtype=torch.uint8, **kw)
    uo = torch.empty(n + 1, dtype=torch.int64, **kw)
    ab = torch.empty(7 * n, dtype=torch.uint8, **kw)
    ao = torch.empty(n + 1, dtype=torch.int64, **kw)
    ts = torch.empty(n, dtype=torch.int64, **kw)
    conv = torch.empty((n, tasks), dtype=torch.int64, **kw)
    pres = torch.empty((n, tasks), dtype=torch.uint8, **kw)
    check(_lib.lattice_synth_impressions(n, tasks, seed, _p(ub), _p(uo), _p(ab), _p(ao), _p(ts),
                                         _p(conv), _p(pres), _stream(stream)))
    return ub, uo, ab, ao, ts, conv, pres


def route_heads(logits, window, tasks, windows, out=None, stream=None):
    """out[b][t] = logits[b][t*windows + window[b]] (the Zipper window mask applied to heads)."""
    import torch
    B = logits.shape[0]
    if out is None:
        out = torch.empty((B, tasks), dtype=torch.float32, device=logits.device)
    check(_lib.lattice_route_heads(B, tasks, windows, _p(logits), _p(window), _p(out), _stream(stream)))
    return out


def correlation_loss(x, y, eps=1e-6, check_errors=True, stream=None):
    """lattice::correlation_loss (numerics.hpp:46) per column of fp64 CUDA matrices x, y [n, cols]
    (1-D vectors are one column). Returns fp64 [cols]."""
    import torch
    if x.dim() == 1:
        x, y = x[:, None], y[:, None]
    n, cols = x.shape
    out = torch.empty(cols, dtype=torch.float64, device=x.device)
    check(_lib.lattice_correlation_loss(n, cols, _p(x), x.stride(0), _p(y), y.stride(0), eps, _p(out),
                                        1 if check_errors else 0, _stream(stream)))
    return out


def window_summary(window, labels, windows, check_errors=True, stream=None):
    """lattice::window_routing_summary (datasets.hpp:262) over device columns: window uint8 [n],
    labels uint8 [n, T, W]. Returns (counts int64 [W], positives int64 [W, T])."""
    import torch
    n = window.shape[0]
    T = labels.shape[1] if labels.dim() == 3 else 0
    counts = torch.empty(windows, dtype=torch.int64, device=window.device)
    pos = torch.empty((windows, T), dtype=torch.int64, device=window.device)
    check(_lib.lattice_window_summary(n, T, windows, _p(window), _p(labels), _p(counts), _p(pos),
                                      1 if check_errors else 0, _stream(stream)))
    return counts, pos


def routed_objectives(logits, window, labels, tasks, windows, eps=1e-6, routed=None, check_errors=True,
                      stream=None, out=None):
    """Post-tower batch step: routed logits, per-task correlation loss (routed label vs
    sigmoid(routed logit), fp64) and the window summary. Returns (routed, corr, counts, positives)."""
    import torch
    n = logits.shape[0]
    dev = logits.device
    if out is None:
        out = (torch.empty((n, tasks), dtype=torch.float32, device=dev),
               torch.empty(tasks, dtype=torch.float64, device=dev),
               torch.empty(windows, dtype=torch.int64, device=dev),
               torch.empty((windows, tasks), dtype=torch.int64, device=dev))
    r, corr, counts, pos = out
    a = ObjectiveArgs(n, tasks, windows, _p(logits), _p(window), _p(labels), eps, _p(r), _p(corr), _p(counts),
                      _p(pos), 1 if check_errors else 0)
    check(_lib.lattice_routed_objectives(ctypes.byref(a), _stream(stream)))
    return out


def stable_hash(bytes_, off, seed, stream=None):
    import torch
    n = off.shape[0] - 1
    out = torch.empty(n, dtype=torch.int64, device=off.device)
    check(_lib.lattice_stable_hash(n, _p(bytes_), _p(off), seed, _p(out), _stream(stream)))
    return out


# ---- embedding bag ----------------------------------------------------------------------------

def embedding_bag(tables, offsets, ids, batch, out=None, out_dtype=None, sample_pos=None,
                  normalize=False, out_row_stride=None, out_feature_offset=0, check_errors=True,
                  stream=None, table_ptrs=None, rows=None, sources=1, slice_cap=0):
    """Sum-pooled embedding bags. tables: list of [rows_f, D] CUDA tensors (f32 or bf16).
    offsets int64 [R*F*B+1] CSR with bags laid out [R][F][B] (R = sources, 1 = plain
    feature-major), ids int32. Returns out [R*B, F, D]."""
    import torch
    F = len(tables)
    D = tables[0].shape[1]
    tdt = tables[0].dtype
    odt = out_dtype or tdt
    dev = tables[0].device
    if table_ptrs is None:
        table_ptrs = torch.tensor([t.data_ptr() for t in tables], dtype=torch.int64, device=dev)
    if rows is None:
        rows = torch.tensor([t.shape[0] for t in tables], dtype=torch.int64, device=dev)
    if out is None:
        out = torch.empty((sources * batch, F, D), dtype=odt, device=dev)
    stride = out_row_stride if out_row_stride is not None else F * D
    a = BagArgs(F, batch, D, F32 if tdt == torch.float32 else BF16, _p(table_ptrs), _p(rows),
                _p(offsets), _p(ids), F32 if odt == torch.float32 else BF16, _p(out), stride,
                out_feature_offset, _p(sample_pos), 1 if normalize else 0, 1 if check_errors else 0,
                sources, slice_cap)
    check(_lib.lattice_embedding_bag(ctypes.byref(a), _stream(stream)))
    return out


def peer_embedding_bag(rank, world, tables, table_ptrs, rows, feature_base, batch, offsets_ptrs,
                       ids_ptrs, pos_ptrs, out_ptrs, out_row_stride, out_dtype=None, normalize=True,
                       check_errors=False, stream=None):
    """Owner side of the peer-memory sharded embedding stage (lattice_peer_embedding_bag):
    the *_ptrs arguments are int64 CUDA tensors [world] of (peer-mapped) device pointers."""
    import torch
    D = tables[0].shape[1]
    tdt = tables[0].dtype
    odt = out_dtype or tdt
    a = PeerBagArgs(rank, world, len(tables), feature_base, batch, D, F32 if tdt == torch.float32 else BF16,
                    _p(table_ptrs), _p(rows), _p(offsets_ptrs), _p(ids_ptrs), _p(pos_ptrs), _p(out_ptrs),
                    F32 if odt == torch.float32 else BF16, out_row_stride, 1 if normalize else 0,
                    1 if check_errors else 0)
    check(_lib.lattice_peer_embedding_bag(ctypes.byref(a), _stream(stream)))


IPC_HANDLE_BYTES = 64


def ipc_handle(ptr):
    """-> (64-byte handle of the allocation holding device pointer `ptr`, byte offset)."""
    buf = (ctypes.c_uint8 * IPC_HANDLE_BYTES)()
    off = _I64()
    check(_lib.lattice_ipc_handle(ctypes.c_void_p(int(ptr)), buf, ctypes.byref(off)))
    return bytes(buf), off.value


def ipc_open(handle, offset):
    """Map a peer rank's exported allocation; returns the device pointer at `offset`."""
    buf = (ctypes.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(handle)
    out = ctypes.c_void_p()
    check(_lib.lattice_ipc_open(buf, offset, ctypes.byref(out)))
    return out.value


def ipc_close(ptr):
    check(_lib.lattice_ipc_close(ctypes.c_void_p(int(ptr))))


def peer_barrier(flag_ptrs, rank, world, status, timeout_s=30.0, stream=None):
    """Stream-ordered cross-GPU barrier over peer-mapped flag arrays (lattice_peer_barrier)."""
    check(_lib.lattice_peer_barrier(_p(flag_ptrs), rank, world, timeout_s, _p(status), _stream(stream)))


def peer_reduce_sgd(grad_ptrs, master, segs, n, rank, world, lr, stream=None):
    """lattice_peer_reduce_sgd: grad_ptrs int64 device tensor [world] of peer-mapped pointers;
    master: this rank's flat fp32 masters (its shard is updated); segs: list of
    (offset, count, mode, dst_dtype, dst_ptrs tensor [world])."""
    arr = (PeerSeg * len(segs))()
    for i, (off, cnt, mode, dt, dst) in enumerate(segs):
        arr[i] = PeerSeg(off, cnt, mode, dt, ctypes.c_void_p(dst.data_ptr()))
    check(_lib.lattice_peer_reduce_sgd(_p(grad_ptrs), _p(master), arr, len(segs), n, rank, world, lr,
                                       _stream(stream)))


def merge_dense(domain, values, src_col, out_width, out_dtype=None, check_errors=True, stream=None):
    """merge_domains for dense values (datasets.hpp:144-173): domain int32 [n], values fp32
    [n, max_declared] in each record's domain order, src_col int32 [G, out_width] (union column ->
    declared index or -1). Returns [n, out_width] (bf16 by default) with zero padding."""
    import torch
    n, md = values.shape
    G = src_col.shape[0]
    odt = out_dtype or torch.bfloat16
    out = torch.empty((n, out_width), dtype=odt, device=values.device)
    code = {torch.float32: F32, torch.bfloat16: BF16, torch.float64: F64}
    check(_lib.lattice_merge_dense(n, G, md, _p(domain), _p(values), code[values.dtype], _p(src_col), out_width,
                                   code[odt], _p(out), 1 if check_errors else 0, _stream(stream)))
    return out


def jsonl_columns(content, source="records", stream=None):
    """parse_jsonl_records (serde.hpp:158-170) on the GPU: content = the JSONL file as bytes or a
    uint8 CUDA tensor. Returns a dict of CUDA tensors: domain/user/ad (+ _off [records+1]), ts,
    line, feature_off/feature_key/feature_key_off/feature_val, conversion_* (lattice_jsonl_extract).
    A bad line raises DataError("<source>:<line>: ...")."""
    import torch
    if isinstance(content, (bytes, bytearray)):
        buf = torch.frombuffer(bytearray(content), dtype=torch.uint8) if len(content) else torch.empty(0, dtype=torch.uint8)
        content = buf.cuda()
    dev = content.device
    h = _P()
    info = JsonlInfo()
    check(_lib.lattice_jsonl_open(_p(content) if content.numel() else None, content.numel(), source.encode(),
                                  ctypes.byref(h), ctypes.byref(info), _stream(stream)))
    try:
        N = info.records
        u8 = lambda n: torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        i64 = lambda n: torch.empty(n, dtype=torch.int64, device=dev)
        out = {"domain": u8(info.domain_bytes), "domain_off": i64(N + 1), "user": u8(info.user_bytes),
               "user_off": i64(N + 1), "ad": u8(info.ad_bytes), "ad_off": i64(N + 1), "ts": i64(max(N, 1)),
               "line": i64(max(N, 1)), "feature_off": i64(N + 1), "feature_key": u8(info.feature_key_bytes),
               "feature_key_off": i64(info.feature_entries + 1),
               "feature_val": torch.empty(max(info.feature_entries, 1), dtype=torch.float64, device=dev),
               "conversion_off": i64(N + 1), "conversion_key": u8(info.conversion_key_bytes),
               "conversion_key_off": i64(info.conversion_entries + 1),
               "conversion_val": i64(max(info.conversion_entries, 1))}
        cols = JsonlColumns(**{k: _p(v) for k, v in out.items()})
        check(_lib.lattice_jsonl_extract(h, ctypes.byref(cols), _stream(stream)))
    finally:
        _lib.lattice_jsonl_close(h)
    out["records"], out["lines"] = N, info.lines
    return out


def jsonl_task_columns(cols, tasks, stream=None):
    """Conversion entries -> the Zipper's label inputs for `tasks` (names): conv int64 [N, T],
    present uint8 [N, T] (lattice_jsonl_task_columns)."""
    import torch
    N, dev = cols["records"], cols["ts"].device
    tb = b"".join(t.encode() for t in tasks)
    toff = [0]
    for t in tasks:
        toff.append(toff[-1] + len(t.encode()))
    tbytes = torch.tensor(list(tb) or [0], dtype=torch.uint8, device=dev)
    toff = torch.tensor(toff, dtype=torch.int64, device=dev)
    conv = torch.zeros((max(N, 1), len(tasks)), dtype=torch.int64, device=dev)
    pres = torch.zeros((max(N, 1), len(tasks)), dtype=torch.uint8, device=dev)
    check(_lib.lattice_jsonl_task_columns(N, _p(cols["conversion_off"]), _p(cols["conversion_key"]),
                                          _p(cols["conversion_key_off"]), _p(cols["conversion_val"]), len(tasks),
                                          _p(tbytes), _p(toff), _p(conv), _p(pres), _stream(stream)))
    return conv[:N], pres[:N]


def jsonl_records(content, source="records"):
    """parse_jsonl_records as Python records (dicts with the reference's DomainRecord fields;
    strings decoded as UTF-8), for tests and small files."""
    c = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in jsonl_columns(content, source).items()}
    s = lambda buf, off, i: bytes(buf[off[i]:off[i + 1]]).decode("utf-8")
    recs = []
    for r in range(c["records"]):
        feats = {}
        for e in range(c["feature_off"][r], c["feature_off"][r + 1]):
            feats[s(c["feature_key"], c["feature_key_off"], e)] = float(c["feature_val"][e])
        convs = {}
        for e in range(c["conversion_off"][r], c["conversion_off"][r + 1]):
            convs[s(c["conversion_key"], c["conversion_key_off"], e)] = int(c["conversion_val"][e])
        recs.append({"domain": s(c["domain"], c["domain_off"], r), "user_id": s(c["user"], c["user_off"], r),
                     "ad_id": s(c["ad"], c["ad_off"], r), "impression_time_ms": int(c["ts"][r]),
                     "features": feats, "conversions": convs, "line": int(c["line"][r])})
    return recs


def union_schema(declared):
    """First-seen union of feature names (datasets.hpp:125-132) and the src_col map merge_dense
    takes: declared = list of per-domain feature-name lists -> (union names, src_col [G][len(union)])
    (pad the columns with -1 for a wider, GEMM-aligned output)."""
    union, seen = [], set()
    for feats in declared:
        for f in feats:
            if f not in seen:
                seen.add(f)
                union.append(f)
    src = [[feats.index(u) if u in feats else -1 for u in union] for feats in declared]
    return union, src


def student_inputs(base, slot, store_emb, written_at, ttl_ms, now, store_logit=None, clip=0.0, smoothing=-1.0,
                   out_dtype=None, stream=None):
    """KTAP student-input assembly (ktap.hpp:133-152, 221-229): rows [n, base_dim + dim] =
    [base || clip(teacher embedding) on a valid hit, zeros otherwise], the (smoothed) teacher
    logit (NaN on a miss) and the hit flags. base fp32 [n, base_dim], slot int64 [n] (-1 absent),
    store_emb fp32 [entries, dim], written_at int64 [entries]."""
    import torch
    n, bd = base.shape
    dim = store_emb.shape[1]
    odt = out_dtype or torch.bfloat16
    out = torch.empty((n, bd + dim), dtype=odt, device=base.device)
    logit = torch.empty(n, dtype=torch.float32, device=base.device) if store_logit is not None else None
    hit = torch.empty(n, dtype=torch.uint8, device=base.device)
    a = StudentArgs(n, bd, dim, _p(base), _p(slot), _p(store_emb), _p(store_logit), _p(written_at), ttl_ms, now,
                    clip, smoothing, F32 if odt == torch.float32 else BF16, _p(out), _p(logit), _p(hit))
    check(_lib.lattice_student_inputs(ctypes.byref(a), _stream(stream)))
    return out, logit, hit


def clip_features(x, c, stream=None):
    """numerics.hpp:139 on an fp64 CUDA tensor."""
    import torch
    out = torch.empty_like(x)
    check(_lib.lattice_clip_features(x.numel(), _p(x), c, _p(out), _stream(stream)))
    return out


def smooth_labels(y, eps_s, check_errors=True, stream=None):
    """numerics.hpp:147 on an fp64 CUDA tensor of 0/1 labels."""
    import torch
    out = torch.empty_like(y)
    check(_lib.lattice_smooth_labels(y.numel(), _p(y), eps_s, _p(out), 1 if check_errors else 0, _stream(stream)))
    return out


def swish_rn_jvp(x, tangent, eps=1e-6, check_errors=True, stream=None):
    """numerics.hpp:113 per row of fp64 CUDA matrices (1-D = one row)."""
    import torch
    if x.shape != tangent.shape:
        raise UsageError("swish_rn_jvp: length mismatch")
    width = x.shape[-1] if x.dim() else 0
    rows = x.numel() // width if width else 0
    out = torch.empty_like(x)
    check(_lib.lattice_swish_rn_jvp(rows, width, eps, _p(x), _p(tangent), _p(out), 1 if check_errors else 0,
                                    _stream(stream)))
    return out


def lengths_to_offsets(lengths, out=None, stream=None):
    """int32 bag lengths [n] -> int64 CSR offsets [n+1] (exclusive scan on the GPU)."""
    import torch
    n = lengths.numel()
    if out is None:
        out = torch.empty(n + 1, dtype=torch.int64, device=lengths.device)
    check(_lib.lattice_lengths_to_offsets(n, _p(lengths), _p(out), _stream(stream)))
    return out


def pack_slices(bounds, ids, cap, out, overflow, stream=None):
    """out[o][j] = ids[bounds[o] + j] for the W = len(bounds)-1 slices; sizes read on device."""
    check(_lib.lattice_pack_slices(bounds.numel() - 1, _p(bounds), _p(ids), cap, _p(out), _p(overflow),
                                   _stream(stream)))
    return out


def rownorm(x, mode=1, eps=1e-6, check_errors=True, stream=None):
    """mode 0 rms_norm, 1 swish_rn, 2 swish_rn_hard over the last dim of an fp32 matrix (the
    epilogue arithmetic) or an fp64 one (the reference's arithmetic, lattice_rownorm_f64)."""
    import torch
    x = x.contiguous()
    out = torch.empty_like(x)
    rows = x.numel() // x.shape[-1] if x.numel() else 0
    fn = _lib.lattice_rownorm_f64 if x.dtype == torch.float64 else _lib.lattice_rownorm
    check(fn(mode, rows, x.shape[-1], eps, _p(x), _p(out), 1 if check_errors else 0, _stream(stream)))
    return out


def fill_tables(tables, seed, feature_base=0, rows_total=None, stream=None):
    """tables: contiguous [F, rows, D] tensor (f32 or bf16)."""
    import torch
    F, R, D = tables.shape
    check(_lib.lattice_fill_tables(_p(tables), F32 if tables.dtype == torch.float32 else BF16, F,
                                   R, D, seed, feature_base, rows_total or R, _stream(stream)))
    return tables


def fill_weights(w, seed, tag, stream=None):
    import torch
    out_f, fan_in = w.shape[-2], w.shape[-1]
    rows = w.numel() // fan_in
    check(_lib.lattice_fill_weights(_p(w), F32 if w.dtype == torch.float32 else BF16, rows,
                                    fan_in, seed, tag, _stream(stream)))
    return w


def synth_bags(F, B, max_len, rows, seed, device="cuda", stream=None):
    import torch
    offsets = torch.empty(F * B + 1, dtype=torch.int64, device=device)
    ids = torch.empty(max(F * B * max_len, 1), dtype=torch.int32, device=device)
    check(_lib.lattice_synth_bags(F, B, max_len, rows, seed, _p(offsets), _p(ids), _stream(stream)))
    return offsets, ids


def synth_domains(B, G, seed, device="cuda", stream=None):
    import torch
    dom = torch.empty(B, dtype=torch.int32, device=device)
    check(_lib.lattice_synth_domains(B, G, seed, _p(dom), _stream(stream)))
    return dom


def domain_bucket(domain, G, stream=None):
    import torch
    B = domain.shape[0]
    pos = torch.empty(B, dtype=torch.int32, device=domain.device)
    order = torch.empty(B, dtype=torch.int32, device=domain.device)
    seg = torch.empty(G + 1, dtype=torch.int32, device=domain.device)
    check(_lib.lattice_domain_bucket(B, G, _p(domain), _p(pos), _p(order), _p(seg), _stream(stream)))
    return pos, order, seg


# ---- GEMM ---------------------------------------------------------------------------------------

EPI_STORE, EPI_SWISH, EPI_SWISH_HARD, EPI_RESID_NORM = 0, 1, 2, 3


def gemm(A, B, epilogue=EPI_STORE, out_dtype=None, resid=None, group=128, out=None, stream=None,
         a_t=False, b_t=False):
    """C = A @ B^T with A [M,K], B [N,K] both bf16 (kind::f16) or both fp32 (kind::tf32) on
    tcgen05; fused epilogue. resid (epilogue 3) has the output dtype. a_t / b_t: the operand is
    given transposed (A as [K,M], B as [K,N], bf16) and read MN-major in place."""
    import torch
    M, K = (A.shape[1], A.shape[0]) if a_t else A.shape
    N = B.shape[1] if b_t else B.shape[0]
    f32_in = A.dtype == torch.float32
    odt = out_dtype or (torch.float32 if f32_in else torch.bfloat16)
    if out is None:
        out = torch.empty((M, N), dtype=odt, device=A.device)
    a = GemmArgs(M, N, K, _p(A), A.stride(0), _p(B), B.stride(0), _p(out), out.stride(0),
                 F32 if odt == torch.float32 else BF16, epilogue, _p(resid),
                 resid.stride(0) if resid is not None else 0, group, F32 if f32_in else BF16,
                 1 if a_t else 0, 1 if b_t else 0)
    check(_lib.lattice_gemm(ctypes.byref(a), _stream(stream)))
    return out


def fm_lcb(X, YT, WL, nF, Fin=None, Xout=None, stream=None):
    """K2 alone (lattice_fm_lcb): X [B, n, d], YT [k, n], WL [nL, n], all bf16 (or all fp32).
    Returns (Fin [B, n*k], Xout [B, n, d] with rows [nF, n) written)."""
    import torch
    B, n, d = X.shape
    k, nL = YT.shape[0], WL.shape[0]
    if Fin is None:
        Fin = torch.empty((B, n * k), dtype=X.dtype, device=X.device)
    if Xout is None:
        Xout = torch.zeros_like(X)
    a = FmLcbArgs(B, n, d, k, nF, nL, F32 if X.dtype == torch.float32 else BF16, _p(X), _p(YT),
                  _p(WL) if nL else None, _p(Fin), _p(Xout))
    check(_lib.lattice_fm_lcb(ctypes.byref(a), _stream(stream)))
    return Fin, Xout


def rownorm_vjp(x, g, mode=1, eps=1e-6, stream=None):
    """J(x)^T g per row (lattice_rownorm_vjp): mode 0 rms_norm, 1 swish_rn, 2 swish_rn_hard;
    x, g fp32 or fp64 CUDA matrices [rows, width]."""
    import torch
    x, g = x.contiguous(), g.contiguous()
    out = torch.empty_like(x)
    rows = x.numel() // x.shape[-1] if x.numel() else 0
    check(_lib.lattice_rownorm_vjp(mode, rows, x.shape[-1], eps, F64 if x.dtype == torch.float64 else F32, _p(x),
                                   _p(g), _p(out), _stream(stream)))
    return out


def routed_bce(logits, window, labels, tasks, windows, dlogits=None, loss=None, stream=None):
    """Window-routed BCE of the heads (lattice_routed_bce): (loss fp64 scalar tensor, dlogits)."""
    import torch
    n = logits.shape[0]
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if loss is None:
        loss = torch.empty((), dtype=torch.float64, device=logits.device)
    check(_lib.lattice_routed_bce(n, tasks, windows, _p(logits), _p(window), _p(labels), _p(dlogits), _p(loss),
                                  _stream(stream)))
    return loss, dlogits


def device_check(stream=None):
    """lattice_device_check: synchronise and raise CudaError if a swish GEMM's row-statistics
    exchange timed out since the last check."""
    check(_lib.lattice_device_check(_stream(stream)))


# ---- network -------------------------------------------------------------------------------------

class _CAI:
    """Minimal __cuda_array_interface__ holder to view library-owned device memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def _view(ptr, shape, dtype):
    import torch
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CAI(ptr, shape, "<i2"), device="cuda").view(torch.bfloat16)
    return torch.as_tensor(_CAI(ptr, shape, "<f4"), device="cuda")


def _pad16(x):
    return (x + 15) // 16 * 16


class Network:
    """lattice::Network over the C ABI (lattice_net_*). Weights live on the current device."""

    def __init__(self, n, d, blocks, nF, nL, k, mlp, domains, heads, tower_hidden, hard=False,
                 max_batch=32768, weight_seed=0x1A78, dtype="bf16", dense_features=0, dense_in=0,
                 dense_hidden=0):
        """dtype "bf16" (kind::f16 tensor cores) or "f32" (fp32 storage, kind::tf32; d=64).
        dense_features > 0: the last dense_features of the n embeddings come from the dense
        processor over a [B, dense_in] dense matrix (forward(dense=...))."""
        self.cfg = dict(n=n, d=d, blocks=blocks, nF=nF, nL=nL, k=k, mlp=list(mlp), domains=domains,
                        heads=heads, tower_hidden=tower_hidden, hard=hard, max_batch=max_batch,
                        weight_seed=weight_seed, dtype=dtype, dense_features=dense_features,
                        dense_in=dense_in, dense_hidden=dense_hidden)
        c = NetConfig()
        c.n, c.d, c.blocks, c.nF, c.nL, c.k = n, d, blocks, nF, nL, k
        c.n_mlp = len(mlp) - 1
        for i, w in enumerate(mlp):
            c.mlp[i] = w
        c.domains, c.heads, c.tower_hidden, c.hard = domains, heads, tower_hidden, int(hard)
        c.max_batch, c.weight_seed = max_batch, weight_seed
        c.dtype = F32 if dtype in ("f32", "fp32", "float32") else BF16
        c.dense_features, c.dense_in, c.dense_hidden = dense_features, dense_in, dense_hidden
        h = ctypes.c_void_p()
        check(_lib.lattice_net_create(ctypes.byref(c), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.lattice_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, domain, offsets=None, ids=None, table_ptrs=None, rows=None,
                table_dtype=None, pooled=None, logits=None, stream=None, shards=0, dense=None,
                check_errors=False):
        """shards > 0: `pooled` is the table-wise sharded, owner-normalised bf16 layout
        [S][B][n/S][d] received from the pooled all-to-all. check_errors: synchronise after the
        embedding stage and raise DataError for an id outside its table (lattice_batch.check)."""
        import torch
        B = domain.shape[0]
        if logits is None:
            logits = torch.empty((B, self.cfg["heads"]), dtype=torch.float32, device=domain.device)
        b = Batch()
        b.batch = B
        b.domain = _p(domain)
        if pooled is not None:
            b.table_dtype = F32 if pooled.dtype == torch.float32 else BF16
            b.pooled = _p(pooled)
            b.pooled_layout = 1 if shards else 0
            b.shards = shards
        else:
            b.table_dtype = F32 if table_dtype == torch.float32 else BF16
            b.tables, b.rows, b.offsets, b.ids = _p(table_ptrs), _p(rows), _p(offsets), _p(ids)
        b.dense = _p(dense)
        b.check = 1 if check_errors else 0
        check(_lib.lattice_net_forward(self._h, ctypes.byref(b), _p(logits), _stream(stream)))
        return logits

    def bucket(self, domain, stream=None):
        """Domain bucketing ahead of an in-place forward (lattice_net_bucket)."""
        check(_lib.lattice_net_bucket(self._h, domain.shape[0], _p(domain), _stream(stream)))

    def buffer(self, which):
        """Device pointer of a workspace buffer (lattice_net_buffer): 0 = X0 / even blocks'
        input, 1 = sample_pos, 2 = odd blocks' input, 3 = the last block's MLP input Fin."""
        p = _lib.lattice_net_buffer(self._h, which)
        if not p:
            raise UsageError(f"lattice_net_buffer: unknown buffer {which}")
        return p

    def activations(self, layer, batch):
        """X_layer of the last forward in the caller's sample order, [batch, n, d] (a copy):
        layer = blocks (the towers' input) or blocks - 1 (the last block's input)."""
        import torch
        c = self.cfg
        if layer not in (c["blocks"], c["blocks"] - 1):
            raise UsageError("activations: only X_L and X_{L-1} survive a forward")
        dt = torch.float32 if c["dtype"] in ("f32", "fp32", "float32") else torch.bfloat16
        X = _view(self.buffer(2 if layer & 1 else 0), (batch, c["n"], c["d"]), dt)
        pos = torch.as_tensor(_CAI(self.buffer(1), (batch,), "<i4"), device="cuda").long()
        return X[pos].clone()

    def forward_in_place(self, domain, logits=None, stream=None, dense=None):
        """Forward over an X0 already filled by lattice_peer_embedding_bag (pooled_layout 2)."""
        import torch
        B = domain.shape[0]
        if logits is None:
            logits = torch.empty((B, self.cfg["heads"]), dtype=torch.float32, device=domain.device)
        b = Batch()
        b.batch = B
        b.domain = _p(domain)
        b.table_dtype = F32 if self.cfg["dtype"] in ("f32", "fp32", "float32") else BF16
        b.pooled_layout = 2
        b.dense = _p(dense)
        check(_lib.lattice_net_forward(self._h, ctypes.byref(b), _p(logits), _stream(stream)))
        return logits

    def tower_backward(self, dlogits, dW1=None, dW2=None, dX=None, dx_dtype=None, stream=None):
        """Gradients of the untied towers after a forward of dlogits.shape[0] samples
        (lattice_net_tower_backward): dW1 fp32 [G, th, n*d], dW2 fp32 [G, heads, th], and with
        dx_dtype the towers' input gradient [B, n*d] in domain-sorted rows."""
        import torch
        c = self.cfg
        B = dlogits.shape[0]
        G, th, nd = c["domains"], c["tower_hidden"], c["n"] * c["d"]
        dev = dlogits.device
        if dW1 is None:
            dW1 = torch.empty((G, th, nd), dtype=torch.float32, device=dev)
        if dW2 is None:
            dW2 = torch.empty((G, c["heads"], th), dtype=torch.float32, device=dev)
        if dx_dtype is not None and dX is None:
            dX = torch.empty((B, nd), dtype=dx_dtype, device=dev)
        check(_lib.lattice_net_tower_backward(self._h, B, _p(dlogits.contiguous()), _p(dW1), _p(dW2), _p(dX),
                                              BF16 if dX is not None and dX.dtype == torch.bfloat16 else F32,
                                              _stream(stream)))
        return dW1, dW2, dX

    def tower_sgd(self, lr, dW1, dW2, master_W1, master_W2, stream=None):
        """master -= lr * grad and the network's tower weights refreshed (lattice_net_tower_sgd)."""
        check(_lib.lattice_net_tower_sgd(self._h, lr, _p(dW1), _p(dW2), _p(master_W1), _p(master_W2),
                                         _stream(stream)))

    def mlp_backward(self, dXout, dW=None, dFin=False, dResid=False, stream=None):
        """Gradients of the last block's FMB half (lattice_net_mlp_backward) from dXout fp32
        [B, n*d] (d loss / d X_L, domain-sorted rows): returns (dW list of fp32 [out, in] per MLP
        layer, dFin [B, n*k] or None, dResid [B, nF*d] or None)."""
        import torch
        c = self.cfg
        B = dXout.shape[0]
        widths = c["mlp"]
        dev = dXout.device
        if dW is None:
            dW = [torch.empty((widths[i + 1], widths[i]), dtype=torch.float32, device=dev)
                  for i in range(len(widths) - 1)]
        fin = torch.empty((B, widths[0]), dtype=torch.float32, device=dev) if dFin else None
        res = torch.empty((B, c["nF"] * c["d"]), dtype=torch.float32, device=dev) if dResid else None
        ptrs = (ctypes.c_void_p * len(dW))(*[t.data_ptr() for t in dW])
        check(_lib.lattice_net_mlp_backward(self._h, B, _p(dXout.contiguous()), ptrs, _p(fin), _p(res),
                                            _stream(stream)))
        return dW, fin, res

    def weight_sgd(self, block, kind, index, lr, grad, master, stream=None):
        """master -= lr * grad on one weight, the network's copy refreshed (lattice_net_weight_sgd)."""
        check(_lib.lattice_net_weight_sgd(self._h, block, kind, index, lr, _p(grad), _p(master), _stream(stream)))

    def mlp_masters(self, block=None):
        """fp32 device copies of one block's MLP weights [out, in] (default: the last block)."""
        c = self.cfg
        import torch
        blk = c["blocks"] - 1 if block is None else block
        wdt = torch.float32 if c["dtype"] in ("f32", "fp32", "float32") else torch.bfloat16
        w = c["mlp"]
        return [_view(_lib.lattice_net_weight(self._h, blk, 3, i), (w[i + 1], w[i]), wdt).float().clone()
                for i in range(len(w) - 1)]

    def weight_ptr(self, block, kind, index=0):
        """Device pointer of one weight buffer (lattice_net_weight; kinds as set_weight)."""
        p = _lib.lattice_net_weight(self._h, block, kind, index)
        if not p:
            raise UsageError(f"lattice_net_weight: no weight (block {block}, kind {kind}, index {index})")
        return p

    def tower_masters(self):
        """fp32 device copies of the towers' W1 [G, th, n*d] and W2 [G, heads, th] (SGD masters)."""
        c = self.cfg
        G, th, nd = c["domains"], c["tower_hidden"], c["n"] * c["d"]
        import torch
        wdt = torch.float32 if c["dtype"] in ("f32", "fp32", "float32") else torch.bfloat16
        W1 = _view(_lib.lattice_net_weight(self._h, 0, 4, 0), (G, th, nd), wdt).float().clone()
        W2 = _view(_lib.lattice_net_weight(self._h, 0, 5, 0), (G, c["heads"], th), torch.float32).clone()
        return W1, W2

    def set_timing(self, on=True):
        check(_lib.lattice_net_set_timing(self._h, 1 if on else 0))

    def stage_times(self):
        buf = (ctypes.c_float * 64)()
        n = _I32()
        check(_lib.lattice_net_stage_times(self._h, buf, 64, ctypes.byref(n)))
        return [buf[i] for i in range(n.value)]

    def set_weight(self, kind, src, block=0, index=0, stream=None):
        """Load caller-owned weights (lattice_net_set_weight): src a CUDA tensor, fp32 or the net
        dtype, unpadded, in the layout weights() returns (kind 1 YT, 2 WL, 3 MLP layer `index`,
        4 T1 [G, th, n*d], 5 T2 [G, heads, th], 6 D1, 7 D2)."""
        import torch
        src = src.contiguous()
        dt = F32 if src.dtype == torch.float32 else BF16
        check(_lib.lattice_net_set_weight(self._h, block, kind, index, _p(src), dt, _stream(stream)))

    def weights(self):
        """Host fp32 copies of every weight, unpadded, in the oracle's layout."""
        import torch
        c = self.cfg
        n, d, k, nL = c["n"], c["d"], c["k"], c["nL"]
        wdt = torch.float32 if c["dtype"] in ("f32", "fp32", "float32") else torch.bfloat16
        out = {"YT": [], "WL": [], "mlp": []}
        for blk in range(c["blocks"]):
            n_pad = (n + 255) // 256 * 256 if n > 256 else _pad16(n)
            yt = _view(_lib.lattice_net_weight(self._h, blk, 1, 0), (_pad16(k), n_pad), wdt)
            wl = _view(_lib.lattice_net_weight(self._h, blk, 2, 0), (256 if nL > 128 else 128, n_pad), wdt)
            out["YT"].append(yt[:k, :n].float().cpu().numpy().copy())
            out["WL"].append(wl[:nL, :n].float().cpu().numpy().copy())
            for li in range(len(c["mlp"]) - 1):
                w = _view(_lib.lattice_net_weight(self._h, blk, 3, li),
                          (c["mlp"][li + 1], c["mlp"][li]), wdt)
                out["mlp"].append(w.float().cpu().numpy().copy())
        G, th, H = c["domains"], c["tower_hidden"], c["heads"]
        out["T1"] = _view(_lib.lattice_net_weight(self._h, 0, 4, 0), (G, th, n * d),
                          wdt).float().cpu().numpy().copy()
        out["T2"] = _view(_lib.lattice_net_weight(self._h, 0, 5, 0), (G, H, th),
                          torch.float32).cpu().numpy().copy()
        if c["dense_features"]:
            nd_, di, dh = c["dense_features"], c["dense_in"], c["dense_hidden"]
            out["D1"] = _view(_lib.lattice_net_weight(self._h, 0, 6, 0), (dh, di), wdt).float().cpu().numpy().copy()
            out["D2"] = _view(_lib.lattice_net_weight(self._h, 0, 7, 0), (nd_ * d, dh), wdt).float().cpu().numpy().copy()
        return out

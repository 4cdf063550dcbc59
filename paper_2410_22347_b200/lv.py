"""ctypes binding of include/lv.h (argument marshalling only; every step runs in liblv.so).

Same names as the C ABI.  Tensors are torch CUDA tensors (device memory and streams are
PyTorch's job here); host outputs are numpy arrays.  There is no fallback: if liblv.so
is missing or the GPU is not sm_100 every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LV_LIB") or os.path.join(HERE, "liblv.so")   # LV_LIB: experiment builds

LV_F32, LV_F16, LV_BF16, LV_I8 = 0, 1, 2, 3
_DT = {"fp32": LV_F32, "f32": LV_F32, "fp16": LV_F16, "f16": LV_F16, "bf16": LV_BF16, "i8": LV_I8, "int8": LV_I8}
_TORCH_DT = {LV_F32: torch.float32, LV_F16: torch.float16, LV_BF16: torch.bfloat16, LV_I8: torch.int8}

EXPORTS = ["lv_last_error", "lv_version", "lv_fit_stats", "lv_index_create", "lv_encode_database",
           "lv_project_queries", "lv_search", "lv_search_host", "lv_timing_collect", "lv_encode_timing", "lv_assign_tags",
           "lv_index_info", "lv_index_export", "lv_index_destroy", "lv_index_set_search_dim",
           "lv_index_get_search_dim", "lv_normalize_rows", "lv_kmeans_assign", "lv_kmeans_centre_sums",
           "lv_index_create_flex", "lv_stream_insert", "lv_stream_remove", "lv_stream_observe_queries",
           "lv_stream_stats", "lv_stream_reproject", "lv_index_export_xprime", "lv_project_queries_i8",
           "lv_index_i8_scales", "lv_index_export_full"]


class LVError(RuntimeError):
    pass


class SearchDebug(ctypes.Structure):
    _fields_ = [("cand_ids", ctypes.c_void_p), ("cand_scores", ctypes.c_void_p), ("raw_scores", ctypes.c_void_p),
                ("timing", ctypes.c_int32), ("phase_ms", ctypes.c_float * 4), ("launches", ctypes.c_int32),
                ("slots", ctypes.c_int32), ("units", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("path", ctypes.c_int32), ("failed", ctypes.c_int32 * 2), ("kernel_ms", ctypes.c_float * 8)]

KERNEL_PHASES = ["project_K1", "sample_stage", "threshold_select", "main_scan", "select_K4", "rerank_K5",
                 "repairs", "total"]


_lib = None


def lib():
    """Load liblv.so (raises if it is missing: the product has no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LVError(f"{LIB_PATH} not built; run paper_2410_22347_b200/build.py (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.lv_last_error.restype = ctypes.c_char_p
        L.lv_version.restype = ctypes.c_char_p
        sig = {
            "lv_fit_stats": [vp, i64, vp, i32, i64, i32, vp, i32, vp, vp, vp],
            "lv_index_create": [ctypes.POINTER(vp), i32, i32, i32, i32, i32, vp, vp],
            "lv_encode_database": [vp, vp, i32, i64, vp, vp],
            "lv_project_queries": [vp, vp, i64, vp, vp],
            "lv_search": [vp, vp, i64, i32, i32, vp, vp, ctypes.POINTER(SearchDebug), vp],
            "lv_search_host": [vp, vp, i64, i32, i32, vp, vp, vp],
            "lv_timing_collect": [vp, vp, ctypes.POINTER(i32)],
            "lv_encode_timing": [vp, vp],
            "lv_index_set_search_dim": [vp, i32],
            "lv_index_get_search_dim": [vp, ctypes.POINTER(i32)],
            "lv_assign_tags": [vp, i32, i64, i32, vp, i32, vp, vp],
            "lv_normalize_rows": [vp, i32, i64, i32, vp, vp],
            "lv_index_create_flex": [ctypes.POINTER(vp), i32, i32, i32, vp, vp, i64],
            "lv_project_queries_i8": [vp, vp, i64, vp, vp, vp],
            "lv_index_i8_scales": [vp, vp],
            "lv_stream_insert": [vp, vp, i32, i64, vp, vp],
            "lv_stream_remove": [vp, vp, i64, vp],
            "lv_stream_observe_queries": [vp, vp, i64, vp],
            "lv_stream_stats": [vp, vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64), vp],
            "lv_stream_reproject": [vp, vp, vp, vp],
            "lv_index_export_xprime": [vp, vp, vp, vp],
            "lv_kmeans_assign": [vp, i32, i64, i32, vp, i32, vp, vp, i32, vp],
            "lv_kmeans_centre_sums": [vp, i32, i64, i32, vp, i32, vp, vp, vp],
            "lv_index_info": [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32),
                              ctypes.POINTER(i32), ctypes.POINTER(i32)],
            "lv_index_export": [vp, vp, vp, vp, vp],
            "lv_index_export_full": [vp, vp, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.lv_index_destroy.argtypes = [vp]
        L.lv_index_destroy.restype = None
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise LVError(f"{what}: status {status}: {lib().lv_last_error().decode()}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, dtype=None) -> torch.Tensor:
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise LVError("expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise LVError(f"expected dtype {dtype}, got {t.dtype}")
    return t.contiguous()


def _out(t, shape, dtype, what: str, host: bool = False):
    """Caller-supplied output buffer: exact shape, dtype, device and contiguity (the library writes
    [shape] elements through the raw pointer)."""
    if not isinstance(t, torch.Tensor):
        raise LVError(f"{what}: expected a torch tensor")
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or t.is_cuda == host:
        raise LVError(f"{what}: need a contiguous {'host' if host else 'CUDA'} {dtype} tensor of shape {tuple(shape)}, "
                      f"got {t.dtype} {tuple(t.shape)} on {t.device} (contiguous={t.is_contiguous()})")
    return t


def _xdtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return LV_F32
    if t.dtype == torch.float16:
        return LV_F16
    raise LVError(f"unsupported vector dtype {t.dtype}")


def lv_version() -> str:
    return lib().lv_version().decode()


def lv_fit_stats(Q_learn: torch.Tensor, X_learn: torch.Tensor, assign_learn: torch.Tensor | None = None, C: int = 1):
    """K_Q = sum q q^T and K_X[c] = sum_{x in X_c} x x^T.  Returns fp64 numpy."""
    Q = _dev(Q_learn, torch.float32)
    X = _dev(X_learn)
    D = Q.shape[1]
    a = None if assign_learn is None else _dev(assign_learn, torch.int32)
    KQ = np.zeros((D, D), dtype=np.float64)
    KX = np.zeros((C, D, D), dtype=np.float64)
    _check(lib().lv_fit_stats(_ptr(Q), Q.shape[0], _ptr(X), _xdtype(X), X.shape[0], D, _ptr(a), C,
                              KQ.ctypes.data_as(ctypes.c_void_p), KX.ctypes.data_as(ctypes.c_void_p), _stream()),
           "lv_fit_stats")
    return KQ, KX


class Index:
    """Owns an lv_index* (freed by lv_index_destroy)."""

    def __init__(self, D: int, d: int, C: int, low: str, full: str, A_stack, B_stack, id_capacity: int = 0):
        A = _dev(torch.as_tensor(A_stack, dtype=torch.float32, device="cuda"), torch.float32)
        B = _dev(torch.as_tensor(B_stack, dtype=torch.float32, device="cuda"), torch.float32)
        h = ctypes.c_void_p()
        self.flex = id_capacity > 0
        if self.flex:
            if tuple(A.shape) != (D, D) or tuple(B.shape) != (D, D):
                raise LVError("lv_index_create_flex: A', B' must be [D, D]")
            _check(lib().lv_index_create_flex(ctypes.byref(h), D, d, _DT[low], _ptr(A), _ptr(B), int(id_capacity)),
                   "lv_index_create_flex")
        else:
            _check(lib().lv_index_create(ctypes.byref(h), D, d, C, _DT[low], _DT[full], _ptr(A), _ptr(B)),
                   "lv_index_create")
        self.h = h
        self.D, self.d, self.C, self.low, self.full = D, d, C, low, full
        torch.cuda.synchronize()

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                lib().lv_index_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        n, n_pad = ctypes.c_int64(), ctypes.c_int64()
        D, d, C = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().lv_index_info(self.h, ctypes.byref(n), ctypes.byref(n_pad), ctypes.byref(D),
                                   ctypes.byref(d), ctypes.byref(C)), "lv_index_info")
        return {"n": n.value, "n_pad": n_pad.value, "D": D.value, "d": d.value, "C": C.value}


def lv_index_create(D, d, C, low, full, A_stack, B_stack) -> Index:
    return Index(D, d, C, low, full, A_stack, B_stack)


def lv_index_create_flex(D: int, d: int, low: str, A_prime, B_prime, id_capacity: int) -> Index:
    """§3.1 index storing x' = B'x (A' = P'W^+, B' = P'W, [D, D]); X_low = the first d coordinates."""
    return Index(D, d, 1, low, "fp32", A_prime, B_prime, id_capacity=id_capacity)


def _host_ids(ids) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
    if a.ndim != 1:
        raise LVError("ids must be a 1-D array")
    return a


def lv_stream_insert(index: Index, X: torch.Tensor, ids):
    X = _dev(X)
    a = _host_ids(ids)
    if a.shape[0] != X.shape[0]:
        raise LVError("lv_stream_insert: one id per row")
    _check(lib().lv_stream_insert(index.h, _ptr(X), _xdtype(X), X.shape[0], a.ctypes.data_as(ctypes.c_void_p),
                                  _stream()), "lv_stream_insert")


def lv_stream_remove(index: Index, ids):
    a = _host_ids(ids)
    _check(lib().lv_stream_remove(index.h, a.ctypes.data_as(ctypes.c_void_p), a.shape[0], _stream()), "lv_stream_remove")


def lv_stream_observe_queries(index: Index, Q: torch.Tensor):
    Q = _dev(Q, torch.float32)
    _check(lib().lv_stream_observe_queries(index.h, _ptr(Q), Q.shape[0], _stream()), "lv_stream_observe_queries")


def lv_stream_stats(index: Index):
    """(K_Q, K_X) fp64 [D, D] numpy, m_q, n."""
    KQ = np.zeros((index.D, index.D))
    KX = np.zeros((index.D, index.D))
    mq, n = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().lv_stream_stats(index.h, KQ.ctypes.data_as(ctypes.c_void_p), KX.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(mq), ctypes.byref(n), _stream()), "lv_stream_stats")
    return KQ, KX, mq.value, n.value


def lv_stream_reproject(index: Index, A_prime, B_prime):
    A = _dev(torch.as_tensor(A_prime, dtype=torch.float32, device="cuda"), torch.float32)
    B = _dev(torch.as_tensor(B_prime, dtype=torch.float32, device="cuda"), torch.float32)
    if tuple(A.shape) != (index.D, index.D) or tuple(B.shape) != (index.D, index.D):
        raise LVError("lv_stream_reproject: A', B' must be [D, D]")
    _check(lib().lv_stream_reproject(index.h, _ptr(A), _ptr(B), _stream()), "lv_stream_reproject")


def lv_index_export_xprime(index: Index):
    """(x' fp32 [n, D], ids int32 [n]) in row order (CUDA tensors)."""
    n = index.info()["n"]
    Xp = torch.empty((n, index.D), dtype=torch.float32, device="cuda")
    ids = torch.empty(n, dtype=torch.int32, device="cuda")
    _check(lib().lv_index_export_xprime(index.h, _ptr(Xp), _ptr(ids), _stream()), "lv_index_export_xprime")
    return Xp, ids


def lv_encode_database(index: Index, X: torch.Tensor, assign: torch.Tensor | None = None):
    X = _dev(X)
    a = None if assign is None else _dev(assign, torch.int32)
    _check(lib().lv_encode_database(index.h, _ptr(X), _xdtype(X), X.shape[0], _ptr(a), _stream()),
           "lv_encode_database")


def lv_index_set_search_dim(index: Index, d_search: int):
    """§3.1 flexible d: search on the first d_search reduced coordinates (<= 0: the stored d)."""
    _check(lib().lv_index_set_search_dim(index.h, int(d_search)), "lv_index_set_search_dim")


def lv_index_get_search_dim(index: Index) -> int:
    ds = ctypes.c_int32()
    _check(lib().lv_index_get_search_dim(index.h, ctypes.byref(ds)), "lv_index_get_search_dim")
    return ds.value


def lv_project_queries(index: Index, Q: torch.Tensor) -> torch.Tensor:
    """Q' [m, C * d_search] (d_search = the stored d unless lv_index_set_search_dim changed it)."""
    Q = _dev(Q, torch.float32)
    Qp = torch.empty((Q.shape[0], index.C * lv_index_get_search_dim(index)), dtype=_TORCH_DT[_DT[index.low]],
                     device=Q.device)
    _check(lib().lv_project_queries(index.h, _ptr(Q), Q.shape[0], _ptr(Qp), _stream()), "lv_project_queries")
    return Qp


def lv_project_queries_i8(index: Index, Q: torch.Tensor):
    """int8 index: query codes int8 [m, C * d_search] and scales fp32 [m, C] (R21)."""
    Q = _dev(Q, torch.float32)
    ds = lv_index_get_search_dim(index)
    codes = torch.empty((Q.shape[0], index.C * ds), dtype=torch.int8, device=Q.device)
    scales = torch.empty((Q.shape[0], index.C), dtype=torch.float32, device=Q.device)
    _check(lib().lv_project_queries_i8(index.h, _ptr(Q), Q.shape[0], _ptr(codes), _ptr(scales), _stream()),
           "lv_project_queries_i8")
    return codes, scales


def lv_index_i8_scales(index: Index) -> np.ndarray:
    """delta [C, d] fp32 of an encoded int8 index."""
    out = np.zeros((index.C, index.d), dtype=np.float32)
    _check(lib().lv_index_i8_scales(index.h, out.ctypes.data_as(ctypes.c_void_p)), "lv_index_i8_scales")
    return out


def lv_search(index: Index, Q: torch.Tensor, k: int, R: int, cand: bool = False, raw: bool = False,
              timing: int = 0, out=None):
    """Alg. 1 hot path.  Returns (ids int32 [m,k], scores fp32 [m,k], debug dict)."""
    Q = _dev(Q, torch.float32)
    m = Q.shape[0]
    if out is None:
        ids = torch.empty((m, k), dtype=torch.int32, device=Q.device)
        sc = torch.empty((m, k), dtype=torch.float32, device=Q.device)
    else:
        ids = _out(out[0], (m, k), torch.int32, "lv_search ids")
        sc = _out(out[1], (m, k), torch.float32, "lv_search scores")
    dbg = SearchDebug()
    keep = {}
    if cand:
        keep["cand_ids"] = torch.empty((m, R), dtype=torch.int32, device=Q.device)
        keep["cand_scores"] = torch.empty((m, R), dtype=torch.float32, device=Q.device)
        dbg.cand_ids = keep["cand_ids"].data_ptr()
        dbg.cand_scores = keep["cand_scores"].data_ptr()
    if raw:
        info = index.info()
        m_pad = (m + 255) // 256 * 256
        keep["raw"] = torch.full((m_pad, info["n_pad"]), float("nan"), dtype=torch.float32, device=Q.device)
        dbg.raw_scores = keep["raw"].data_ptr()
    dbg.timing = int(timing)   # 0 none, 1 synchronous (phase_ms / kernel_ms), 2 deferred (lv_timing_collect)
    _check(lib().lv_search(index.h, _ptr(Q), m, k, R, _ptr(ids), _ptr(sc), ctypes.byref(dbg), _stream()),
           "lv_search")
    keep.update({"phase_ms": list(dbg.phase_ms), "launches": dbg.launches, "slots": dbg.slots,
                 "units": dbg.units, "grid": dbg.grid, "path": dbg.path, "failed": list(dbg.failed),
                 "kernel_ms": dict(zip(KERNEL_PHASES, list(dbg.kernel_ms)))})
    return ids, sc, keep


def lv_timing_collect(index: Index):
    """Average per-kernel times (ms) of the lv_search calls made with timing=2 since the last collect."""
    ms = (ctypes.c_float * 8)()
    calls = ctypes.c_int32()
    _check(lib().lv_timing_collect(index.h, ms, ctypes.byref(calls)), "lv_timing_collect")
    return dict(zip(KERNEL_PHASES, list(ms))), calls.value


def lv_encode_timing(index: Index):
    """Kernel times (ms) of the last lv_encode_database: sort (C > 1), K6 encode, full copy."""
    ms = (ctypes.c_float * 3)()
    _check(lib().lv_encode_timing(index.h, ms), "lv_encode_timing")
    return dict(zip(["sort", "encode_K6", "full_copy"], list(ms)))


def lv_search_host(index: Index, Q_host: torch.Tensor, k: int, R: int, ids_host=None, scores_host=None):
    """lv_search on HOST buffers (copies inside the call).  Q_host: CPU fp32 (pinned is faster)."""
    Q = Q_host.contiguous()
    if Q.dtype != torch.float32 or Q.is_cuda or Q.dim() != 2 or Q.shape[1] != index.D:
        raise LVError(f"lv_search_host: need a host fp32 [m, {index.D}] query tensor")
    m = Q.shape[0]
    if ids_host is None:
        ids_host = torch.empty((m, k), dtype=torch.int32, pin_memory=Q.is_pinned())
        scores_host = torch.empty((m, k), dtype=torch.float32, pin_memory=Q.is_pinned())
    else:
        _out(ids_host, (m, k), torch.int32, "lv_search_host ids", host=True)
        _out(scores_host, (m, k), torch.float32, "lv_search_host scores", host=True)
    _check(lib().lv_search_host(index.h, ctypes.c_void_p(Q.data_ptr()), m, k, R,
                                ctypes.c_void_p(ids_host.data_ptr()), ctypes.c_void_p(scores_host.data_ptr()),
                                _stream()), "lv_search_host")
    return ids_host, scores_host


def lv_assign_tags(X: torch.Tensor, centres: torch.Tensor) -> torch.Tensor:
    X = _dev(X)
    mu = _dev(centres, torch.float32)
    out = torch.empty(X.shape[0], dtype=torch.int32, device=X.device)
    _check(lib().lv_assign_tags(_ptr(X), _xdtype(X), X.shape[0], X.shape[1], _ptr(mu), mu.shape[0], _ptr(out),
                                _stream()), "lv_assign_tags")
    return out


def lv_normalize_rows(X: torch.Tensor) -> torch.Tensor:
    """x~ = x / ||x|| (Alg. 5 line 1), fp32 out."""
    X = _dev(X)
    out = torch.empty(X.shape, dtype=torch.float32, device=X.device)
    _check(lib().lv_normalize_rows(_ptr(X), _xdtype(X), X.shape[0], X.shape[1], _ptr(out), _stream()),
           "lv_normalize_rows")
    return out


def lv_kmeans_assign(X: torch.Tensor, centres: torch.Tensor, assign: bool = True, best: torch.Tensor | None = None,
                     accumulate: bool = False):
    """E-step tags and/or the best similarity max_c <x, mu_c> (k-means++: accumulate=True keeps the
    running max in `best`).  Returns (assign or None, best)."""
    X = _dev(X)
    mu = _dev(centres, torch.float32)
    a = torch.empty(X.shape[0], dtype=torch.int32, device=X.device) if assign else None
    if best is None:
        if accumulate:
            raise LVError("lv_kmeans_assign: accumulate needs a best tensor")
        best = torch.empty(X.shape[0], dtype=torch.float32, device=X.device)
    else:
        _out(best, (X.shape[0],), torch.float32, "lv_kmeans_assign best")
    _check(lib().lv_kmeans_assign(_ptr(X), _xdtype(X), X.shape[0], X.shape[1], _ptr(mu), mu.shape[0], _ptr(a),
                                  _ptr(best), int(accumulate), _stream()), "lv_kmeans_assign")
    return a, best


def lv_kmeans_centre_sums(X: torch.Tensor, assign: torch.Tensor, C: int):
    """M-step sums per cluster (fp64 [C, D]) and counts (int64 [C]), host numpy."""
    X = _dev(X)
    a = _dev(assign, torch.int32)
    sums = np.zeros((C, X.shape[1]), dtype=np.float64)
    counts = np.zeros(C, dtype=np.int64)
    _check(lib().lv_kmeans_centre_sums(_ptr(X), _xdtype(X), X.shape[0], X.shape[1], _ptr(a), C,
                                       sums.ctypes.data_as(ctypes.c_void_p), counts.ctypes.data_as(ctypes.c_void_p),
                                       _stream()), "lv_kmeans_centre_sums")
    return sums, counts


def lv_index_export_full(index: Index):
    """X_full [n, D] in the index's full dtype, original row order (CUDA tensor)."""
    n = index.info()["n"]
    Xf = torch.empty((n, index.D), dtype=_TORCH_DT[_DT[index.full]], device="cuda")
    _check(lib().lv_index_export_full(index.h, _ptr(Xf), _stream()), "lv_index_export_full")
    return Xf


def lv_index_export(index: Index):
    info = index.info()
    X_low = torch.empty((info["n_pad"], info["d"]), dtype=_TORCH_DT[_DT[index.low]], device="cuda")
    perm = torch.empty(info["n_pad"], dtype=torch.int32, device="cuda")
    offs = np.zeros(info["C"] + 1, dtype=np.int64)
    _check(lib().lv_index_export(index.h, _ptr(X_low), _ptr(perm), offs.ctypes.data_as(ctypes.c_void_p), _stream()),
           "lv_index_export")
    return X_low, perm, offs

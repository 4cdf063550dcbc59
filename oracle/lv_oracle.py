"""fp64 oracle of the method (TEST INFRASTRUCTURE; see oracle/__init__.py).

Notation follows PAPER.md: rows of X are database vectors x_i, rows of
Q are queries q; the paper stacks them horizontally as columns,
we keep row arrays and transpose where the paper's matrices are formed.

Functions (pin in tests/test_oracle_pins.py named in brackets):
  sphering_matrix      Alg. 2 l.2-3, W = U S U^T          [Eq.(7), S:141, S:142]
  sphering_fit         Alg. 2 (LeanVec-Sphering)           [A B^T = I, d=D exact, loss optimum, S:150/S:160]
  svd_baseline_fit     query-agnostic SVD baseline [loss >= sphering]
  leanvec_loss         Problem (4) via the Eq.(6) trace form [naive double loop]
  spherical_kmeans     App. A EM with k-means++ seeding    [monotone objective, C=1 closed form]
  assign_tags          Eq.(13)                              [S:246-248 examples]
  gleanvec_fit         Alg. 5                               [C=1 == LeanVec-Sphering, per-cluster loss <= global]
  round_storage        RNE to bf16 / fp16                   [bit patterns of known values]
  encode / project     Eq.(5)/(14), Alg. 4 preprocess       [d=D exactness]
  reduced_search       Alg. 1 l.2 exhaustive + top-R        [brute force vs full sort, S:469]
  rerank_topk          Alg. 1 l.3                           [R=n -> exact k-NN]
  exact_topk, recall_at_k   P:46-48 (MIPS), P:545-546     [S:469, S:476-478]
  flexible_fit         §3.1 A' = P'W^+, B' = P'W, D x D     [<A'q, B'x> = <q,x>, prefix = smaller fit]
  eig_fit_from_stats   §3.2 eig route from K_Q, K_X          [equals the SVD route]
  StreamingIndex       §3.2 insert/remove/observe/refresh    [K_X = definition, x' = B'_new x, Eq.(12)]
  quantize_db_i8 / quantize_queries_i8 / search_i8
                       P:129, P:211 scalar quantisation (R21) [rounding bound, |code| <= 127, extremes at
                                                               +-127, exact-integer special case]
"""
from __future__ import annotations

import numpy as np

try:
    import ml_dtypes as _mld
except Exception:  # pragma: no cover
    _mld = None

PINV_EPS = 1e-6   # pseudoinverse cut-off relative to sigma_max (reading of P:194)


# ----------------------------------------------------------------------------------
# LeanVec-Sphering (Section 3, Alg. 2)
# ----------------------------------------------------------------------------------
def sphering_matrix(Qcols: np.ndarray):
    """Alg. 2 lines 2-3: SVD U S V^T of the D x m query matrix Q, W = U S U^T.

    Returns (W, W_pinv).  W_pinv = U S^+ U^T, singular values below
    PINV_EPS * sigma_max treated as zero ("we can use a pseudoinverse").
    """
    U, S, _ = np.linalg.svd(np.asarray(Qcols, dtype=np.float64), full_matrices=False)
    W = (U * S[None, :]) @ U.T
    cut = PINV_EPS * (S.max() if S.size else 0.0)
    Sinv = np.where(S > cut, 1.0 / np.where(S > cut, S, 1.0), 0.0)
    Wp = (U * Sinv[None, :]) @ U.T
    return W, Wp


def _sign_canonical_rows(P: np.ndarray) -> np.ndarray:
    """Flip each row so its largest-|entry| coordinate is positive (S:191 reading)."""
    idx = np.argmax(np.abs(P), axis=1)
    s = np.sign(P[np.arange(P.shape[0]), idx])
    s[s == 0] = 1.0
    return P * s[:, None]


def top_left_singular_rows(Y: np.ndarray, d: int) -> tuple[np.ndarray, np.ndarray]:
    """First d left singular vectors of Y (as rows, sign-canonical) and all singular values."""
    D, ncol = Y.shape
    U, S, _ = np.linalg.svd(Y, full_matrices=(ncol < d))
    S_full = np.zeros(D)
    S_full[:S.size] = S
    return _sign_canonical_rows(U[:, :d].T.copy()), S_full


def sphering_fit(Q_learn: np.ndarray, X_learn: np.ndarray, d: int, Wpair=None) -> dict:
    """Alg. 2, LeanVec-Sphering.

    1. Form Q (D x m_l) and X (D x n_l) by stacking the learning vectors.
       Q is scaled by 1/sqrt(m_l): W -> W/sqrt(m_l), A -> A sqrt(m_l), B -> B/sqrt(m_l),
       A^T B unchanged (reading R2; the product uses the same scale).
    2. W = U S U^T from the SVD of Q.
    3. P = the d left singular vectors of W X with largest singular values.
    4. A = P W^{-1}, B = P W.
    `Wpair` lets GleanVec share one W across clusters (Alg. 5 calls Alg. 2 with the
    same Q_learn for every cluster).
    """
    Q = np.asarray(Q_learn, dtype=np.float64)
    X = np.asarray(X_learn, dtype=np.float64)
    if Wpair is None:
        Wpair = sphering_matrix(Q.T / np.sqrt(Q.shape[0]))
    W, Wp = Wpair
    Y = W @ X.T
    P, sig = top_left_singular_rows(Y, d)
    return {"W": W, "Wp": Wp, "P": P, "A": P @ Wp, "B": P @ W, "sigma": sig}


def svd_baseline_fit(X_learn: np.ndarray, d: int) -> dict:
    """Query-agnostic baseline of P:555 / P:99: A = B = top-d left singular vectors of X."""
    P, sig = top_left_singular_rows(np.asarray(X_learn, dtype=np.float64).T, d)
    return {"A": P, "B": P, "P": P, "sigma": sig}


def leanvec_loss(A, B, Q_rows, X_rows) -> float:
    """Problem (4) via Eq.(6)'s first line:
    L = sum_x || Q^T (A^T B x - x) ||^2 = || Q^T (A^T B - I) X ||_F^2, Q, X stacked as columns.
    Evaluated as tr((M-I)^T K_Q (M-I) K_X), K_Q = Q Q^T, K_X = X X^T."""
    Qm = np.asarray(Q_rows, dtype=np.float64)
    Xm = np.asarray(X_rows, dtype=np.float64)
    M = np.asarray(A, dtype=np.float64).T @ np.asarray(B, dtype=np.float64)
    E = M - np.eye(M.shape[0])
    KQ = Qm.T @ Qm
    KX = Xm.T @ Xm
    return float(np.trace(E.T @ KQ @ E @ KX))


def leanvec_loss_naive(A, B, Q_rows, X_rows) -> float:
    """Problem (4) literally: sum_q sum_x (<Aq,Bx> - <q,x>)^2 (tiny inputs only)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    tot = 0.0
    for q in np.asarray(Q_rows, dtype=np.float64):
        for x in np.asarray(X_rows, dtype=np.float64):
            tot += (float(np.dot(A @ q, B @ x)) - float(np.dot(q, x))) ** 2
    return tot


# ----------------------------------------------------------------------------------
# GleanVec (Section 4, Alg. 5, Appendix A)
# ----------------------------------------------------------------------------------
def assign_tags(X: np.ndarray, centres: np.ndarray) -> np.ndarray:
    """Eq.(13): c_i = argmax_c <x_i, mu_c>; ties -> lowest index."""
    S = np.asarray(X, dtype=np.float64) @ np.asarray(centres, dtype=np.float64).T
    return np.argmax(S, axis=1).astype(np.int32)


def spherical_kmeans(Xn: np.ndarray, C: int, draws: np.ndarray, max_iter: int = 50):
    """Spherical k-means (App. A) on unit vectors Xn.

    Seeding: k-means++  with D^2(x) = 2 - 2 max_c <x, mu_c> (squared
    chordal distance on the sphere); draws[j] in [0,1) picks centre j by inverse
    CDF (the first centre: index floor(draws[0] * n)).  EM steps:
      c_i <- argmax_c <x_i, mu_c>;  mu_c <- normalize(sum_{c_i=c} x_i).
    Stops when assignments do not change or after max_iter iterations.
    An empty cluster is re-seeded with the point of lowest similarity to its
    centre (S:288 reading).  Returns (centres, assign, objective history).
    """
    X = np.asarray(Xn, dtype=np.float64)
    n = X.shape[0]
    mu = np.empty((C, X.shape[1]))
    first = min(int(draws[0] * n), n - 1)
    mu[0] = X[first]
    best = X @ mu[0]
    for j in range(1, C):
        w = np.maximum(2.0 - 2.0 * best, 0.0)
        cdf = np.cumsum(w)
        if cdf[-1] <= 0:
            pick = min(int(draws[j] * n), n - 1)
        else:
            pick = int(np.searchsorted(cdf, draws[j] * cdf[-1], side="right"))
            pick = min(pick, n - 1)
        mu[j] = X[pick]
        best = np.maximum(best, X @ mu[j])
    assign = None
    hist = []
    for _ in range(max_iter):
        S = X @ mu.T
        new = np.argmax(S, axis=1).astype(np.int32)
        hist.append(float(S[np.arange(n), new].sum()))
        if assign is not None and np.array_equal(new, assign):
            break
        assign = new
        for c in range(C):
            members = X[assign == c]
            if members.shape[0] == 0:
                sim = S[np.arange(n), assign]
                far = int(np.argmin(sim))
                mu[c] = X[far]
            else:
                s = members.sum(axis=0)
                mu[c] = s / np.linalg.norm(s)
    return mu, assign, hist


def gleanvec_fit(Q_learn, X_learn, C: int, d: int, draws, max_iter: int = 50) -> dict:
    """Alg. 5.
    1. X~ = {x / ||x||}.
    2. landmarks mu_c by spherical k-means on X~.
    3. X_c = {x in X_learn : c = argmax_c' <x/||x||, mu_c'>}.
    4. A_c, B_c by Alg. 2 from Q_learn and X_c; W shared because Q_learn is.
    """
    X = np.asarray(X_learn, dtype=np.float64)
    Q = np.asarray(Q_learn, dtype=np.float64)
    Xn = X / np.linalg.norm(X, axis=1, keepdims=True)
    if C == 1:
        centres = (Xn.sum(axis=0) / np.linalg.norm(Xn.sum(axis=0)))[None, :]
        assign = np.zeros(X.shape[0], dtype=np.int32)
    else:
        centres, _, _ = spherical_kmeans(Xn, C, draws, max_iter)
        assign = assign_tags(Xn, centres)
    Wpair = sphering_matrix(Q.T / np.sqrt(Q.shape[0]))
    A = np.empty((C, d, X.shape[1]))
    B = np.empty_like(A)
    sig = []
    for c in range(C):
        f = sphering_fit(Q, X[assign == c], d, Wpair=Wpair)
        A[c], B[c] = f["A"], f["B"]
        sig.append(f["sigma"])
    return {"centres": centres, "assign_learn": assign, "A": A, "B": B,
            "W": Wpair[0], "Wp": Wpair[1], "sigma": np.array(sig)}


# ----------------------------------------------------------------------------------
# Storage rounding (precision contract)
# ----------------------------------------------------------------------------------
def round_storage(a: np.ndarray, dtype: str) -> np.ndarray:
    """Round-to-nearest-even to the storage type, returned as fp64."""
    a = np.asarray(a, dtype=np.float64)
    if dtype == "fp16":
        return a.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        return a.astype(_mld.bfloat16).astype(np.float64)
    if dtype in ("fp32", "f32"):
        return a.astype(np.float32).astype(np.float64)
    if dtype in ("fp64", "none", None):
        return a
    raise ValueError(dtype)


# ----------------------------------------------------------------------------------
# Encode / project (Eq.(5), Eq.(14) read with g, Alg. 4)
# ----------------------------------------------------------------------------------
def encode(X, B_stack, assign=None, store: str | None = None) -> np.ndarray:
    """x_low_i = g_{c_i}(x_i) = B_{c_i} x_i (Eq.(14) with the f->g reading; Eq.(5))."""
    X = np.asarray(X, dtype=np.float64)
    B = np.asarray(B_stack, dtype=np.float64)
    if B.ndim == 2:
        B = B[None]
    if assign is None:
        assign = np.zeros(X.shape[0], dtype=np.int32)
    out = np.empty((X.shape[0], B.shape[1]))
    for c in range(B.shape[0]):
        idx = np.nonzero(assign == c)[0]
        if idx.size:
            out[idx] = X[idx] @ B[c].T
    return round_storage(out, store) if store else out


def project(Q, A_stack, store: str | None = None) -> np.ndarray:
    """Alg. 4 preprocess: q_c = A_c q for every c; Alg. 1 l.1 for C=1.
    Returns [m, C, d]."""
    Q = np.asarray(Q, dtype=np.float64)
    A = np.asarray(A_stack, dtype=np.float64)
    if A.ndim == 2:
        A = A[None]
    out = np.einsum("mD,cdD->mcd", Q, A)
    return round_storage(out, store) if store else out


# ----------------------------------------------------------------------------------
# Search (Alg. 1 with an exhaustive main step)
# ----------------------------------------------------------------------------------
def topk_total_order(scores: np.ndarray, ids: np.ndarray, k: int):
    """Top-k of one row under the total order (score desc, id asc) (reading R7)."""
    k = min(k, scores.size)
    if k <= 0:
        return np.empty(0, dtype=np.int64), np.empty(0)
    if scores.size > k:
        thr = np.partition(scores, scores.size - k)[scores.size - k]
        sel = np.nonzero(scores >= thr)[0]
    else:
        sel = np.arange(scores.size)
    order = np.lexsort((ids[sel], -scores[sel]))[:k]
    return ids[sel][order], scores[sel][order]


def reduced_scores(Qp, Xlow, assign=None) -> np.ndarray:
    """s_ji = <q'_{j, c_i}, x_low_i> (Eq.(15); C=1: Eq.(9)). [m, n]"""
    Qp = np.asarray(Qp, dtype=np.float64)
    if Qp.ndim == 2:
        Qp = Qp[:, None, :]
    Xlow = np.asarray(Xlow, dtype=np.float64)
    if assign is None:
        assign = np.zeros(Xlow.shape[0], dtype=np.int32)
    S = np.empty((Qp.shape[0], Xlow.shape[0]))
    for c in range(Qp.shape[1]):
        idx = np.nonzero(assign == c)[0]
        if idx.size:
            S[:, idx] = Qp[:, c, :] @ Xlow[idx].T
    return S


def reduced_search(Qp, Xlow, assign, R: int, chunk: int = 1 << 18, score_fp32: bool = False):
    """Alg. 1 line 2 as an exhaustive scan: N_low(j) = the R best ids under
    (reduced score desc, id asc).  Chunked over database rows, merging running lists.
    score_fp32: the scores are rounded to fp32 before ranking (the int8 path, whose scores the
    precision contract defines as fp32 values, R21).  Returns ids [m, R] int64 and scores [m, R]."""
    Xlow = np.asarray(Xlow, dtype=np.float64)
    n = Xlow.shape[0]
    assign = np.zeros(n, dtype=np.int32) if assign is None else np.asarray(assign)
    m = np.asarray(Qp).shape[0]
    R = min(R, n)
    best_ids = [np.empty(0, dtype=np.int64) for _ in range(m)]
    best_sc = [np.empty(0) for _ in range(m)]
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        S = reduced_scores(Qp, Xlow[lo:hi], assign[lo:hi])
        if score_fp32:
            S = S.astype(np.float32).astype(np.float64)
        ids = np.arange(lo, hi, dtype=np.int64)
        for j in range(m):
            cid, csc = topk_total_order(S[j], ids, R)
            allid = np.concatenate([best_ids[j], cid])
            allsc = np.concatenate([best_sc[j], csc])
            best_ids[j], best_sc[j] = topk_total_order(allsc, allid, R)
    return np.stack(best_ids), np.stack(best_sc)


def rerank_topk(Q, X, cand_ids, k: int):
    """Alg. 1 line 3: r_ji = <q_j, x_i> at full D for i in N_low(j), top-k by
    (r desc, id asc).  Returns ids [m, k], scores [m, k]."""
    Q = np.asarray(Q, dtype=np.float64)
    out_i, out_s = [], []
    for j in range(Q.shape[0]):
        ids = np.asarray(cand_ids[j], dtype=np.int64)
        r = np.asarray(X[ids], dtype=np.float64) @ Q[j]
        i, s = topk_total_order(r, ids, k)
        out_i.append(i)
        out_s.append(s)
    return np.stack(out_i), np.stack(out_s)


def exact_topk(Q, X, k: int, chunk: int = 1 << 18):
    """MIPS ground truth: top-k of <q, x_i> over all i, fp64, lowest id on ties."""
    Q = np.asarray(Q, dtype=np.float64)
    n = X.shape[0]
    m = Q.shape[0]
    best_ids = [np.empty(0, dtype=np.int64) for _ in range(m)]
    best_sc = [np.empty(0) for _ in range(m)]
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        S = Q @ np.asarray(X[lo:hi], dtype=np.float64).T
        ids = np.arange(lo, hi, dtype=np.int64)
        for j in range(m):
            cid, csc = topk_total_order(S[j], ids, k)
            best_ids[j], best_sc[j] = topk_total_order(np.concatenate([best_sc[j], csc]),
                                                       np.concatenate([best_ids[j], cid]), k)
    return np.stack(best_ids), np.stack(best_sc)


def recall_at_k(ids, gt, K: int = 10) -> float:
    """K-recall@k = |S cap G_t| / K, averaged over queries."""
    ids = np.asarray(ids)
    gt = np.asarray(gt)
    tot = 0.0
    for j in range(ids.shape[0]):
        tot += len(set(ids[j].tolist()) & set(gt[j, :K].tolist())) / K
    return tot / ids.shape[0]


def search(Q, X, A_stack, B_stack, assign, R: int, k: int, store: str | None = None,
           X_low=None):
    """Whole hot path (Alg. 1 with Eq.(15)): project, exhaustive reduced top-R, re-rank, top-k.
    `store` = storage dtype for x_low and q' ("emulated" mode) or None ("pure" fp64 mode)."""
    Qp = project(Q, A_stack, store)
    if X_low is None:
        X_low = encode(X, B_stack, assign, store)
    cand, cand_sc = reduced_search(Qp, X_low, assign, R)
    ids, sc = rerank_topk(Q, X, cand, k)
    return {"ids": ids, "scores": sc, "cand": cand, "cand_scores": cand_sc, "Qp": Qp, "X_low": X_low}


# ----------------------------------------------------------------------------------
# Flexible target dimensionality and streaming (Sections 3.1-3.2)
# ----------------------------------------------------------------------------------
def flexible_fit(Q_learn, X_learn) -> dict:
    """Sec. 3.1: P' = all D left singular vectors of W X sorted by decreasing singular
    value (Alg. 2 with d = D), A' = P'W^+, B' = P'W; x' = B'x is stored and the first d rows of A'
    and coordinates of x' give the d-dimensional reduction."""
    X = np.asarray(X_learn, dtype=np.float64)
    return sphering_fit(Q_learn, X, X.shape[1])


def eig_fit_from_stats(K_Q, m_q: int, K_X) -> dict:
    """Sec. 3.2: the two SVDs of Alg. 2 replaced by eigendecompositions:
    W = (K_Q / m_q)^{1/2} from eig(K_Q) (the SVD of Q gives W = U S U^T with S^2 = eig(Q Q^T); the
    1/sqrt(m) scale as in sphering_fit), P' = eigenvectors of W K_X W by decreasing eigenvalue
    (the left singular vectors of W X), sign-canonical rows; A' = P'W^+, B' = P'W (all D rows)."""
    lam, U = np.linalg.eigh(np.asarray(K_Q, dtype=np.float64) / float(m_q))
    sq = np.sqrt(np.maximum(lam, 0.0))
    W = (U * sq[None, :]) @ U.T
    cut = PINV_EPS * (sq.max() if sq.size else 0.0)
    sinv = np.where(sq > cut, 1.0 / np.where(sq > cut, sq, 1.0), 0.0)
    Wp = (U * sinv[None, :]) @ U.T
    M = W @ np.asarray(K_X, dtype=np.float64) @ W
    mu, V = np.linalg.eigh(0.5 * (M + M.T))
    order = np.argsort(mu)[::-1]
    P = _sign_canonical_rows(V[:, order].T.copy())
    return {"W": W, "Wp": Wp, "P": P, "A": P @ Wp, "B": P @ W, "eig": mu[order]}


class StreamingIndex:
    """Sec. 3.2, literally: the database X_t changes by inserts and removals of vectors
    with unique ids; K_X = sum_{x in X_t} x x^T and K_Q = sum q q^T are updated by adding or
    subtracting outer products; the stored vectors are x' = P'_{t'} W_{t'} x;
    a refresh recomputes W, P' by the eig route and applies
    P'_{t'+1} W_{t'+1} (P'_{t'} W_{t'})^{-1} to every stored x'; new vectors are
    stored as P'_{t'+1} W_{t'+1} x.  fp64; the raw vectors are kept here only to define
    K_X updates and to check the stored x' (the oracle is not memory-constrained)."""

    def __init__(self, D: int, A_prime, B_prime):
        self.D = D
        self.A = np.asarray(A_prime, dtype=np.float64)
        self.B = np.asarray(B_prime, dtype=np.float64)
        self.x = {}
        self.xp = {}
        self.K_X = np.zeros((D, D))
        self.K_Q = np.zeros((D, D))
        self.m_q = 0

    def insert(self, ids, X):
        for i, v in zip(np.asarray(ids).tolist(), np.asarray(X, dtype=np.float64)):
            assert i not in self.x
            self.x[i] = v
            self.xp[i] = self.B @ v
            self.K_X += np.outer(v, v)

    def remove(self, ids):
        for i in np.asarray(ids).tolist():
            v = self.x.pop(i)
            self.xp.pop(i)
            self.K_X -= np.outer(v, v)

    def observe(self, Q):
        Q = np.asarray(Q, dtype=np.float64)
        self.K_Q += Q.T @ Q
        self.m_q += Q.shape[0]

    def refresh(self):
        f = eig_fit_from_stats(self.K_Q, self.m_q, self.K_X)
        T = f["B"] @ np.linalg.inv(self.B)          # P'_{t'+1} W_{t'+1} (P'_{t'} W_{t'})^{-1}
        for i in self.xp:
            self.xp[i] = T @ self.xp[i]
        self.A, self.B = f["A"], f["B"]
        return f

    def current(self):
        ids = np.array(sorted(self.x), dtype=np.int64)
        return ids, np.stack([self.x[i] for i in ids]), np.stack([self.xp[i] for i in ids])


# ----------------------------------------------------------------------------------
# 8-bit reduced vectors (scalar quantisation of B x; reading R21)
# ----------------------------------------------------------------------------------
def quantize_db_i8(X_low, assign, C: int):
    """Per cluster c and coordinate e: delta_{c,e} = max_{i: c_i = c} |x_{i,e}| / 127 and
    code_{i,e} = RNE(x_{i,e} / delta_{c_i,e}) clipped to [-127, 127] (a zero column: delta = 1).
    x is the fp32 value of the reduced vector (the fp64 product rounded once to fp32); every
    operation is an fp32 operation with RNE (the quantiser's decisions are taken in fp32 on both
    sides, R21).  Returns (codes int8 [n, d], delta fp32 [C, d])."""
    x = np.asarray(X_low, dtype=np.float64).astype(np.float32)
    a = np.zeros(x.shape[0], dtype=np.int64) if assign is None else np.asarray(assign, dtype=np.int64)
    delta = np.ones((C, x.shape[1]), dtype=np.float32)
    for c in range(C):
        rows = x[a == c]
        if rows.shape[0]:
            amax = np.abs(rows).max(axis=0)
            delta[c] = np.where(amax > 0, amax / np.float32(127.0), np.float32(1.0))
    codes = np.clip(np.rint(x / delta[a]), -127, 127).astype(np.int8)
    return codes, delta


def quantize_queries_i8(Qp, delta):
    """Query side of the int8 scan: per query j and view c, q~ = q'_{j,c} * delta_c (fp32 product),
    s_{j,c} = max_e |q~_e| / 127 and codes = RNE(q~ / s_{j,c}) clipped to [-127, 127] (an all-zero
    view: s = 1).  Then s_{j,c} * <codes_{j,c}, x codes_i> = sum_e (q'_e delta_e)(x_e / delta_e)
    approximates <q'_{j,c}, x_i>.  Qp [m, C, d] (fp64, rounded to fp32 here).
    Returns (codes int8 [m, C, d], s fp32 [m, C])."""
    q = np.asarray(Qp, dtype=np.float64).astype(np.float32)
    qt = q * np.asarray(delta, dtype=np.float32)[None]
    amax = np.abs(qt).max(axis=2)
    s = np.where(amax > 0, amax / np.float32(127.0), np.float32(1.0)).astype(np.float32)
    codes = np.clip(np.rint(qt / s[:, :, None]), -127, 127).astype(np.int8)
    return codes, s


def search_i8(Q, X, A_stack, B_stack, assign, R: int, k: int, C: int | None = None):
    """The hot path with 8-bit reduced vectors: the reduced score of (q_j, x_i) is the fp32 value
    fl32(s_{j,c_i} * <q codes_{j,c_i}, x codes_i>) (an exact integer dot product scaled once),
    exhaustive top-R on it (Alg. 1 l.2), fp64 re-rank on the canonical vectors and top-k (l.3)."""
    A = np.asarray(A_stack, dtype=np.float64)
    C = C or (1 if A.ndim == 2 else A.shape[0])
    Qp = project(Q, A_stack)                                   # [m, C, d] fp64
    X_low = encode(X, B_stack, assign)                         # fp64
    xc, delta = quantize_db_i8(X_low, assign, C)
    qc, s = quantize_queries_i8(Qp, delta)
    Qeff = s[:, :, None].astype(np.float64) * qc.astype(np.float64)   # exact: s * code
    cand, cand_sc = reduced_search(Qeff, xc.astype(np.float64), assign, R, score_fp32=True)
    ids, sc = rerank_topk(Q, X, cand, k)
    return {"ids": ids, "scores": sc, "cand": cand, "cand_scores": cand_sc, "q_codes": qc, "q_scales": s,
            "x_codes": xc, "delta": delta, "Qeff": Qeff}


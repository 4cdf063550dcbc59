"""Index-build fit glue (off the search path): §3.2 statistics route to Alg. 2 / Alg. 5.

The GPU computes the D x D second moments (lv_fit_stats, K7); the host does the two
D x D eigendecompositions that replace Alg. 2's SVDs:
  W   = (K_Q / m_learn)^{1/2}              (eig of K_Q; P:228-231 with the 1/sqrt(m) scale, R2)
  P_c = top-d eigenvectors of W K_X[c] W    (per cluster for GleanVec)
  A_c = P_c W^+,  B_c = P_c W               (pseudoinverse per P:194)
GleanVec's spherical k-means (App. A) runs every pass over the rows on the GPU:
row normalisation (lv_normalize_rows), E-step tags and k-means++ similarities
(lv_kmeans_assign), M-step sums (lv_kmeans_centre_sums).  The host only draws the k-means++
seeds from the D^2 weights and normalises the C centre sums.
"""
from __future__ import annotations

import numpy as np
import torch

from . import lv

PINV_EPS = 1e-6


def sphering_from_KQ(KQ: np.ndarray, m_learn: int):
    lam, U = np.linalg.eigh(KQ / float(m_learn))
    s = np.sqrt(np.maximum(lam, 0.0))
    W = (U * s) @ U.T
    cut = PINV_EPS * s.max()
    sinv = np.where(s > cut, 1.0 / np.where(s > cut, s, 1.0), 0.0)
    Wp = (U * sinv) @ U.T
    return W, Wp


def _sign_canonical(P: np.ndarray) -> np.ndarray:
    idx = np.argmax(np.abs(P), axis=1)
    sg = np.sign(P[np.arange(P.shape[0]), idx])
    sg[sg == 0] = 1.0
    return P * sg[:, None]


def fit_from_stats(KQ: np.ndarray, KX: np.ndarray, m_learn: int, d: int) -> dict:
    """A_c, B_c (fp64, [C, d, D]) from the statistics; also returns W and eigengaps."""
    W, Wp = sphering_from_KQ(KQ, m_learn)
    C, D, _ = KX.shape
    A = np.empty((C, d, D))
    B = np.empty((C, d, D))
    gaps = []
    for c in range(C):
        M = W @ KX[c] @ W
        lam, V = np.linalg.eigh(0.5 * (M + M.T))
        order = np.argsort(lam)[::-1]
        lam, V = lam[order], V[:, order]
        P = _sign_canonical(V[:, :d].T)
        A[c] = P @ Wp
        B[c] = P @ W
        gaps.append(float(lam[d - 1] / lam[d] - 1.0) if d < D and lam[d] > 0 else float("inf"))
    return {"A": A, "B": B, "W": W, "Wp": Wp, "gaps": gaps}


def flexible_from_stats(KQ: np.ndarray, KX: np.ndarray, m_learn: int) -> dict:
    """§3.1-3.2: A' = P'W^+, B' = P'W with all D eigenvectors P' of W K_X W by decreasing
    eigenvalue (the stored x' = B'x admits any prefix d, and <A'q, x'> = <q, x>, Eq.(12)); used for
    lv_index_create_flex and for every streaming refresh (lv_stream_stats -> lv_stream_reproject)."""
    D = KQ.shape[0]
    f = fit_from_stats(KQ, np.asarray(KX).reshape(1, D, D), m_learn, D)
    return {"A": f["A"][0], "B": f["B"][0], "W": f["W"], "Wp": f["Wp"]}


def stream_refresh(index) -> dict:
    """One refresh of the streaming index: statistics -> eig route -> re-projection of
    every stored x' on the GPU."""
    KQ, KX, m_q, _ = lv.lv_stream_stats(index)
    f = flexible_from_stats(KQ, KX, m_q)
    lv.lv_stream_reproject(index, f["A"], f["B"])
    return f


def leanvec_sphering_fit(Q_learn: torch.Tensor, X_learn: torch.Tensor, d: int) -> dict:
    """Alg. 2 through the statistics route: lv_fit_stats on the GPU + host eig."""
    KQ, KX = lv.lv_fit_stats(Q_learn, X_learn, None, 1)
    out = fit_from_stats(KQ, KX, Q_learn.shape[0], d)
    out["KQ"], out["KX"] = KQ, KX
    return out


def gleanvec_fit(Q_learn: torch.Tensor, X_learn: torch.Tensor, C: int, d: int, draws: np.ndarray,
                 max_iter: int = 50) -> dict:
    """Alg. 5: normalise, spherical k-means, tags of the learning rows
    with the final centres, per-cluster Alg. 2 with one shared W via the statistics."""
    Xn = lv.lv_normalize_rows(X_learn)
    if C == 1:
        sums, _ = lv.lv_kmeans_centre_sums(Xn, torch.zeros(Xn.shape[0], dtype=torch.int32, device=Xn.device), 1)
        centres = sums / np.linalg.norm(sums[0])
    else:
        centres, _ = spherical_kmeans(Xn, C, draws, max_iter)
    assign, _ = lv.lv_kmeans_assign(Xn, torch.as_tensor(centres, dtype=torch.float32, device=Xn.device))
    KQ, KX = lv.lv_fit_stats(Q_learn, X_learn, assign, C)
    out = fit_from_stats(KQ, KX, Q_learn.shape[0], d)
    out.update({"centres": centres, "assign_learn": assign, "KQ": KQ, "KX": KX})
    return out


def spherical_kmeans(Xn: torch.Tensor, C: int, draws: np.ndarray, max_iter: int = 50):
    """App. A on unit rows Xn (CUDA fp32), every pass over the rows on the GPU:
    k-means++ seeding with D^2(x) = 2 - 2 max_c <x, mu_c> (lv_kmeans_assign keeps the
    running maximum; the host draws the next seed from the D^2 weights by inverse CDF with the
    shared uniform draws), then EM: E-step = Eq.(13) tags (lv_kmeans_assign), M-step =
    per-cluster sums (lv_kmeans_centre_sums) normalised on the host (C x D).  Stops when the tags do
    not change or after max_iter passes; an empty cluster takes the row least similar to its own
    centre (R14).  Returns (centres fp64 [C, D], last tags)."""
    n, D = Xn.shape
    dev = Xn.device
    mu = np.empty((C, D))
    first = min(int(draws[0] * n), n - 1)
    mu[0] = Xn[first].double().cpu().numpy()
    _, best = lv.lv_kmeans_assign(Xn, Xn[first:first + 1], assign=False)
    for j in range(1, C):
        w = np.maximum(2.0 - 2.0 * best.double().cpu().numpy(), 0.0)
        cdf = np.cumsum(w)
        if cdf[-1] <= 0:
            pick = min(int(draws[j] * n), n - 1)
        else:
            pick = min(int(np.searchsorted(cdf, draws[j] * cdf[-1], side="right")), n - 1)
        mu[j] = Xn[pick].double().cpu().numpy()
        lv.lv_kmeans_assign(Xn, Xn[pick:pick + 1], assign=False, best=best, accumulate=True)
    assign = None
    for _ in range(max_iter):
        new, best = lv.lv_kmeans_assign(Xn, torch.as_tensor(mu, dtype=torch.float32, device=dev))
        if assign is not None and torch.equal(new, assign):
            break
        assign = new
        sums, counts = lv.lv_kmeans_centre_sums(Xn, assign, C)
        far = None
        for c in range(C):
            if counts[c] == 0:
                if far is None:
                    far = int(np.argmin(best.cpu().numpy()))   # lowest index among the minima
                mu[c] = Xn[far].double().cpu().numpy()
            else:
                mu[c] = sums[c] / np.linalg.norm(sums[c])
    return mu, assign

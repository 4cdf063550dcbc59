"""Index-build fit glue (off the search path): §3.2 statistics route to Alg. 2 / Alg. 5.

The GPU computes the D x D second moments (lv_fit_stats, K7); the host does the two
D x D eigendecompositions that replace Alg. 2's SVDs:
  W   = (K_Q / m_learn)^{1/2}              (eig of K_Q; P:228-231 with the 1/sqrt(m) scale, R2)
  P_c = top-d eigenvectors of W K_X[c] W    (per cluster for GleanVec)
  A_c = P_c W^+,  B_c = P_c W               (pseudoinverse per P:194)
GleanVec's spherical k-means (App. A) runs its E-step (Eq.(13) tags) and
k-means++ similarities on the GPU (lv_assign_tags); the M-step centre sums use the same
GPU statistics path.  The host only samples k-means++ seeds and normalises C centres.
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


def leanvec_sphering_fit(Q_learn: torch.Tensor, X_learn: torch.Tensor, d: int) -> dict:
    """Alg. 2 through the statistics route: lv_fit_stats on the GPU + host eig."""
    KQ, KX = lv.lv_fit_stats(Q_learn, X_learn, None, 1)
    out = fit_from_stats(KQ, KX, Q_learn.shape[0], d)
    out["KQ"], out["KX"] = KQ, KX
    return out


def gleanvec_fit(Q_learn: torch.Tensor, X_learn: torch.Tensor, C: int, d: int, draws: np.ndarray,
                 max_iter: int = 50) -> dict:
    """Alg. 5: normalise, spherical k-means, per-cluster Alg. 2 with a shared W."""
    Xn = X_learn.float()
    Xn = Xn / torch.linalg.vector_norm(Xn, dim=1, keepdim=True)
    centres, assign = spherical_kmeans(Xn, C, draws, max_iter)
    KQ, KX = lv.lv_fit_stats(Q_learn, X_learn, assign, C)
    out = fit_from_stats(KQ, KX, Q_learn.shape[0], d)
    out.update({"centres": centres, "assign_learn": assign, "KQ": KQ, "KX": KX})
    return out


def _centre_sums(Xn: torch.Tensor, assign: torch.Tensor, C: int) -> np.ndarray:
    """M-step sums sum_{c_i = c} x~_i via the statistics kernel: with rows [x~; 1]
    the per-cluster second moment holds sum x~ in its last column."""
    n, D = Xn.shape
    aug = torch.zeros((n, D + 4), dtype=torch.float32, device=Xn.device)   # keep rows 16-byte aligned
    aug[:, :D] = Xn
    aug[:, D] = 1.0
    ones = torch.zeros((1, D + 4), dtype=torch.float32, device=Xn.device)
    ones[0, 0] = 1.0
    _, KX = lv.lv_fit_stats(ones, aug, assign, C)
    # K_X[c][:D, D] = sum_{c_i=c} x~_i * 1
    return KX[:, :D, D]


def spherical_kmeans(Xn: torch.Tensor, C: int, draws: np.ndarray, max_iter: int = 50):
    """App. A on unit rows Xn (CUDA fp32).  k-means++ seeding with D^2 = 2 - 2 max<x,mu>
    (the per-row max similarity is one lv_assign_tags-style pass per new centre), then EM:
    E-step = Eq.(13) tags on the GPU (lv_assign_tags), M-step = normalised per-cluster sums."""
    n, D = Xn.shape
    mu = np.empty((C, D))
    first = min(int(draws[0] * n), n - 1)
    mu[0] = Xn[first].double().cpu().numpy()
    best = (Xn @ Xn[first]).double().cpu().numpy()   # TODO(lv): move to a kernel
    for j in range(1, C):
        w = np.maximum(2.0 - 2.0 * best, 0.0)
        cdf = np.cumsum(w)
        if cdf[-1] <= 0:
            pick = min(int(draws[j] * n), n - 1)
        else:
            pick = min(int(np.searchsorted(cdf, draws[j] * cdf[-1], side="right")), n - 1)
        mu[j] = Xn[pick].double().cpu().numpy()
        best = np.maximum(best, (Xn @ Xn[pick]).double().cpu().numpy())
    assign = None
    for _ in range(max_iter):
        new = lv.lv_assign_tags(Xn, torch.as_tensor(mu, dtype=torch.float32, device=Xn.device))
        if assign is not None and torch.equal(new, assign):
            break
        assign = new
        sums = _centre_sums(Xn, assign, C)
        for c in range(C):
            nrm = np.linalg.norm(sums[c])
            if nrm > 0:
                mu[c] = sums[c] / nrm
    return mu, assign

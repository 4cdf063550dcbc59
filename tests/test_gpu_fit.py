"""Fit parity (SURVEY §8(c) "route equivalence / fit parity") and GPU k-means parity
(App. A): the PRODUCT's index build (fit.py: lv_fit_stats + host eig, GPU spherical
k-means through lv_normalize_rows / lv_kmeans_assign / lv_kmeans_centre_sums) against the
oracle's SVD-route fit (Alg. 2 / Alg. 5 literally) on the same learning sets.

Gates:
  K_Q, K_X       ||K_lib - K_ref||_F / ||K_ref||_F <= 1e-6
  M_c = A_c^T B_c ||M_lib - M_ref||_F / ||M_ref||_F <= 1e-5 max(1, 1e-2 / gap_c), gap_c = lambda_d /
                 lambda_{d+1} - 1 of W K_{X_c} W (sign-, scale- and in-subspace-rotation invariant)
  k-means        identical tags except rows whose two best centre similarities (oracle fp64) are
                 within 1e-5; centres within 1e-5 where the memberships agree
"""
import numpy as np
import pytest
import torch

import lvgen
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lv():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_22347_b200 import lv as L
    return L


@pytest.fixture(scope="module")
def fit():
    from paper_2410_22347_b200 import fit as F
    return F


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _gap(sig, d):
    lam = np.asarray(sig, dtype=np.float64) ** 2
    return lam[d - 1] / lam[d] - 1.0 if d < lam.size and lam[d] > 0 else np.inf


def _learn_sets(cfg_id, n, m_learn, n_learn, family=None):
    c = lvgen.get_config(cfg_id, n=n)
    X = lvgen.database(c)
    Ql = lvgen.queries(c, "learn", family=family, m=m_learn)
    Xl = X[lvgen.learn_rows(c.replace(n_learn=n_learn))]
    return c, Ql, Xl


@pytest.mark.parametrize("cfg_id,family", [(2, None), (4, "id"), (4, "ood")])
def test_sphering_fit_parity(lv, fit, cfg_id, family):
    """LeanVec-Sphering: stats + eig route (product) vs two SVDs (oracle, Alg. 2), 10^5 learning
    queries and a 10^5-row learning sample of the config's database distribution."""
    c, Ql, Xl = _learn_sets(cfg_id, 400_000, 100_000, 100_000, family)
    got = fit.leanvec_sphering_fit(torch.from_numpy(Ql).cuda(), torch.from_numpy(Xl).cuda(), c.d)
    ref = O.sphering_fit(Ql, Xl, c.d)
    Q64, X64 = Ql.astype(np.float64), Xl.astype(np.float64)
    assert _rel(got["KQ"], Q64.T @ Q64) <= 1e-6
    assert _rel(got["KX"][0], X64.T @ X64) <= 1e-6
    M_lib = got["A"][0].T @ got["B"][0]
    M_ref = ref["A"].T @ ref["B"]
    gap = _gap(ref["sigma"], c.d)
    assert _rel(M_lib, M_ref) <= 1e-5 * max(1.0, 1e-2 / gap), (_rel(M_lib, M_ref), gap)
    # the product's matrices satisfy the paper's conditions themselves: A B^T = I_d
    assert np.abs(got["A"][0] @ got["B"][0].T - np.eye(c.d)).max() < 1e-9


def test_kmeans_parity(lv, fit):
    """GPU spherical k-means (k-means++ seeding with shared draws, EM) vs the oracle's, on the
    normalised 10^5-row learning sample of the config-3 mixture (C = 16)."""
    c, Ql, Xl = _learn_sets(3, 400_000, 1000, 100_000)
    X64 = Xl.astype(np.float64)
    Xn64 = X64 / np.linalg.norm(X64, axis=1, keepdims=True)
    draws = lvgen.kmeanspp_draws(c)
    mu_ref, a_ref, hist = O.spherical_kmeans(Xn64, c.C, draws, max_iter=50)
    Xn = lv.lv_normalize_rows(torch.from_numpy(Xl).cuda())
    assert np.abs(Xn.cpu().numpy() - Xn64).max() < 1e-6
    mu_gpu, a_gpu = fit.spherical_kmeans(Xn, c.C, draws, max_iter=50)
    a_gpu = a_gpu.cpu().numpy()
    S = Xn64 @ mu_ref.T
    top2 = np.sort(S, axis=1)[:, -2:]
    diff = np.nonzero(a_gpu != a_ref)[0]
    assert np.all(top2[diff, 1] - top2[diff, 0] < 1e-5), diff[:10]
    assert diff.size <= max(5, Xn64.shape[0] // 10_000)
    assert np.abs(mu_gpu - mu_ref).max() < 1e-4 if diff.size else np.abs(mu_gpu - mu_ref).max() < 1e-5


def test_kmeans_kernels_match_definitions(lv):
    """lv_kmeans_assign (tags, best similarity, running max) and lv_kmeans_centre_sums against the
    plain definitions (E-step argmax with lowest-index ties, M-step sums and counts), incl. an
    empty cluster, fp16 rows and C = 37 (not a power of two)."""
    rng = np.random.default_rng(5)
    n, D, C = 20_011, 200, 37
    X = rng.standard_normal((n, D)).astype(np.float32)
    mu = rng.standard_normal((C, D))
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    mu32 = mu.astype(np.float32)
    for xd in (np.float32, np.float16):
        Xc = X.astype(xd)
        Xt = torch.from_numpy(Xc).cuda()
        a, best = lv.lv_kmeans_assign(Xt, torch.from_numpy(mu32).cuda())
        S = Xc.astype(np.float64) @ mu32.astype(np.float64).T
        ref = np.argmax(S, axis=1)
        a = a.cpu().numpy()
        for i in np.nonzero(a != ref)[0]:
            assert S[i, ref[i]] - S[i, a[i]] < 1e-4
        assert np.abs(best.cpu().numpy() - S.max(axis=1)).max() < 1e-4
        # running maximum over two calls == one call over both centres
        _, b2 = lv.lv_kmeans_assign(Xt, torch.from_numpy(mu32[:5]).cuda(), assign=False)
        lv.lv_kmeans_assign(Xt, torch.from_numpy(mu32[5:]).cuda(), assign=False, best=b2, accumulate=True)
        assert torch.equal(b2, best)
        asg = rng.integers(0, C, n).astype(np.int32)
        asg[asg == 3] = 4                                   # cluster 3 empty
        sums, counts = lv.lv_kmeans_centre_sums(Xt, torch.from_numpy(asg).cuda(), C)
        for cc in range(C):
            rows = Xc[asg == cc].astype(np.float64)
            assert counts[cc] == rows.shape[0]
            ref_s = rows.sum(axis=0) if rows.shape[0] else np.zeros(D)
            assert np.abs(sums[cc] - ref_s).max() <= 1e-5 * max(1.0, np.abs(rows).sum(axis=0).max() if rows.size else 1)


def test_gleanvec_fit_parity(lv, fit):
    """GleanVec (Alg. 5): the product's whole build (GPU k-means + stats + eig) vs the oracle's,
    config-3 shape (C = 16, d = 96, 10^5 learning rows and queries).  Per cluster, M_c at the
    gap-aware gate; tags as in test_kmeans_parity."""
    c, Ql, Xl = _learn_sets(3, 400_000, 100_000, 100_000)
    draws = lvgen.kmeanspp_draws(c)
    got = fit.gleanvec_fit(torch.from_numpy(Ql).cuda(), torch.from_numpy(Xl).cuda(), c.C, c.d, draws)
    ref = O.gleanvec_fit(Ql, Xl, c.C, c.d, draws)
    a_got = got["assign_learn"].cpu().numpy()
    agree = a_got == ref["assign_learn"]
    assert agree.mean() >= 0.9999, agree.mean()
    if agree.all():
        for cc in range(c.C):
            M_lib = got["A"][cc].T @ got["B"][cc]
            M_ref = ref["A"][cc].T @ ref["B"][cc]
            gap = _gap(ref["sigma"][cc], c.d)
            assert _rel(M_lib, M_ref) <= 1e-5 * max(1.0, 1e-2 / gap), (cc, _rel(M_lib, M_ref), gap)
    # the stats route itself on the ORACLE's tags (independent of k-means near-ties)
    KQ, KX = lv.lv_fit_stats(torch.from_numpy(Ql).cuda(), torch.from_numpy(Xl).cuda(),
                             torch.from_numpy(ref["assign_learn"]).cuda(), c.C)
    f2 = fit.fit_from_stats(KQ, KX, Ql.shape[0], c.d)
    for cc in range(c.C):
        M_lib = f2["A"][cc].T @ f2["B"][cc]
        M_ref = ref["A"][cc].T @ ref["B"][cc]
        gap = _gap(ref["sigma"][cc], c.d)
        assert _rel(M_lib, M_ref) <= 1e-5 * max(1.0, 1e-2 / gap), (cc, _rel(M_lib, M_ref), gap)

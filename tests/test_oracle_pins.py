"""Pins of the fp64 oracle against what the paper and the mathematics fix (CPU only).

Each test names the passage it pins.  None of them retypes the oracle's formula:
they check identities (Eq.(7)), closed forms (Eckart-Young optimum of Problem (4)),
special cases reducing to other library routines (eigh vs svd, full sort),
hand-worked examples (tests/golden/spec_examples.json) and brute force on tiny inputs.
"""
import json
import os
import struct

import numpy as np
import pytest

import oracle as O
import lvgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rng(s=0):
    return np.random.default_rng(s)


def _ood_pair(rng, m=400, n=600, D=12):
    """Small anisotropic OOD pair: X and Q with different principal axes."""
    lam = np.arange(1, D + 1) ** -1.0
    MX = np.linalg.qr(rng.standard_normal((D, D)))[0]
    MQ = np.linalg.qr(rng.standard_normal((D, D)))[0]
    X = (rng.standard_normal((n, D)) * np.sqrt(lam)) @ MX.T
    Q = (rng.standard_normal((m, D)) * np.sqrt(lam)) @ MQ.T
    return Q, X


# ---------------------------------------------------------------- sphering matrix
def test_sphering_diag_example():
    g = GOLD["sphering_diag"]
    W, Wp = O.sphering_matrix(np.array(g["Q_cols"], float).T)
    assert np.allclose(W, g["W"], atol=1e-14)
    assert np.allclose(Wp, g["W_pinv"], atol=1e-14)


def test_sphering_rank1_pseudoinverse():
    g = GOLD["sphering_rank1"]
    W, Wp = O.sphering_matrix(np.array(g["Q_cols"], float).T)
    assert np.allclose(W, g["W"], atol=1e-12)
    assert np.allclose(Wp, g["W_pinv"], atol=1e-12)


def test_eq7_QQt_equals_WtW_and_whitening():
    """Eq.(7): QQ^T = W^T W; W symmetric PSD; W^+ Q Q^T W^+ = I ("spherical")."""
    rng = _rng(1)
    Qc = rng.standard_normal((16, 100)) * np.linspace(0.2, 3, 16)[:, None]
    W, Wp = O.sphering_matrix(Qc)
    K = Qc @ Qc.T
    assert np.linalg.norm(W.T @ W - K) / np.linalg.norm(K) < 1e-12
    assert np.allclose(W, W.T, atol=1e-12)
    assert np.linalg.eigvalsh(W).min() > -1e-10
    assert np.allclose(Wp @ K @ Wp, np.eye(16), atol=1e-10)


# ---------------------------------------------------------------- LeanVec-Sphering fit
def test_slice_example():
    g = GOLD["slice_example"]
    Wpair = O.sphering_matrix(np.array(g["Q_cols"], float).T)
    f = O.sphering_fit(np.zeros((1, 2)), np.array(g["X_cols"], float), g["d"], Wpair=Wpair)
    assert np.allclose(f["P"], g["P"], atol=1e-14)
    assert np.allclose(f["A"], g["A"], atol=1e-14)
    assert np.allclose(f["B"], g["B"], atol=1e-14)


def test_dominant_axis_example():
    g = GOLD["dominant_axis"]
    Wpair = O.sphering_matrix(np.array(g["Q_cols"], float).T)
    f = O.sphering_fit(np.zeros((1, 2)), np.array(g["X_cols"], float), g["d"], Wpair=Wpair)
    assert np.allclose(f["P"], g["P"], atol=1e-14)


def test_fig1_query_aware_direction():
    """Fig. 1 caption: X dominant along e1, Q along e2 -> the retained direction
    of A serves e2 (the query-aware choice), unlike the SVD baseline (e1)."""
    rng = _rng(2)
    X = np.c_[3.0 * rng.standard_normal(500), 0.7 * rng.standard_normal(500)]
    Q = np.c_[0.05 * rng.standard_normal(500), 1.0 * rng.standard_normal(500)]
    f = O.sphering_fit(Q, X, 1)
    a = f["A"][0] / np.linalg.norm(f["A"][0])
    assert abs(a[1]) > abs(a[0])
    b = O.svd_baseline_fit(X, 1)["A"][0]
    assert abs(b[0]) > abs(b[1])
    assert O.leanvec_loss(f["A"], f["B"], Q, X) < O.leanvec_loss(b[None], b[None], Q, X)


def test_fit_orthogonality_and_AB_identity():
    """P in St(D,d); A B^T = P W^+ W P^T = I_d."""
    Q, X = _ood_pair(_rng(3))
    f = O.sphering_fit(Q, X, 5)
    assert np.allclose(f["P"] @ f["P"].T, np.eye(5), atol=1e-12)
    assert np.allclose(f["A"] @ f["B"].T, np.eye(5), atol=1e-12)


def test_P_rows_are_top_eigvecs_of_WKW():
    """the SVD of W X equals the eigendecomposition of W K_X W (eigh route)."""
    Q, X = _ood_pair(_rng(4))
    d = 4
    f = O.sphering_fit(Q, X, d)
    W = f["W"]
    KX = X.T @ X
    lam, V = np.linalg.eigh(W @ KX @ W)
    Vd = V[:, ::-1][:, :d]
    # same subspace (projectors equal)
    assert np.allclose(f["P"].T @ f["P"], Vd @ Vd.T, atol=1e-9)
    # W from eig of K_Q / m equals the SVD-route W
    KQ = Q.T @ Q / Q.shape[0]
    l2, V2 = np.linalg.eigh(KQ)
    W2 = (V2 * np.sqrt(np.maximum(l2, 0))) @ V2.T
    assert np.allclose(W, W2, atol=1e-12)


def test_d_equals_D_exactness():
    """Eq.(11)/(12) P:259-265 (north star): with d=D reduced scores equal <q,x> to 1e-9."""
    Q, X = _ood_pair(_rng(5))
    D = X.shape[1]
    f = O.sphering_fit(Q, X, D)
    assert np.allclose(f["A"].T @ f["B"], np.eye(D), atol=1e-10)
    q = Q[:7]
    s_red = O.reduced_scores(O.project(q, f["A"]), O.encode(X, f["B"]))
    s_ex = q @ X.T
    assert np.max(np.abs(s_red - s_ex)) <= 1e-9 * max(1.0, np.abs(s_ex).max())


def test_loss_trace_form_vs_naive_double_loop():
    """Problem (4) P:131-136: trace form == literal double sum (SPEC S:165 idea)."""
    rng = _rng(6)
    Q, X = _ood_pair(rng, m=20, n=25, D=6)
    f = O.sphering_fit(Q, X, 3)
    a = O.leanvec_loss(f["A"], f["B"], Q, X)
    b = O.leanvec_loss_naive(f["A"], f["B"], Q, X)
    assert abs(a - b) <= 1e-9 * b


def test_loss_closed_form_optimum_and_orderings():
    """Eckart-Young on Eq.(6): L_sphering(d) = m * sum_{j>d} lambda_j(W K_X W)
    (W from Q/sqrt(m)); it is the global optimum of Problem (4) over rank-d A^T B, hence
    <= the SVD baseline and <= random Stiefel pairs, non-increasing in d, 0 at d=D."""
    rng = _rng(7)
    Q, X = _ood_pair(rng)
    D = X.shape[1]
    m = Q.shape[0]
    losses = []
    for d in range(1, D + 1):
        f = O.sphering_fit(Q, X, d)
        L = O.leanvec_loss(f["A"], f["B"], Q, X)
        lam = np.sort(np.linalg.eigvalsh(f["W"] @ (X.T @ X) @ f["W"]))[::-1]
        closed = m * lam[d:].sum()
        assert abs(L - closed) <= 1e-9 * max(closed, 1e-9 * m * lam.sum())
        b = O.svd_baseline_fit(X, d)
        assert L <= O.leanvec_loss(b["A"], b["B"], Q, X) * (1 + 1e-12) + 1e-9
        for _ in range(3):
            A = np.linalg.qr(rng.standard_normal((D, d)))[0].T
            Bm = np.linalg.qr(rng.standard_normal((D, d)))[0].T
            assert L <= O.leanvec_loss(A, Bm, Q, X)
        losses.append(L)
    assert all(losses[i + 1] <= losses[i] * (1 + 1e-12) + 1e-9 for i in range(D - 1))
    assert losses[-1] <= 1e-9 * losses[0]


def test_flexible_d_prefix_is_the_smaller_fit():
    """§3.1: P' holds the singular vectors in decreasing order, so searching on the
    first d2 coordinates of x' = P'Wx and of P'W^-1 q IS the d2 reduction: its loss is the
    Eckart-Young optimum m * sum_{j>d2} lambda_j(W K_X W) (a closed form, not the oracle's fit
    route), and the prefix scores equal <A_d2 q, B_d2 x>."""
    Q, X = _ood_pair(_rng(11))
    m, D = Q.shape
    full = O.sphering_fit(Q, X, D)                       # P' = D x D (Eq. 10's storage)
    lam = np.sort(np.linalg.eigvalsh(full["W"] @ (X.T @ X) @ full["W"]))[::-1]
    q = Q[:9]
    for d2 in (2, 5, 9):
        A2, B2 = full["A"][:d2], full["B"][:d2]          # first d2 rows = first d2 coordinates
        L = O.leanvec_loss(A2, B2, Q, X)
        closed = m * lam[d2:].sum()
        assert abs(L - closed) <= 1e-9 * closed
        s_pre = O.reduced_scores(O.project(q, full["A"])[:, :, :d2], O.encode(X, full["B"])[:, :d2])
        s_d2 = O.reduced_scores(O.project(q, A2), O.encode(X, B2))
        assert np.allclose(s_pre, s_d2, rtol=0, atol=1e-12)


def test_flexible_fit_exact_rerank_eq12():
    """Eq.(12): with A' = P'W^+, B' = P'W (D x D), <A'q, x'> = <q, x> for any q and x,
    not only the learning sets (the 'undistorted similarities' claim); x' = B'x is invertible by
    A'^T (A'^T B' = I)."""
    rng = _rng(21)
    Q, X = _ood_pair(rng)
    f = O.flexible_fit(Q, X)
    q = rng.standard_normal((7, X.shape[1]))
    x = rng.standard_normal((11, X.shape[1]))
    assert np.allclose((q @ f["A"].T) @ (x @ f["B"].T).T, q @ x.T, rtol=0, atol=1e-9)
    assert np.allclose(f["A"].T @ f["B"], np.eye(X.shape[1]), atol=1e-10)


def test_eig_route_from_stats_equals_svd_route():
    """§3.2: eigendecompositions of K_Q and W K_X W give the same W and the same P' (up to
    the sign rule) as Alg. 2's two SVDs; checked on every prefix d with a spectral gap via
    M_d = A'_d^T B'_d (invariant to the sign and to rotations inside degenerate blocks)."""
    Q, X = _ood_pair(_rng(22))
    svd = O.flexible_fit(Q, X)
    eig = O.eig_fit_from_stats(Q.T @ Q, Q.shape[0], X.T @ X)
    assert np.allclose(eig["W"], svd["W"], atol=1e-12)
    lam = eig["eig"]
    for d in range(1, X.shape[1]):
        if lam[d - 1] / lam[d] - 1 > 1e-6:
            Ms = svd["A"][:d].T @ svd["B"][:d]
            Me = eig["A"][:d].T @ eig["B"][:d]
            assert np.abs(Ms - Me).max() < 1e-8 * max(1.0, np.abs(Ms).max())


def test_streaming_stats_reprojection_and_fresh_fit():
    """§3.2: after inserts, removals and new queries, (1) K_X equals sum x x^T over the
    CURRENT set and K_Q sum q q^T over every observed query (their definitions);
    (2) after a refresh, every stored x' = T x'_old equals P'_{t'+1} W_{t'+1} x of its raw vector
    (the undo/redo identity of P:302-307), and vectors inserted afterwards are stored the same way
    (P:308); (3) the refreshed A', B' equal a fresh Alg. 2 SVD fit on the current set with all
    observed queries (route equivalence), so the index equals a fresh fit + encode."""
    rng = _rng(23)
    D = 10
    Q0, X0 = _ood_pair(rng, m=300, n=400, D=D)
    Q1, X1 = _ood_pair(_rng(24), m=200, n=150, D=D)
    f0 = O.flexible_fit(Q0, X0)
    st = O.StreamingIndex(D, f0["A"], f0["B"])
    st.insert(np.arange(400), X0)
    st.observe(Q0)
    st.insert(np.arange(1000, 1150), X1)
    gone = rng.choice(np.concatenate([np.arange(400), np.arange(1000, 1150)]), 120, replace=False)
    st.remove(gone)
    st.observe(Q1)
    ids, X, Xp = st.current()
    assert ids.size == 550 - 120 and not set(gone.tolist()) & set(ids.tolist())
    Kx = X.T @ X
    assert np.abs(st.K_X - Kx).max() <= 1e-10 * np.abs(Kx).max()
    Qall = np.vstack([Q0, Q1])
    assert np.abs(st.K_Q - Qall.T @ Qall).max() <= 1e-10 * np.abs(Qall.T @ Qall).max()
    f1 = st.refresh()
    ids, X, Xp = st.current()
    assert np.allclose(Xp, X @ f1["B"].T, rtol=0, atol=1e-10)
    st.insert([5000], X1[:1] * 0.5)
    ids, X, Xp = st.current()
    assert np.allclose(Xp, X @ f1["B"].T, rtol=0, atol=1e-10)
    fresh = O.flexible_fit(Qall, X[ids != 5000])
    lam = f1["eig"]
    for d in (2, 4, 7):
        if lam[d - 1] / lam[d] - 1 > 1e-6:
            assert np.abs(fresh["A"][:d].T @ fresh["B"][:d] - f1["A"][:d].T @ f1["B"][:d]).max() < 1e-8


def test_i8_quantiser_bounds_and_exact_case():
    """R21 (scalar quantisation of B x): every code within [-127, 127], each column's
    extreme maps to +-127, |x - delta code| <= delta / 2 (round to nearest); the quantised score
    s <q_code, x_code> differs from <q', x> by at most the closed-form rounding bound
    sum_e (s/2 |x_code_e| + |q~_e| / 2); integer data with column maximum 127 and query maximum 127
    quantise exactly (delta = s = 1), so the int8 search equals the plain search."""
    rng = _rng(31)
    n, d, C = 500, 16, 3
    X = rng.standard_normal((n, d)) * np.linspace(3, 0.1, d)
    a = rng.integers(0, C, n)
    codes, delta = O.quantize_db_i8(X, a, C)
    x32 = X.astype(np.float32).astype(np.float64)
    assert codes.dtype == np.int8 and np.abs(codes.astype(int)).max() <= 127
    for c in range(C):
        assert (np.abs(codes[a == c].astype(int)).max(axis=0) == 127).all()
    rec = codes.astype(np.float64) * delta[a].astype(np.float64)
    assert (np.abs(x32 - rec) <= delta[a].astype(np.float64) / 2 * (1 + 1e-6)).all()
    Qp = rng.standard_normal((7, C, d))
    qc, s = O.quantize_queries_i8(Qp, delta)
    q32 = Qp.astype(np.float32).astype(np.float64)
    for j in range(7):
        for i in range(0, n, 37):
            c = a[i]
            approx = float(s[j, c]) * float(qc[j, c].astype(np.int64) @ codes[i].astype(np.int64))
            exact = float(q32[j, c] @ x32[i])
            qt = np.abs(q32[j, c] * delta[c])
            bound = float(np.sum(s[j, c] / 2 * np.abs(codes[i].astype(np.float64)) + qt / 2)) * (1 + 1e-5)
            assert abs(approx - exact) <= bound
    # exact special case: integer reduced vectors with column max 127 and integer queries with max 127
    Xi = rng.integers(-127, 128, (200, 8)).astype(np.float64)
    Xi[0] = 127
    Bi = np.eye(8)
    Qi = rng.integers(-127, 128, (5, 8)).astype(np.float64)
    Qi[:, 0] = 127
    r8 = O.search_i8(Qi, Xi, Bi, Bi, None, 30, 5)
    rp = O.search(Qi, Xi, Bi, Bi, None, 30, 5)
    assert np.array_equal(r8["delta"], np.ones((1, 8), np.float32)) and np.array_equal(r8["q_scales"], np.ones((5, 1)))
    assert np.array_equal(r8["cand"], rp["cand"]) and np.array_equal(r8["ids"], rp["ids"])


def test_scale_invariance_of_AtB():
    """Q -> cQ leaves A^T B unchanged."""
    Q, X = _ood_pair(_rng(8))
    f1 = O.sphering_fit(Q, X, 4)
    f2 = O.sphering_fit(3.7 * Q, X, 4)
    assert np.allclose(f1["A"].T @ f1["B"], f2["A"].T @ f2["B"], atol=1e-12)


# ---------------------------------------------------------------- GleanVec
def test_assign_tag_examples():
    g = GOLD["assign_tag"]
    assert O.assign_tags(np.array(g["x"], float), np.array(g["centres"], float)).tolist() == g["tags"]


def test_kmeans_properties():
    """App. A: objective non-decreasing under EM, ||mu_c|| = 1."""
    rng = _rng(9)
    X = rng.standard_normal((600, 8)) + 2.0 * np.eye(8)[rng.integers(0, 4, 600)]
    Xn = X / np.linalg.norm(X, axis=1, keepdims=True)
    mu, assign, hist = O.spherical_kmeans(Xn, 4, rng.random(4))
    assert np.allclose(np.linalg.norm(mu, axis=1), 1.0, atol=1e-12)
    assert all(hist[i + 1] >= hist[i] - 1e-9 for i in range(len(hist) - 1))
    assert set(np.unique(assign).tolist()) <= set(range(4))


def test_kmeans_C1_is_normalised_mean():
    rng = _rng(10)
    X = rng.standard_normal((200, 5)) + np.array([3, 0, 0, 0, 0])
    Xn = X / np.linalg.norm(X, axis=1, keepdims=True)
    mu, _, _ = O.spherical_kmeans(Xn, 1, np.array([0.3]))
    s = Xn.sum(0)
    assert np.allclose(mu[0], s / np.linalg.norm(s), atol=1e-12)


def test_kmeans_antipodal_clouds():
    """two antipodal clouds, C=2 -> centres within 0.05 rad of the cloud axes."""
    rng = _rng(11)
    a = np.array([1.0, 0.0])
    pts = np.r_[a + 0.05 * rng.standard_normal((50, 2)), -a + 0.05 * rng.standard_normal((50, 2))]
    Xn = pts / np.linalg.norm(pts, axis=1, keepdims=True)
    mu, _, _ = O.spherical_kmeans(Xn, 2, np.array([0.1, 0.5]))
    ang = sorted(np.degrees(np.arccos(np.clip(mu @ a, -1, 1))))
    assert ang[0] < np.degrees(0.05) and ang[1] > 180 - np.degrees(0.05)


def test_gleanvec_C1_reproduces_leanvec():
    """North star / S:255: GleanVec with one cluster == LeanVec-Sphering (A_1=A, B_1=B)."""
    Q, X = _ood_pair(_rng(12))
    g = O.gleanvec_fit(Q, X, 1, 4, np.array([0.5]))
    f = O.sphering_fit(Q, X, 4)
    assert np.allclose(g["A"][0], f["A"], atol=1e-12)
    assert np.allclose(g["B"][0], f["B"], atol=1e-12)


def test_gleanvec_per_cluster_loss_not_worse():
    """Derived: each cluster's pair is its own global rank-d optimum and the global pair is
    feasible for every cluster, so sum_c L_c <= L_global on X_learn."""
    rng = _rng(13)
    D = 10
    X = np.r_[(rng.standard_normal((300, D)) * np.r_[3, np.ones(D - 1) * 0.3]),
              (rng.standard_normal((300, D)) * np.r_[np.ones(D - 1) * 0.3, 3]) + 1.0]
    Q = rng.standard_normal((300, D))
    d = 2
    g = O.gleanvec_fit(Q, X, 2, d, np.array([0.2, 0.7]))
    f = O.sphering_fit(Q, X, d)
    a = g["assign_learn"]
    Lc = sum(O.leanvec_loss(g["A"][c], g["B"][c], Q, X[a == c]) for c in range(2))
    Lg = sum(O.leanvec_loss(f["A"], f["B"], Q, X[a == c]) for c in range(2))
    assert Lc <= Lg * (1 + 1e-12)
    for c in range(2):
        Pc = g["A"][c] @ g["W"]
        assert np.allclose(Pc @ Pc.T, np.eye(d), atol=1e-10)


# ---------------------------------------------------------------- storage rounding
def _bf16_rne_bits(x: float) -> float:
    """Textbook fp32 -> bf16 RNE via bit arithmetic (independent of ml_dtypes)."""
    u = struct.unpack("<I", struct.pack("<f", x))[0]
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return struct.unpack("<f", struct.pack("<I", u))[0]


def test_round_storage_bf16_fp16():
    vals = [1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -9, 0.1, 1e-3, 3.14159, -2.5e-5]
    r = O.round_storage(np.array(vals), "bf16")
    assert r[0] == 1.0 and r[1] == 1.0 + 2 ** -6      # ties to even
    for v, got in zip(vals, r):
        assert got == _bf16_rne_bits(np.float32(v))
    h = O.round_storage(np.array([1.0 + 2 ** -11, 1.0 + 3 * 2 ** -11, 65504.0]), "fp16")
    assert h[0] == 1.0 and h[1] == 1.0 + 2 ** -9 and h[2] == 65504.0


# ---------------------------------------------------------------- search
def test_brute_force_example():
    g = GOLD["brute_force_topk"]
    ids, _ = O.exact_topk(np.array([g["q"]], float), np.array(g["X"], float), g["k"])
    assert ids[0].tolist() == g["ids"]


def test_recall_examples():
    for c in GOLD["recall"]["cases"]:
        assert O.recall_at_k(np.array([c["S"]]), np.array([c["G"]]), 10) == pytest.approx(c["recall"])


def test_reduced_search_vs_full_sort_with_ties():
    """Exhaustive top-R equals the first R of a full stable sort by (-s, id), chunking
    and duplicate rows (exact ties) included (S:113, S:435 tie rule)."""
    rng = _rng(14)
    n, d, m = 700, 8, 9
    Xl = rng.standard_normal((n, d))
    Xl[100] = Xl[5]
    Xl[650] = Xl[5]          # exact ties
    Xl[300:310] = 0.0        # a block of equal (zero) scores
    Qp = rng.standard_normal((m, d))
    for R in (1, 37, n):
        ids, sc = O.reduced_search(Qp, Xl, None, R, chunk=128)
        S = Qp @ Xl.T
        for j in range(m):
            order = sorted(range(n), key=lambda i: (-S[j, i], i))[:R]
            assert ids[j].tolist() == order


def test_exact_topk_chunk_merge_vs_full_sort():
    """exact_topk (the recall ground truth) with chunk = 64 over 300 rows (5 chunks and a
    ragged tail) equals the first k of a full stable sort by (-<q, x>, id), exact ties included."""
    rng = _rng(17)
    n, D, m = 300, 6, 7
    X = rng.standard_normal((n, D))
    X[200] = X[3]
    X[290] = X[3]            # exact ties across chunks
    X[100:140] = 0.0         # equal (zero) scores spanning a chunk boundary
    Q = rng.standard_normal((m, D))
    S = Q @ X.T
    for k in (1, 10, 70, n):
        ids, sc = O.exact_topk(Q, X, k, chunk=64)
        for j in range(m):
            order = sorted(range(n), key=lambda i: (-S[j, i], i))[:k]
            assert ids[j].tolist() == order
            assert np.allclose(sc[j], S[j, order], rtol=0, atol=1e-12)


def test_grouped_scores_select_cluster_view():
    """Eq.(15)/Alg. 4: each row is scored with its own cluster's query view; equals the
    lazy form <A_{c_i} q, x_low_i> (Alg. 3) computed per pair."""
    rng = _rng(15)
    n, D, d, C = 60, 7, 3, 4
    X = rng.standard_normal((n, D))
    A = rng.standard_normal((C, d, D))
    B = rng.standard_normal((C, d, D))
    a = rng.integers(0, C, n).astype(np.int32)
    q = rng.standard_normal((2, D))
    S = O.reduced_scores(O.project(q, A), O.encode(X, B, a), a)
    for j in range(2):
        for i in range(n):
            lazy = float(np.dot(A[a[i]] @ q[j], B[a[i]] @ X[i]))
            assert abs(S[j, i] - lazy) < 1e-12


def test_rerank_full_R_is_exact_knn_and_dD_is_exact():
    """R = n -> result = exact k-NN; d = D (pure) -> identical to exact search."""
    rng = _rng(16)
    Q, X = _ood_pair(rng, m=50, n=300, D=10)
    gt, gts = O.exact_topk(Q[:6], X, 10)
    f = O.sphering_fit(Q, X, 3)
    r = O.search(Q[:6], X, f["A"], f["B"], None, R=300, k=10)
    assert np.array_equal(r["ids"], gt)
    f = O.sphering_fit(Q, X, 10)
    r = O.search(Q[:6], X, f["A"], f["B"], None, R=12, k=10)
    assert np.array_equal(r["ids"], gt)
    assert O.recall_at_k(gt, gt) == 1.0


# ---------------------------------------------------------------- generator
def test_generator_prefix_and_determinism():
    c = lvgen.get_config(2, n=70_000)
    small = lvgen.get_config(2, n=1000)
    X1 = lvgen.database_rows(c, 65_000, 66_000)
    X2 = lvgen.database(c, workers=1)[65_000:66_000]
    assert np.array_equal(X1, X2)
    assert np.array_equal(lvgen.database(small, workers=1), lvgen.database(c, workers=1)[:1000])
    assert np.allclose(np.linalg.norm(X1.astype(np.float64), axis=1), 1.0, atol=1e-6)
    q = lvgen.queries(c, "test", m=64)
    assert q.dtype == np.float32 and np.allclose(np.linalg.norm(q, axis=1), 1, atol=1e-6)
    assert not np.array_equal(q, lvgen.queries(c, "learn", m=64))

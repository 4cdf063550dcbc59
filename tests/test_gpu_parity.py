"""GPU parity of the C-ABI path against the fp64 oracle (gates G1-G6 of DESIGN.md §4).

A/B stacks and tags come from the ORACLE's fit (cast to fp32, the library's input type),
so no oracle input is produced by the CUDA path.  The "emulated" oracle rounds x_low and
q' to the storage dtype exactly where the precision contract says.
"""
import numpy as np
import pytest
import torch

import lvgen
import oracle as O

pytestmark = pytest.mark.gpu

TOL_RED = 2e-3      # reduced scores (north star)
TOL_RR = 1e-5       # re-rank scores (north star)


@pytest.fixture(scope="module")
def lv():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_22347_b200 import lv as L
    return L


def _case(cfg_id=1, n=4097, m=300, d=None, C=1, R=None, k=10, D=None, seed_rows=None):
    if d is not None and d > lvgen.get_config(cfg_id).D:
        cfg_id = 2
    c = lvgen.get_config(cfg_id)
    over = {"n": n, "m_test": m}
    if d is not None:
        over["d"] = d
    c = c.replace(**over)
    X = lvgen.database(c, workers=1)
    Q = lvgen.queries(c, "test")
    Ql = lvgen.queries(c, "learn", m=min(c.m_learn, 2000))
    lr = lvgen.learn_rows(c.replace(n_learn=min(n, 5000)))
    Xl = X[lr].astype(np.float64)
    if C == 1:
        f = O.sphering_fit(Ql, Xl, c.d)
        A = f["A"][None]
        B = f["B"][None]
        assign = np.zeros(n, dtype=np.int32)
    else:
        g = O.gleanvec_fit(Ql, Xl, C, c.d, lvgen.kmeanspp_draws(c, C), max_iter=20)
        A, B = g["A"], g["B"]
        assign = O.assign_tags(X.astype(np.float64), g["centres"])
    A32 = A.astype(np.float32)
    B32 = B.astype(np.float32)
    return c, X, Q, A32, B32, assign, (R or c.R), k


def _gpu_index(lv, c, X, A32, B32, assign, C):
    ix = lv.lv_index_create(c.D, c.d, C, c.low_dtype, c.full_dtype, torch.from_numpy(A32).cuda(),
                            torch.from_numpy(B32).cuda())
    Xt = torch.from_numpy(X).cuda()
    lv.lv_encode_database(ix, Xt, torch.from_numpy(assign).cuda() if C > 1 else None)
    return ix


def _ulp_diff(a, b, dtype):
    """|a - b| in units of the storage ulp of b."""
    import ml_dtypes
    t = ml_dtypes.bfloat16 if dtype == "bf16" else np.float16
    bb = b.astype(t)
    nxt = np.nextafter(bb, np.array(np.inf, dtype=t)).astype(np.float64) - bb.astype(np.float64)
    nxt = np.where(nxt == 0, 1e-30, np.abs(nxt))
    return np.abs(a - b) / nxt


def _g1_ok(got, ref, absdot, dtype, D):
    """G1: |got - ref| <= 1 storage ulp(ref) + the fp32-accumulation bound D 2^-24 sum_k |b_k x_k|
    (the kernel accumulates in fp32, the oracle in fp64; near-zero outputs of cancelling dot
    products may differ by more than one of their own tiny ulps).  Returns (all ok, flip frac)."""
    u = _ulp_diff(got, ref, dtype)
    ulp = np.where(u > 0, np.abs(got - ref) / np.maximum(u, 1e-300), 0)
    import ml_dtypes
    t = ml_dtypes.bfloat16 if dtype == "bf16" else np.float16
    bb = ref.astype(t)
    # one storage ulp in either direction: at a power of two the neighbour away from zero is twice
    # as far as the one towards zero, and a flip may go either way
    up = np.abs(np.nextafter(bb, np.array(np.inf, dtype=t)).astype(np.float64) - bb.astype(np.float64))
    dn = np.abs(np.nextafter(bb, np.array(-np.inf, dtype=t)).astype(np.float64) - bb.astype(np.float64))
    one = np.maximum(up, dn)
    ok = np.abs(got - ref) <= one + D * 2.0 ** -24 * absdot
    return ok.all(), float((got != ref).mean())


def _tol_ok(got, ref, tol, scale):
    return np.abs(got - ref) <= tol * np.maximum(np.abs(ref), 1e-2 * scale)


@pytest.mark.parametrize("d", [32, 64, 96, 128, 160])
def test_g1_encode_project_and_raw_scores(lv, d):
    """G1 (x_low, q' within 1 storage ulp; flip fraction < 0.5 %) and the raw tensor-core scores
    against fp64 dots of the oracle's rounded operands.  A 1-ulp operand flip moves a score by up
    to ulp * |q'_e x_e|, so: every score within the flip bound 2^-7 sum_e |q'_e x_e| + 2e-3 |s|, and
    >= 99.9 % within the north-star 2e-3 relative tolerance (reading R11)."""
    C = 1
    c, X, Q, A32, B32, assign, R, k = _case(1, n=4097, m=300, d=d)
    ix = _gpu_index(lv, c, X, A32, B32, assign, C)
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    valid = perm >= 0
    assert np.array_equal(perm[valid], np.arange(c.n))
    xl_gpu = X_low.float().cpu().numpy().astype(np.float64)[valid]
    xl_ref = O.encode(X, B32[0], None, store=c.low_dtype)
    ok, flips = _g1_ok(xl_gpu, xl_ref, np.abs(X.astype(np.float64)) @ np.abs(B32[0].astype(np.float64)).T,
                       c.low_dtype, c.D)
    assert ok and flips < 5e-3, flips
    Qp = lv.lv_project_queries(ix, torch.from_numpy(Q).cuda()).float().cpu().numpy().astype(np.float64)
    qp_ref = O.project(Q, A32, store=c.low_dtype)[:, 0, :]
    ok, flips = _g1_ok(Qp, qp_ref, np.abs(Q.astype(np.float64)) @ np.abs(A32[0].astype(np.float64)).T,
                       c.low_dtype, c.D)
    assert ok and flips < 5e-3, flips
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, R, raw=True)
    raw = dbg["raw"].cpu().numpy()[: c.m_test][:, valid].astype(np.float64)
    ref = qp_ref @ xl_ref.T
    scale = np.linalg.norm(qp_ref, axis=1)[:, None] * np.linalg.norm(xl_ref, axis=1)[None, :]
    ok = _tol_ok(raw, ref, TOL_RED, scale)
    assert ok.mean() >= 0.999, (np.abs(raw - ref).max(), (~ok).sum())
    flip = 2.0 ** -7 * (np.abs(qp_ref) @ np.abs(xl_ref).T) + TOL_RED * np.abs(ref) + 1e-6
    assert (np.abs(raw - ref) <= flip).all()


@pytest.mark.parametrize("D,d,C,xdt,low", [(200, 64, 1, "f32", "fp16"), (132, 32, 1, "f32", "bf16"),
                                           (132, 32, 2, "f16", "bf16"),
                                           (96, 96, 3, "f16", "bf16"), (768, 160, 2, "f32", "bf16"),
                                           (512, 128, 1, "f16", "fp16"), (256, 192, 1, "f32", "bf16")])
def test_g1_encode_shapes(lv, D, d, C, xdt, low, monkeypatch, planes="3"):
    """K6 (tensor-core encode) G1 across the shapes its layout depends on: ragged D (a partial last
    64-wide K block), fp16 input rows (D % 8 != 0: the scalar loads), several clusters (per-tile B
    rows, padded tiles), every d tile width.  x_low within 1 storage ulp + the fp32 accumulation
    bound of the oracle's fp64 B_c x, flips < 0.5 %."""
    monkeypatch.setenv("LV_K6_PLANES", planes)   # "2": the opt-in two-plane split (bf16 storage, R18)
    rng = np.random.default_rng(D * 7 + d)
    n = 3000
    X = rng.standard_normal((n, D)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    if xdt == "f16":
        X = X.astype(np.float16)
    B = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    A = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    assign = rng.integers(0, C, n).astype(np.int32)
    ix = lv.lv_index_create(D, d, C, low, "fp32", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), torch.from_numpy(assign).cuda() if C > 1 else None)
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    valid = perm >= 0
    X64 = X.astype(np.float64)
    a = assign if C > 1 else None
    B1 = B if C > 1 else B[0]
    xl_ref = O.encode(X64, B1, a, store=low)[perm[valid]]
    absdot = O.encode(np.abs(X64), np.abs(B1), a)[perm[valid]]
    got = X_low.float().cpu().numpy().astype(np.float64)
    if planes == "3":
        ok, flips = _g1_ok(got[valid], xl_ref, absdot, low, D)
        assert ok and flips < 5e-3, flips
    else:
        # two planes: 16 significant bits per operand, dropped terms <= 3 * 2^-18 sum|b x| (R18), on
        # top of the fp32 accumulation bound D 2^-24 sum|b x| of _g1_ok
        ok, flips = _g1_ok(got[valid], xl_ref, absdot * (1.0 + 3 * 2.0 ** -18 / 2.0 ** -24 / D), low, D)
        assert ok and flips < 1e-2, flips
    assert np.all(got[~valid] == 0)            # padded rows of a cluster's last tile encode to 0


@pytest.mark.parametrize("D,d,C,low,hplanes,direct", [(768, 160, 2, "bf16", "0", "1"), (200, 64, 1, "fp16", "0", "1"),
                                                       (512, 128, 3, "bf16", "3", "1"), (72, 32, 1, "bf16", "0", "1"),
                                                       (520, 96, 2, "fp16", "0", "1"), (768, 160, 2, "bf16", "0", "0")])
def test_g1_encode_fp16_rows_scaled_weights(lv, D, d, C, low, hplanes, direct, monkeypatch):
    """K6 for fp16 rows (R23): the rows are the fp16 operand as stored, B goes in as
    row-scaled fp16 planes bs = h + 2^-11 (m + l).  Weights whose rows span 2^-12..2^12 and whose
    entries span four decades inside a row, rows with entries over three decades (fp16 subnormals
    included): G1 against the oracle's fp64 B_c x, two planes (bf16 storage) and three; the last
    case runs the three-bf16-plane kernel (LV_K6_DIRECT=0) on the same inputs."""
    monkeypatch.setenv("LV_K6_HPLANES", hplanes)
    monkeypatch.setenv("LV_K6_DIRECT", direct)
    rng = np.random.default_rng(D * 11 + d)
    n = 2500
    X = rng.standard_normal((n, D)) * 10.0 ** rng.uniform(-3, 0, (n, D))
    X[:, ::7] *= 1e-4                                     # fp16 subnormals
    X = X.astype(np.float16)
    B = rng.standard_normal((C, d, D)) / np.sqrt(D) * 10.0 ** rng.uniform(-4, 0, (C, d, D))
    B *= 2.0 ** rng.integers(-12, 13, (C, d, 1))
    B[0, 1, :] = 0.0                                      # an all-zero weight row
    B = B.astype(np.float32)
    A = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    assign = rng.integers(0, C, n).astype(np.int32)
    ix = lv.lv_index_create(D, d, C, low, "fp16", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), torch.from_numpy(assign).cuda() if C > 1 else None)
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    valid = perm >= 0
    X64 = X.astype(np.float64)
    a = assign if C > 1 else None
    B1 = B if C > 1 else B[0]
    xl_ref = O.encode(X64, B1, a, store=low)[perm[valid]]
    absdot = O.encode(np.abs(X64), np.abs(B1), a)[perm[valid]]
    got = X_low.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all()
    # two fp16 planes carry b to 2^-22 relative: 2^-22 sum|b x| on top of _g1_ok's bound
    extra = 1.0 if hplanes == "3" or low == "fp16" or direct == "0" else 1.0 + 4.0 / D
    ok, flips = _g1_ok(got[valid], xl_ref, absdot * extra, low, D)
    assert ok and flips < 5e-3, flips
    assert np.all(got[~valid] == 0)
    assert np.all(got[valid][assign[perm[valid]] == 0, 1] == 0)   # the zero weight row


@pytest.mark.parametrize("D,d,C,xdt,full", [(512, 128, 1, "f32", "fp32"), (768, 160, 3, "f16", "fp16"),
                                             (200, 64, 2, "f32", "fp16"), (328, 96, 2, "f16", "fp32"),
                                             (204, 32, 1, "f32", "fp32"), (64, 32, 1, "f32", "fp32")])
def test_encode_full_copy_is_exact(lv, D, d, C, xdt, full):
    """X_full (the re-rank's full-precision rows, Alg. 1 l.3 P:92-95): bit-identical to X when the
    types agree, RNE(x) for fp32 -> fp16, x for fp16 -> fp32; original row order whatever the
    cluster sort does; n not a multiple of 128 and more tiles than one round of the persistent K6."""
    rng = np.random.default_rng(D + d)
    n = 128 * 150 + 77
    X = (rng.standard_normal((n, D)) * 10.0 ** rng.uniform(-3, 1, (n, 1))).astype(np.float32)
    if xdt == "f16":
        X = X.astype(np.float16)
    B = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    assign = rng.integers(0, C, n).astype(np.int32)
    ix = lv.lv_index_create(D, d, C, "bf16", full, torch.from_numpy(B).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), torch.from_numpy(assign).cuda() if C > 1 else None)
    Xf = lv.lv_index_export_full(ix).cpu().numpy()
    want = X.astype(np.float16 if full == "fp16" else np.float32)
    bits = np.uint16 if full == "fp16" else np.uint32
    assert Xf.dtype == want.dtype and np.array_equal(Xf.view(bits), want.view(bits))


@pytest.mark.parametrize("D,d,C", [(768, 160, 2), (200, 64, 1), (512, 128, 1)])
def test_g1_encode_two_planes_bf16(lv, D, d, C, monkeypatch):
    """The opt-in two-plane encode (LV_K6_PLANES=2, bf16 storage) within its own bound (R18)."""
    test_g1_encode_shapes(lv, D, d, C, "f32", "bf16", monkeypatch, planes="2")


@pytest.mark.parametrize("d,low", [(32, "bf16"), (64, "bf16"), (96, "bf16"), (128, "fp16"), (160, "bf16"),
                                   (64, "fp16")])
def test_mma_exact_operands(lv, d, low):
    """Tensor-core layout pin: signed selection matrices A, B and small-integer Q, X make every
    x_low, q' exactly representable and every score an exact integer, so the scan's raw scores
    must equal the fp64 dot products bit for bit (catches transposed operands, wrong swizzle or
    K offsets, lane/column mix-ups in the TMEM epilogue)."""
    rng = np.random.default_rng(d)
    D, n, m = 256, 3001, 260
    X = rng.integers(-4, 5, size=(n, D)).astype(np.float32)
    Q = rng.integers(-4, 5, size=(m, D)).astype(np.float32)
    A = np.zeros((1, d, D), np.float32)
    B = np.zeros((1, d, D), np.float32)
    A[0, np.arange(d), rng.permutation(D)[:d]] = rng.choice([-1.0, 1.0], d)
    B[0, np.arange(d), rng.permutation(D)[:d]] = rng.choice([-1.0, 1.0], d)
    ix = lv.lv_index_create(D, d, 1, low, "fp32", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda())
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, 64, raw=True)
    raw = dbg["raw"].cpu().numpy()
    ref = O.project(Q, A)[:, 0, :] @ O.encode(X, B).T
    assert np.array_equal(raw[:m, :n], ref)
    assert np.all(raw[:m, n:] < -1e30)          # padded tail columns are masked


def _check_search(lv, c, X, Q, A32, B32, assign, R, k, C, check_recall=True, timing=False):
    ix = _gpu_index(lv, c, X, A32, B32, assign, C)
    Qt = torch.from_numpy(Q).cuda()
    ids, sc, dbg = lv.lv_search(ix, Qt, k, R, cand=True, timing=timing)
    ids = ids.cpu().numpy().astype(np.int64)
    sc = sc.cpu().numpy().astype(np.float64)
    cid = dbg["cand_ids"].cpu().numpy().astype(np.int64)
    csc = dbg["cand_scores"].cpu().numpy().astype(np.float64)
    ref = O.search(Q, X, A32, B32, assign if C > 1 else None, R, k, store=c.low_dtype)
    m = Q.shape[0]
    check_g2_strict(lv, ix, Qt, cid, csc, C)
    # G2: candidate reduced scores vs oracle fp64 reduced scores of the same (q, id).  A one-ulp
    # storage flip of one operand element moves a score by <= 2^-8 |q'_e x_e| (R11):
    # every score within the flip bound F = 2^-7 sum_e |q'_e x_e| + 2e-3 |s|, >= 99.9 % within 2e-3
    S = O.reduced_scores(ref["Qp"], ref["X_low"], assign if C > 1 else None)
    F = 2.0 ** -7 * O.reduced_scores(np.abs(ref["Qp"]), np.abs(ref["X_low"]), assign if C > 1 else None)
    rows = np.arange(m)[:, None]
    got = csc
    exp = S[rows, cid]
    scale = np.abs(S).max()
    ok = _tol_ok(got, exp, TOL_RED, scale)
    assert ok.mean() >= 0.999, (~ok).sum()
    assert (np.abs(got - exp) <= F[rows, cid] + TOL_RED * np.abs(exp) + 1e-6).all()
    # G3: candidate sets equal except ids near the oracle's R-th score (2e-3 plus both flip bounds)
    for j in range(m):
        a, b = set(cid[j].tolist()), set(ref["cand"][j].tolist())
        thr = ref["cand_scores"][j, -1]
        iR = int(ref["cand"][j, -1])
        for i in a ^ b:
            band = TOL_RED * max(abs(thr), 1e-2) + F[j, i] + F[j, iR]
            assert abs(S[j, i] - thr) <= band, (j, i, S[j, i], thr)
        # sorted order of the GPU list follows (score desc, id asc) on its own scores
        keys = list(zip(-csc[j], cid[j]))
        assert keys == sorted(keys)
    # G4: re-rank scores vs fp64 <q, x> on canonical X
    check_topk_order(ids, sc)
    ex = np.einsum("md,mkd->mk", Q.astype(np.float64), X[ids].astype(np.float64))
    assert (np.abs(sc - ex) <= TOL_RR * np.maximum(np.abs(ex), 1e-2)).all(), np.abs(sc - ex).max()
    # G5: final ids equal except k-boundary near-ties or R-boundary swaps
    for j in range(m):
        if not np.array_equal(ids[j], ref["ids"][j]):
            a, b = set(ids[j].tolist()), set(ref["ids"][j].tolist())
            kth = ref["scores"][j, -1]
            thr = ref["cand_scores"][j, -1]
            iR = int(ref["cand"][j, -1])
            for i in a ^ b:
                rr = float(Q[j].astype(np.float64) @ X[i].astype(np.float64))
                near_k = abs(rr - kth) <= TOL_RR * max(abs(kth), 1e-2)
                near_r = abs(S[j, i] - thr) <= TOL_RED * max(abs(thr), 1e-2) + F[j, i] + F[j, iR]
                assert near_k or near_r, (j, i)
    # G6: recall against exact search
    if check_recall:
        gt, _ = O.exact_topk(Q, X, 10)
        r_gpu = O.recall_at_k(ids, gt, 10)
        r_ora = O.recall_at_k(ref["ids"], gt, 10)
        assert abs(r_gpu - r_ora) <= 1e-3 + 1e-12, (r_gpu, r_ora)
    return dbg


def check_topk_order(ids, sc):
    """Every returned row is ordered by (exact score desc, id asc) (reading R7)."""
    for j in range(ids.shape[0]):
        keys = list(zip((-sc[j]).tolist(), ids[j].tolist()))
        assert keys == sorted(keys), (j, keys)
        assert len(set(ids[j].tolist())) == ids.shape[1]


def check_g2_strict(lv, ix, Qt, cid, csc, C):
    """Strict G2: the candidates' reduced scores against fp64 dot products of the
    GPU's OWN stored operands (exported X_low, projected Q').  The tensor cores multiply those
    bf16/fp16 values exactly and accumulate in fp32, so every score is within the fp32
    accumulation bound d 2^-23 sum_e |q'_e x_e| (+1e-7), far inside the north-star 2e-3."""
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    Qp = lv.lv_project_queries(ix, Qt).float().cpu().numpy().astype(np.float64)
    d = Qp.shape[1] // C                            # the search width (a prefix of the stored d)
    xl = X_low.float().cpu().numpy().astype(np.float64)[:, :d]
    pos = np.full(perm.max() + 1, -1, dtype=np.int64)
    valid = perm >= 0
    pos[perm[valid]] = np.nonzero(valid)[0]
    cl = np.zeros(perm.shape[0], dtype=np.int64)
    for c in range(C):
        cl[offs[c]:offs[c + 1]] = c
    for j in range(cid.shape[0]):
        p = pos[cid[j]]
        assert (p >= 0).all()
        q = Qp[j].reshape(-1, d)[cl[p]]            # the view of each candidate's cluster
        s_ref = np.einsum("rd,rd->r", q, xl[p])
        bound = d * 2.0 ** -23 * np.einsum("rd,rd->r", np.abs(q), np.abs(xl[p])) + 1e-7
        assert (np.abs(csc[j] - s_ref) <= bound).all(), (j, np.abs(csc[j] - s_ref).max())
        assert (np.abs(csc[j] - s_ref) <= TOL_RED * np.maximum(np.abs(s_ref), 1e-2)).all()


def test_search_parity_config1_full(lv):
    """Config 1 at its full size (n=10 000, m=100, d=32, R=50, k=10)."""
    c, X, Q, A32, B32, assign, R, k = _case(1, n=10_000, m=100)
    _check_search(lv, c, X, Q, A32, B32, assign, R, k, 1)


@pytest.mark.parametrize("m,n,d,R", [(1, 4097, 64, 50), (257, 5000, 96, 100), (300, 1000, 128, 200),
                                     (129, 777, 160, 64), (40, 300, 32, 256)])
def test_search_parity_shapes(lv, m, n, d, R):
    """Ragged m (1, 129, 257, 300), ragged n, every d, R up to n (R = n: exact k-NN)."""
    c, X, Q, A32, B32, assign, _, k = _case(1, n=n, m=m, d=d)
    _check_search(lv, c, X, Q, A32, B32, assign, R, k, 1)


def test_search_R_equals_n_is_exact_knn(lv):
    c, X, Q, A32, B32, assign, _, k = _case(1, n=256, m=40, d=32)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 1)
    ids, sc, _ = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, 256)
    gt, gts = O.exact_topk(Q, X, k)
    ids = ids.cpu().numpy()
    sc = sc.cpu().numpy().astype(np.float64)
    check_topk_order(ids, sc)
    for j in range(Q.shape[0]):
        if not np.array_equal(ids[j], gt[j]):
            # R = n: the candidate set is the whole database, so only fp32-vs-fp64 re-rank near-ties
            # (within the 1e-5 re-rank tolerance of the k-th exact score) may change the top-k
            kth = gts[j, -1]
            for i in set(ids[j].tolist()) ^ set(gt[j].tolist()):
                r = float(Q[j].astype(np.float64) @ X[i].astype(np.float64))
                assert abs(r - kth) <= TOL_RR * max(abs(kth), 1e-2), (j, i, r, kth)


def test_duplicates_and_constant_scores(lv):
    """Exact ties: duplicated rows and an all-equal database; ties go to the lowest id."""
    c, X, Q, A32, B32, assign, _, k = _case(1, n=2000, m=50, d=32)
    X = X.copy()
    X[1000:1300] = X[7]                  # 300 duplicates of row 7 (tie block crosses tiles)
    _check_search(lv, c, X, Q, A32, B32, assign, 100, k, 1, check_recall=False)
    Xc = np.repeat(X[:1], 1500, axis=0)  # constant scores for every query
    ix = _gpu_index(lv, c.replace(n=1500), Xc, A32, B32, np.zeros(1500, np.int32), 1)
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, 64, cand=True)
    assert np.array_equal(dbg["cand_ids"].cpu().numpy(), np.tile(np.arange(64), (Q.shape[0], 1)))
    assert np.array_equal(ids.cpu().numpy(), np.tile(np.arange(k), (Q.shape[0], 1)))


def test_gleanvec_parity_small(lv):
    """GleanVec (Eq.(15), Alg. 4) with C=4 oracle clusters, grouped scan over the cluster-sorted
    X_low; includes the perm/offset layout (G1) and the search gates."""
    c, X, Q, A32, B32, assign, R, k = _case(3, n=6000, m=200, d=96, C=4)
    C = 4
    ix = _gpu_index(lv, c, X, A32, B32, assign, C)
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    assert offs[-1] == X_low.shape[0]
    for cc in range(C):
        seg = perm[offs[cc]:offs[cc + 1]]
        seg = seg[seg >= 0]
        assert np.array_equal(seg, np.nonzero(assign == cc)[0])     # stable
    valid = perm >= 0
    xl_ref = O.encode(X, B32, assign, store=c.low_dtype)[perm[valid]]
    absdot = O.encode(np.abs(X), np.abs(B32), assign)[perm[valid]]
    ok, flips = _g1_ok(X_low.float().cpu().numpy().astype(np.float64)[valid], xl_ref, absdot, c.low_dtype, c.D)
    assert ok and flips < 5e-3, flips
    _check_search(lv, c, X, Q, A32, B32, assign, R, k, C)


def test_fit_stats_matches_definition(lv):
    """K7: K_Q = sum q q^T and K_X[c] = sum_{c_i = c} x x^T within 1e-6 relative."""
    c = lvgen.get_config(3, n=20_000)
    X = lvgen.database(c, workers=1)
    Q = lvgen.queries(c, "learn", m=9000)
    rng = np.random.default_rng(0)
    a = rng.integers(0, 5, size=X.shape[0]).astype(np.int32)
    KQ, KX = lv.lv_fit_stats(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda(), torch.from_numpy(a).cuda(), 5)
    Qd = Q.astype(np.float64)
    ref = Qd.T @ Qd
    assert np.linalg.norm(KQ - ref) / np.linalg.norm(ref) < 1e-6
    for cc in range(5):
        Xc = X[a == cc].astype(np.float64)
        ref = Xc.T @ Xc
        assert np.linalg.norm(KX[cc] - ref) / np.linalg.norm(ref) < 1e-6


def test_assign_tags_eq13(lv):
    """Eq.(13) on the GPU vs the oracle; fp32 may only disagree at near-ties."""
    c = lvgen.get_config(5, n=30_000)
    X = lvgen.database(c, workers=1)
    rng = np.random.default_rng(1)
    mu = rng.standard_normal((32, c.D))
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    got = lv.lv_assign_tags(torch.from_numpy(X).cuda(), torch.from_numpy(mu.astype(np.float32)).cuda()).cpu().numpy()
    mu32 = mu.astype(np.float32).astype(np.float64)
    ref = O.assign_tags(X.astype(np.float64), mu32)
    S = X.astype(np.float64) @ mu32.T
    for i in np.nonzero(got != ref)[0]:
        assert abs(S[i, got[i]] - S[i, ref[i]]) < 1e-5


def test_search_host_buffers(lv):
    c, X, Q, A32, B32, assign, R, k = _case(1, n=3000, m=77, d=64)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 1)
    ids_d, sc_d, _ = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, R)
    ids_h, sc_h = lv.lv_search_host(ix, torch.from_numpy(Q).pin_memory(), k, R)
    assert np.array_equal(ids_d.cpu().numpy(), ids_h.numpy())
    assert np.array_equal(sc_d.cpu().numpy(), sc_h.numpy())


def test_bad_arguments_return_status(lv):
    c, X, Q, A32, B32, assign, R, k = _case(1, n=1000, m=10, d=32)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 1)
    with pytest.raises(lv.LVError, match="status 2"):
        lv.lv_search(ix, torch.from_numpy(Q).cuda(), 20, 10)          # k > R
    with pytest.raises(lv.LVError, match="status 2"):
        lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, 2000)        # R > n
    bad = np.full(1000, 7, dtype=np.int32)
    ix2 = lv.lv_index_create(c.D, c.d, 4, "bf16", "fp32", torch.zeros(4, c.d, c.D).cuda(), torch.zeros(4, c.d, c.D).cuda())
    with pytest.raises(lv.LVError, match="status 3"):
        lv.lv_encode_database(ix2, torch.from_numpy(X).cuda(), torch.from_numpy(bad).cuda())


def test_deterministic(lv):
    c, X, Q, A32, B32, assign, R, k = _case(1, n=5000, m=300, d=64)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 1)
    Qt = torch.from_numpy(Q).cuda()
    a = lv.lv_search(ix, Qt, k, R, cand=True)
    b = lv.lv_search(ix, Qt, k, R, cand=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2]["cand_ids"], b[2]["cand_ids"])


def test_sampled_path_parity(lv):
    """A database large enough (>= 64 sampled tiles, >= 8 j1 block maxima) for the sampled-threshold path: sample stage
    of block maxima, per-query threshold, one thresholded main scan, exactness check."""
    c, X, Q, A32, B32, assign, R, k = _case(1, n=200_000, m=300, d=64)
    dbg = _check_search(lv, c, X, Q, A32, B32, assign, R, k, 1, timing=True)
    assert dbg["path"] == 1


def test_sampled_path_stride32(lv, monkeypatch):
    """The sampled path with every 32nd tile sampled (the default from 32 768 tiles on: the 10M-row
    configurations), forced here on a database small enough for the whole oracle comparison: j1
    follows the stride, results stay the exact top-R / top-k."""
    monkeypatch.setenv("LV_SAMPLE_STRIDE", "32")
    c, X, Q, A32, B32, assign, R, k = _case(1, n=300_000, m=300, d=64)
    dbg = _check_search(lv, c, X, Q, A32, B32, assign, R, k, 1, timing=True)
    assert dbg["path"] == 1


def test_sampled_path_repairs(lv, monkeypatch):
    """A deliberately far too high sampled threshold (gamma 0.05: ~64 survivors for R = 256) makes
    every query fail the exactness check; round 1 repairs with the looser bound (about half fail
    again), round 2 without a threshold.  Results must still be the exact top-R / top-k."""
    monkeypatch.setenv("LV_SAMPLE_GAMMA", "0.05")
    c, X, Q, A32, B32, assign, _, k = _case(1, n=200_000, m=200, d=32)
    dbg = _check_search(lv, c, X, Q, A32, B32, assign, 256, k, 1, check_recall=False, timing=True)
    assert dbg["path"] == 1 and dbg["failed"][0] == Q.shape[0] and dbg["failed"][1] > 0, dbg["failed"]


def test_sampled_path_gleanvec(lv):
    """Sampled path on a cluster-sorted GleanVec index (C = 4): the sample is stratified per
    cluster segment, block maxima are indexed across segments."""
    c, X, Q, A32, B32, assign, R, k = _case(3, n=200_000, m=200, d=96, C=4)
    dbg = _check_search(lv, c, X, Q, A32, B32, assign, R, k, 4, timing=True)
    assert dbg["path"] == 1


@pytest.mark.parametrize("d_store,d_search,n", [(128, 64, 20_000), (128, 96, 200_000), (128, 128, 5000),
                                                (96, 32, 6000), (192, 96, 6000), (160, 32, 200_000)])
def test_flexible_search_dim(lv, d_store, d_search, n):
    """§3.1 flexible d: an index encoded at d_store and searched on its first d_search
    coordinates (lv_index_set_search_dim) returns exactly what an index built from the first
    d_search rows of the same A/B returns (the stored prefix and the projected prefix are the same
    numbers: K6 splits its accumulation the same way for both widths when d_store <= 128), on the
    staged and the sampled path; every case also passes the oracle gates on the prefix stacks."""
    c, X, Q, A32, B32, assign, R, k = _case(2, n=n, m=300, d=d_store)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 1)
    lv.lv_index_set_search_dim(ix, d_search)
    assert lv.lv_index_get_search_dim(ix) == d_search
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, R, cand=True)
    cp = c.replace(d=d_search)
    ix2 = _gpu_index(lv, cp, X, np.ascontiguousarray(A32[:, :d_search]), np.ascontiguousarray(B32[:, :d_search]),
                     assign, 1)
    ids2, sc2, dbg2 = lv.lv_search(ix2, torch.from_numpy(Q).cuda(), k, R, cand=True)
    assert dbg["path"] == dbg2["path"]
    Qp = lv.lv_project_queries(ix, torch.from_numpy(Q).cuda())
    assert Qp.shape[1] == d_search and torch.equal(Qp, lv.lv_project_queries(ix2, torch.from_numpy(Q).cuda()))
    if d_store <= 128:
        assert torch.equal(lv.lv_index_export(ix)[0][:, :d_search], lv.lv_index_export(ix2)[0])
        assert torch.equal(ids, ids2) and torch.equal(sc, sc2)
        assert torch.equal(dbg["cand_ids"], dbg2["cand_ids"])
    # and against the oracle on the prefix stacks (G3-G6 gates)
    _check_search(lv, cp, X, Q, np.ascontiguousarray(A32[:, :d_search]), np.ascontiguousarray(B32[:, :d_search]),
                  assign, R, k, 1)
    lv.lv_index_set_search_dim(ix, 0)   # back to the stored d
    assert lv.lv_index_get_search_dim(ix) == d_store


def test_flexible_search_dim_rejects(lv):
    c, X, Q, A32, B32, assign, R, k = _case(3, n=3000, m=50, d=96, C=2)
    ix = _gpu_index(lv, c, X, A32, B32, assign, 2)
    with pytest.raises(lv.LVError):
        lv.lv_index_set_search_dim(ix, 64)     # GleanVec: one P per cluster, no shared prefix
    c1, X1, Q1, A1, B1, a1, _, _ = _case(1, n=2000, m=20, d=64)
    ix1 = _gpu_index(lv, c1, X1, A1, B1, a1, 1)
    for bad in (96, 48):                       # > stored d; not a multiple of 32
        with pytest.raises(lv.LVError):
            lv.lv_index_set_search_dim(ix1, bad)

"""GPU parity of the 8-bit reduced vectors (NEXT-4; scalar quantisation of B x, P:129 / P:211;
DESIGN.md reading R21) against the int8-emulating oracle (oracle.search_i8).

Codes are integer decisions taken in fp32 on both sides; the GPU's fp32 products are
fp32-faithful, the oracle rounds its fp64 products once, so a code may differ by one at a rounding
boundary (the int8 analogue of G1).  With equal codes a score is bit-identical on both sides:
fl32(s * <q codes, x codes>), the integer dot product being exact on the int8 tensor cores.
Gates: G1-i8 codes within 1 (flips < 0.5 %), scales within 2 fp32 ulp; strict G2 (scores equal
fl32(s * dot) of the GPU's own codes, bit for bit); exact-operand pin; G3/G5 against the oracle
with code-flip bands; G4 re-rank within 1e-5; G6 recall within 0.001.
"""
import numpy as np
import pytest
import torch

import lvgen
import oracle as O
from test_gpu_parity import TOL_RED, TOL_RR, check_topk_order

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lv():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_22347_b200 import lv as L
    return L


def _fitted(cfg_id, n, m, d=None, C=1):
    c = lvgen.get_config(cfg_id)
    c = c.replace(n=n, m_test=m, **({"d": d} if d else {}))
    X = lvgen.database(c, workers=1)
    Q = lvgen.queries(c, "test")
    Ql = lvgen.queries(c, "learn", m=2000)
    Xl = X[lvgen.learn_rows(c.replace(n_learn=min(n, 5000)))].astype(np.float64)
    if C == 1:
        f = O.sphering_fit(Ql, Xl, c.d)
        A, B, assign = f["A"][None], f["B"][None], None
    else:
        g = O.gleanvec_fit(Ql, Xl, C, c.d, lvgen.kmeanspp_draws(c, C), max_iter=20)
        A, B = g["A"], g["B"]
        assign = O.assign_tags(X.astype(np.float64), g["centres"])
    return c, X, Q, A.astype(np.float32), B.astype(np.float32), assign


def _index(lv, c, X, A32, B32, assign, C):
    ix = lv.lv_index_create(c.D, c.d, C, "i8", c.full_dtype, torch.from_numpy(A32).cuda(), torch.from_numpy(B32).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), None if assign is None else torch.from_numpy(assign).cuda())
    return ix


def _gpu_codes(lv, ix, c, C):
    X_low, perm, offs = lv.lv_index_export(ix)
    perm = perm.cpu().numpy()
    valid = perm >= 0
    xc = np.zeros((int(perm.max()) + 1, c.d), dtype=np.int8)
    xc[perm[valid]] = X_low.cpu().numpy()[valid]
    return xc, lv.lv_index_i8_scales(ix)


@pytest.mark.parametrize("cfg_id,d,C", [(2, 128, 1), (3, 96, 4), (5, 160, 3), (4, 64, 1)])
def test_i8_codes_match_oracle(lv, cfg_id, d, C):
    """G1-i8: database codes, scales and query codes/scales against the oracle's quantiser."""
    c, X, Q, A32, B32, assign = _fitted(cfg_id, 8000, 300, d, C)
    ix = _index(lv, c, X, A32, B32, assign, C)
    xc, delta = _gpu_codes(lv, ix, c, C)
    B1 = B32 if C > 1 else B32[0]
    x_ref = O.encode(X, B1, assign)
    ref_c, ref_d = O.quantize_db_i8(x_ref, assign, C)
    # delta = max|x| / 127 inherits the fp32-faithful product's error at the column's extreme
    # (G1's accumulation bound D 2^-24 sum_k |b_k x_k|) plus one fp32 ulp of each division
    absdot = O.encode(np.abs(X.astype(np.float64)), np.abs(B1), assign)
    a = np.zeros(X.shape[0], np.int64) if assign is None else assign
    for cc in range(C):
        rows = np.nonzero(a == cc)[0]
        if rows.size == 0:
            continue
        arg = rows[np.argmax(np.abs(x_ref[rows]), axis=0)]
        bound = (c.D * 2.0 ** -24 * absdot[arg, np.arange(c.d)] / 127.0
                 + 2.0 ** -22 * ref_d[cc].astype(np.float64))
        assert np.all(np.abs(delta[cc].astype(np.float64) - ref_d[cc].astype(np.float64)) <= bound), cc
    diff = np.abs(xc.astype(int) - ref_c.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() < 5e-3, (diff > 0).mean()
    qc, qs = lv.lv_project_queries_i8(ix, torch.from_numpy(Q).cuda())
    rq, rs = O.quantize_queries_i8(O.project(Q, A32), delta)   # the GPU's delta: query parity alone
    qd = np.abs(qc.cpu().numpy().reshape(rq.shape).astype(int) - rq.astype(int))
    assert qd.max() <= 1 and (qd > 0).mean() < 5e-3
    # s = max|q' delta| / 127 with the same fp32-accumulation allowance on q' (K1's product)
    qabs = O.project(np.abs(Q.astype(np.float64)), np.abs(A32))                  # [m, C, d]
    sbound = (c.D * 2.0 ** -24 * (qabs * delta[None].astype(np.float64)).max(axis=2) / 127.0
              + 2.0 ** -22 * rs.astype(np.float64))
    assert np.all(np.abs(qs.cpu().numpy().astype(np.float64) - rs.astype(np.float64)) <= sbound)


@pytest.mark.parametrize("d", [32, 64, 96, 128, 160, 192])
def test_i8_exact_operands(lv, d):
    """Layout pin of the kind::i8 scan: integer data whose quantisation is exact (every column of
    x_low reaches 127, every query view reaches 127, so delta = s = 1 and the codes are the
    values): every raw score equals the integer dot product (catches wrong swizzle, K offsets,
    TMEM A packing, lane / column mix-ups)."""
    rng = np.random.default_rng(d)
    D, n, m = 256, 3001, 260
    X = rng.integers(-127, 128, size=(n, D)).astype(np.float32)
    X[0] = 127.0
    sel_b = rng.permutation(D)[:d]
    sel_a = rng.permutation(D)[:d]
    A = np.zeros((1, d, D), np.float32)
    B = np.zeros((1, d, D), np.float32)
    B[0, np.arange(d), sel_b] = 1.0
    A[0, np.arange(d), sel_a] = rng.choice([-1.0, 1.0], d)
    Q = rng.integers(-127, 128, size=(m, D)).astype(np.float32)
    Q[:, sel_a[0]] = 127.0
    ix = lv.lv_index_create(D, d, 1, "i8", "fp32", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda())
    assert np.array_equal(lv.lv_index_i8_scales(ix), np.ones((1, d), np.float32))
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, 64, raw=True)
    raw = dbg["raw"].cpu().numpy()
    ref = O.project(Q, A)[:, 0, :] @ O.encode(X, B).T
    assert np.array_equal(raw[:m, :n], ref)
    assert np.all(raw[:m, n:] < -1e30)


def check_i8_search(lv, ix, c, X, Q, A32, B32, assign, C, R, k, check_recall=True):
    Qt = torch.from_numpy(Q).cuda()
    ids, sc, dbg = lv.lv_search(ix, Qt, k, R, cand=True)
    ids = ids.cpu().numpy().astype(np.int64)
    sc = sc.cpu().numpy().astype(np.float64)
    cid = dbg["cand_ids"].cpu().numpy().astype(np.int64)
    csc = dbg["cand_scores"].cpu().numpy()
    m = Q.shape[0]
    # strict G2: fl32(s * dot) of the GPU's own codes, bit for bit
    xc, delta = _gpu_codes(lv, ix, c, C)
    qc, qs = lv.lv_project_queries_i8(ix, Qt)
    qc = qc.cpu().numpy().reshape(m, C, c.d).astype(np.int64)
    qs = qs.cpu().numpy()
    a = np.zeros(X.shape[0], np.int64) if assign is None else assign.astype(np.int64)
    for j in range(m):
        cl = a[cid[j]]
        dots = np.einsum("rd,rd->r", qc[j, cl], xc[cid[j]].astype(np.int64))
        exp = (qs[j, cl] * dots.astype(np.float32)).astype(np.float32)
        assert np.array_equal(csc[j], exp), j
    # against the oracle (its own codes)
    ref = O.search_i8(Q, X, A32 if C > 1 else A32[0], B32 if C > 1 else B32[0], assign, R, k, C=C)
    S = O.reduced_scores(ref["Qeff"], ref["x_codes"].astype(np.float64), assign).astype(np.float32).astype(np.float64)
    s_ref = ref["q_scales"]
    for j in range(m):
        thr = ref["cand_scores"][j, -1]
        band = TOL_RED * max(abs(thr), 1e-2) + 4 * 127 * float(s_ref[j].max())
        for i in set(cid[j].tolist()) ^ set(ref["cand"][j].tolist()):
            assert abs(S[j, i] - thr) <= band, (j, i, S[j, i], thr)
    check_topk_order(ids, sc)
    ex = np.einsum("md,mkd->mk", Q.astype(np.float64), X[ids].astype(np.float64))
    assert (np.abs(sc - ex) <= TOL_RR * np.maximum(np.abs(ex), 1e-2)).all()
    for j in range(m):
        if not np.array_equal(ids[j], ref["ids"][j]):
            kth = ref["scores"][j, -1]
            thr = ref["cand_scores"][j, -1]
            band = TOL_RED * max(abs(thr), 1e-2) + 4 * 127 * float(s_ref[j].max())
            for i in set(ids[j].tolist()) ^ set(ref["ids"][j].tolist()):
                rr = float(Q[j].astype(np.float64) @ X[i].astype(np.float64))
                assert abs(rr - kth) <= TOL_RR * max(abs(kth), 1e-2) or abs(S[j, i] - thr) <= band, (j, i)
    if check_recall:
        gt, _ = O.exact_topk(Q, X, 10)
        r_gpu, r_ora = O.recall_at_k(ids, gt, 10), O.recall_at_k(ref["ids"], gt, 10)
        assert abs(r_gpu - r_ora) <= 1e-3 + 1e-12, (r_gpu, r_ora)
    return dbg


@pytest.mark.parametrize("cfg_id,n,m,d,C,R", [(2, 5000, 300, 128, 1, 100), (1, 10_000, 100, 32, 1, 50),
                                              (2, 200_000, 300, 64, 1, 100), (3, 200_000, 200, 96, 4, 100),
                                              (5, 30_000, 150, 160, 3, 200)])
def test_i8_search_parity(lv, cfg_id, n, m, d, C, R):
    """Staged and sampled paths, LeanVec-Sphering and GleanVec, fp16 full vectors (cfg 5 shape)."""
    c, X, Q, A32, B32, assign = _fitted(cfg_id, n, m, d, C)
    ix = _index(lv, c, X, A32, B32, assign, C)
    dbg = check_i8_search(lv, ix, c, X, Q, A32, B32, assign, C, R, 10)
    if n >= 200_000:
        assert dbg["path"] == 1


@pytest.mark.slow
def test_i8_fullsize_cfg2_sampled(lv):
    """The int8 scan at configuration 2's full size (1M x 512, d = 128, R = 100, m = 10 000 searched
    in one call, as bench.py --config 2 --low i8 times it); gates on 256 evenly spaced queries:
    strict G2 against the GPU's own codes, G3 / G5 against the oracle's int8 search of the full
    database with code-flip bands, G4 and G6."""
    c = lvgen.get_config(2)
    X = lvgen.database(c)
    Q = lvgen.queries(c, "test")
    Ql = lvgen.queries(c, "learn")
    f = O.sphering_fit(Ql, X[lvgen.learn_rows(c)].astype(np.float64), c.d)
    A32, B32 = f["A"][None].astype(np.float32), f["B"][None].astype(np.float32)
    ix = _index(lv, c, X, A32, B32, None, 1)
    Qt = torch.from_numpy(Q).cuda()
    ids, sc, dbg = lv.lv_search(ix, Qt, c.k, c.R, cand=True)
    assert dbg["path"] == 1
    sel = np.linspace(0, Q.shape[0] - 1, 256).astype(np.int64)
    ids = ids.cpu().numpy()[sel].astype(np.int64)
    sc = sc.cpu().numpy()[sel].astype(np.float64)
    cid = dbg["cand_ids"].cpu().numpy()[sel].astype(np.int64)
    csc = dbg["cand_scores"].cpu().numpy()[sel]
    Qs = Q[sel]
    xc, delta = _gpu_codes(lv, ix, c, 1)
    qc, qs = lv.lv_project_queries_i8(ix, torch.from_numpy(Qs).cuda())
    qc = qc.cpu().numpy().astype(np.int64)
    qs = qs.cpu().numpy()[:, 0]
    for j in range(len(sel)):
        dots = xc[cid[j]].astype(np.int64) @ qc[j]
        assert np.array_equal(csc[j], (qs[j] * dots.astype(np.float32)).astype(np.float32)), j
    ref = O.search_i8(Qs, X, A32[0], B32[0], None, c.R, c.k)
    S = O.reduced_scores(ref["Qeff"], ref["x_codes"].astype(np.float64)).astype(np.float32).astype(np.float64)
    for j in range(len(sel)):
        thr = ref["cand_scores"][j, -1]
        band = TOL_RED * max(abs(thr), 1e-2) + 4 * 127 * float(ref["q_scales"][j].max())
        for i in set(cid[j].tolist()) ^ set(ref["cand"][j].tolist()):
            assert abs(S[j, i] - thr) <= band, (j, i)
    check_topk_order(ids, sc)
    ex = np.einsum("md,mkd->mk", Qs.astype(np.float64), X[ids].astype(np.float64))
    assert (np.abs(sc - ex) <= TOL_RR * np.maximum(np.abs(ex), 1e-2)).all()
    for j in range(len(sel)):
        if not np.array_equal(ids[j], ref["ids"][j]):
            kth, thr = ref["scores"][j, -1], ref["cand_scores"][j, -1]
            band = TOL_RED * max(abs(thr), 1e-2) + 4 * 127 * float(ref["q_scales"][j].max())
            for i in set(ids[j].tolist()) ^ set(ref["ids"][j].tolist()):
                rr = float(Qs[j].astype(np.float64) @ X[i].astype(np.float64))
                assert abs(rr - kth) <= TOL_RR * max(abs(kth), 1e-2) or abs(S[j, i] - thr) <= band, (j, i)
    gt, _ = O.exact_topk(Qs, X, 10)
    assert abs(O.recall_at_k(ids, gt, 10) - O.recall_at_k(ref["ids"], gt, 10)) <= 1e-3 + 1e-12

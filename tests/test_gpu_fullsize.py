"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one lv_search
over the config's whole 10^4-query batch), checked on sampled queries that the fp64 oracle
computes one by one: its exact top-R under the reduced score over the full database (chunked
encode + score + running top-R), then gates G2-G5 of DESIGN.md §4 for those queries.

The A/B stacks come from the ORACLE's fit (cast to fp32, the library's input type) and the tags
from the oracle's k-means, so no oracle input is produced by the CUDA path.
"""
import numpy as np
import pytest
import torch

import lvgen
import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL_RED = 2e-3
TOL_RR = 1e-5
CHUNK = 1 << 17


@pytest.fixture(scope="module")
def lv():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_22347_b200 import lv as L
    return L


def _oracle_topR(Qp_s, X, B32, assign, R, store):
    """Exact top-R (score desc, id asc) of the reduced scores of the sampled queries over all rows:
    the oracle's reduced_search on chunks of its own encode, merged with its total-order top-k."""
    m = Qp_s.shape[0]
    best_i = [np.empty(0, dtype=np.int64) for _ in range(m)]
    best_s = [np.empty(0) for _ in range(m)]
    for lo in range(0, X.shape[0], CHUNK):
        hi = min(X.shape[0], lo + CHUNK)
        a = None if assign is None else assign[lo:hi]
        ci, cs = O.reduced_search(Qp_s, O.encode(X[lo:hi], B32, a, store=store), a, R)
        for j in range(m):
            best_i[j], best_s[j] = O.topk_total_order(np.concatenate([best_s[j], cs[j]]),
                                                      np.concatenate([best_i[j], ci[j] + lo]), R)
    return np.stack(best_i), np.stack(best_s)


@pytest.mark.parametrize("cfg_id,family,n_sample", [(2, None, 1000), (3, None, 1000), (4, "ood", 256), (4, "id", 256),
                                                    (5, None, 256)])
def test_fullsize_sampled_parity(lv, cfg_id, family, n_sample):
    """Gates G2-G6 on n_sample evenly spaced queries of the full 10^4-query search (1 000 at the
    1M-row configs, 256 at the 10M-row configs, where the oracle's full scan costs ~0.2 s/query)."""
    from test_gpu_parity import check_topk_order
    c = lvgen.get_config(cfg_id)
    X = lvgen.database(c)
    Q = lvgen.queries(c, "test", family=family)
    Ql = lvgen.queries(c, "learn", family=family)
    Xl = X[lvgen.learn_rows(c)].astype(np.float64)
    if c.C == 1:
        f = O.sphering_fit(Ql, Xl, c.d)
        A32, B32, assign = f["A"][None].astype(np.float32), f["B"][None].astype(np.float32), None
    else:
        g = O.gleanvec_fit(Ql, Xl, c.C, c.d, lvgen.kmeanspp_draws(c), max_iter=20)
        A32, B32 = g["A"].astype(np.float32), g["B"].astype(np.float32)
        assign = np.concatenate([O.assign_tags(X[lo:lo + CHUNK], g["centres"])
                                 for lo in range(0, X.shape[0], CHUNK)]).astype(np.int32)
    del Xl
    ix = lv.lv_index_create(c.D, c.d, c.C, c.low_dtype, c.full_dtype, torch.from_numpy(A32).cuda(),
                            torch.from_numpy(B32).cuda())
    Xd = torch.from_numpy(X).cuda()
    lv.lv_encode_database(ix, Xd, None if assign is None else torch.from_numpy(assign).cuda())
    del Xd
    ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), c.k, c.R, cand=True, timing=1)
    assert dbg["path"] == 1   # the sampled-threshold path bench.py times at these sizes
    sel = np.linspace(0, Q.shape[0] - 1, n_sample).astype(np.int64)
    ids = ids.cpu().numpy()[sel].astype(np.int64)
    sc = sc.cpu().numpy()[sel].astype(np.float64)
    cid = dbg["cand_ids"].cpu().numpy()[sel].astype(np.int64)
    csc = dbg["cand_scores"].cpu().numpy()[sel].astype(np.float64)
    Qs = Q[sel]
    Qp = O.project(Qs, A32, store=c.low_dtype)                         # [s, C, d]
    ref_i, ref_s = _oracle_topR(Qp, X, B32, assign, c.R, c.low_dtype)
    thr = ref_s[:, -1]
    # G2: the GPU candidates' reduced scores vs the oracle's score of the same (query, id)
    Xc = X[cid]                                                        # [s, R, D]
    n_ok = n_all = 0
    for j in range(len(sel)):
        a = None if assign is None else assign[cid[j]]
        xl = O.encode(Xc[j], B32, a, store=c.low_dtype)
        s_ref = O.reduced_scores(Qp[j:j + 1], xl, a)[0]
        flip = 2.0 ** -7 * O.reduced_scores(np.abs(Qp[j:j + 1]), np.abs(xl), a)[0]   # DESIGN.md R11
        scale = np.linalg.norm(Qp[j]) * np.linalg.norm(xl, axis=1).max()
        ok = np.abs(csc[j] - s_ref) <= TOL_RED * np.maximum(np.abs(s_ref), 1e-2 * scale)
        n_ok += int(ok.sum())
        n_all += ok.size
        assert (np.abs(csc[j] - s_ref) <= flip + TOL_RED * np.abs(s_ref) + 1e-6).all(), j
        # G3: same candidate set except ids near the oracle's R-th reduced score (2e-3 + flips)
        iR = np.array([ref_i[j, -1]])
        aR = None if assign is None else assign[iR]
        xR = O.encode(X[iR], B32, aR, store=c.low_dtype)
        fR = 2.0 ** -7 * O.reduced_scores(np.abs(Qp[j:j + 1]), np.abs(xR), aR)[0, 0]
        diff = set(cid[j].tolist()) ^ set(ref_i[j].tolist())
        for i in diff:
            ii = np.array([i])
            ai = None if assign is None else assign[ii]
            xi = O.encode(X[ii], B32, ai, store=c.low_dtype)
            si = float(O.reduced_scores(Qp[j:j + 1], xi, ai)[0, 0])
            fi = float(2.0 ** -7 * O.reduced_scores(np.abs(Qp[j:j + 1]), np.abs(xi), ai)[0, 0])
            assert abs(si - thr[j]) <= TOL_RED * max(abs(thr[j]), 1e-2) + fi + fR, (j, i, si, thr[j])
    assert n_ok >= 0.999 * n_all, (n_ok, n_all)
    # G4: re-rank scores vs fp64 <q, x> on the canonical vectors; rows ordered (score desc, id asc)
    check_topk_order(ids, sc)
    ex = np.einsum("md,mkd->mk", Qs.astype(np.float64), X[ids].astype(np.float64))
    assert (np.abs(sc - ex) <= TOL_RR * np.maximum(np.abs(ex), 1e-2)).all(), np.abs(sc - ex).max()
    # G5: final ids = the oracle's re-rank top-k of its own N_low, except boundary cases
    o_ids, o_sc = O.rerank_topk(Qs, X, ref_i, c.k)
    for j in range(len(sel)):
        if not np.array_equal(ids[j], o_ids[j]):
            for i in set(ids[j].tolist()) ^ set(o_ids[j].tolist()):
                rr = float(Qs[j].astype(np.float64) @ X[i].astype(np.float64))
                near_k = abs(rr - o_sc[j, -1]) <= TOL_RR * max(abs(o_sc[j, -1]), 1e-2)
                in_band = (i in set(cid[j].tolist())) != (i in set(ref_i[j].tolist()))
                assert near_k or in_band, (j, i)
    # G6: 10-recall@10 on the sample against exact search, GPU vs the emulated oracle
    gt, _ = O.exact_topk(Qs, X, 10)
    r_gpu, r_ora = O.recall_at_k(ids, gt, 10), O.recall_at_k(o_ids, gt, 10)
    assert abs(r_gpu - r_ora) <= 1e-3 + 1e-12, (r_gpu, r_ora)

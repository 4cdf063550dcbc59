"""Edge cases of the search layout: empty and one-row clusters, a database of one
partial tile, a second tile holding one row, many tiny clusters, k = R = n, and query batching
(lv_search splits m into equal-shape batches; results must not depend on it).  Every case goes
through the C ABI and the oracle gates of tests/test_gpu_parity.py (total order: score desc,
id asc, PAPER.md:46-48 / reading R7; Eq.(13) tags P:331-335)."""
import numpy as np
import pytest
import torch

import lvgen
import oracle as O
from test_gpu_parity import _check_search, _gpu_index, check_topk_order

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lv():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_22347_b200 import lv as L
    return L


def _rand_case(n, m, D, d, C, low="bf16", seed=0):
    """Seeded synthetic database / queries and random (not fitted) A_c, B_c: parity does not need
    a good reduction, only the same inputs on both sides."""
    rng = np.random.default_rng(seed)
    c = lvgen.get_config(1).replace(n=n, m_test=m, D=D, d=d, C=C, low_dtype=low)
    X = rng.standard_normal((n, D)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Q = rng.standard_normal((m, D)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    A = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    B = (rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)
    return c, X, Q, A, B


def test_empty_and_single_row_clusters(lv):
    """C = 5 with cluster 1 empty and cluster 3 holding a single row: the empty segment has no
    tiles, the single row is a 1-of-128 valid tile; both must neither be scanned wrongly nor
    returned."""
    c, X, Q, A, B = _rand_case(3000, 150, 128, 64, 5, seed=1)
    rng = np.random.default_rng(2)
    assign = rng.choice([0, 2, 4], size=c.n).astype(np.int32)
    assign[1234] = 3
    ix = _gpu_index(lv, c, X, A, B, assign, 5)
    X_low, perm, offs = lv.lv_index_export(ix)
    assert offs[2] - offs[1] == 0 and offs[4] - offs[3] == 128
    _check_search(lv, c, X, Q, A, B, assign, 100, 10, 5)


@pytest.mark.parametrize("C", [16, 32])
def test_many_small_clusters(lv, C):
    """C = 16 / 32 at small n: every cluster segment is one partial tile."""
    c, X, Q, A, B = _rand_case(1500, 200, 96, 32, C, seed=C)
    assign = np.random.default_rng(C).integers(0, C, c.n).astype(np.int32)
    _check_search(lv, c, X, Q, A, B, assign, 50, 10, C)


def test_k_equals_R_equals_n(lv):
    """n = 10, R = k = 10: the candidate list is the whole database; the result is exact k-NN
    (all 10 ids) ordered by the fp32 re-rank scores."""
    c, X, Q, A, B = _rand_case(10, 33, 64, 32, 1, seed=3)
    _check_search(lv, c, X, Q, A, B, np.zeros(10, np.int32), 10, 10, 1, check_recall=False)
    ix = _gpu_index(lv, c, X, A, B, np.zeros(10, np.int32), 1)
    ids, sc, _ = lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, 10)
    ids = ids.cpu().numpy()
    assert all(sorted(r) == list(range(10)) for r in ids.tolist())
    check_topk_order(ids, sc.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("n", [129, 128, 1])
def test_tile_boundaries(lv, n):
    """n = 129 (a second tile with one valid row), 128 (exactly one tile), 1 (one row)."""
    c, X, Q, A, B = _rand_case(n, 70, 64, 32, 1, seed=n)
    R = min(n, 50)
    k = min(R, 10)
    _check_search(lv, c, X, Q, A, B, np.zeros(n, np.int32), R, k, 1, check_recall=False)


def test_query_batching_is_transparent(lv, monkeypatch):
    """m = 700 with LV_MAX_BATCH = 256: three batches of 256 (the last one overlaps the second);
    ids, scores and candidate lists equal one unbatched search, and the host-buffer entry point
    (two overlapped batches) equals both."""
    c, X, Q, A, B = _rand_case(20_000, 700, 128, 64, 1, seed=9)
    ix = _gpu_index(lv, c, X, A, B, np.zeros(c.n, np.int32), 1)
    Qt = torch.from_numpy(Q).cuda()
    i1, s1, d1 = lv.lv_search(ix, Qt, 10, 100, cand=True)
    monkeypatch.setenv("LV_MAX_BATCH", "256")
    i2, s2, d2 = lv.lv_search(ix, Qt, 10, 100, cand=True)
    assert torch.equal(i1, i2) and torch.equal(s1, s2)
    assert torch.equal(d1["cand_ids"], d2["cand_ids"])
    monkeypatch.delenv("LV_MAX_BATCH")
    ih, sh = lv.lv_search_host(ix, torch.from_numpy(Q).pin_memory(), 10, 100)
    assert np.array_equal(ih.numpy(), i1.cpu().numpy()) and np.array_equal(sh.numpy(), s1.cpu().numpy())
    # large enough for the two-batch overlapped host path
    c2, X2, Q2, A2, B2 = _rand_case(30_000, 5000, 128, 64, 1, seed=10)
    ix2 = _gpu_index(lv, c2, X2, A2, B2, np.zeros(c2.n, np.int32), 1)
    i3, s3, _ = lv.lv_search(ix2, torch.from_numpy(Q2).cuda(), 10, 100)
    ih3, sh3 = lv.lv_search_host(ix2, torch.from_numpy(Q2).pin_memory(), 10, 100)
    assert np.array_equal(ih3.numpy(), i3.cpu().numpy()) and np.array_equal(sh3.numpy(), s3.cpu().numpy())


def test_output_buffers_are_checked(lv):
    c, X, Q, A, B = _rand_case(1000, 20, 64, 32, 1, seed=4)
    ix = _gpu_index(lv, c, X, A, B, np.zeros(c.n, np.int32), 1)
    Qt = torch.from_numpy(Q).cuda()
    bad = torch.empty((20, 5), dtype=torch.int32, device="cuda")
    sc = torch.empty((20, 10), dtype=torch.float32, device="cuda")
    with pytest.raises(lv.LVError):
        lv.lv_search(ix, Qt, 10, 50, out=(bad, sc))
    with pytest.raises(lv.LVError):
        lv.lv_search(ix, Qt, 10, 50, out=(torch.empty((20, 10), dtype=torch.int64, device="cuda"), sc))
    with pytest.raises(lv.LVError):
        lv.lv_search_host(ix, torch.from_numpy(Q), 10, 50, torch.empty((20, 10), dtype=torch.int32), torch.empty(3))
    # argument errors come back before any copy is enqueued
    with pytest.raises(lv.LVError, match="status 2"):
        lv.lv_search_host(ix, torch.from_numpy(Q), 20, 10)

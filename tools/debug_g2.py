"""Reproduce test_sampled_path_gleanvec's G2 check and print the mismatching candidates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O
from test_gpu_parity import _case, _gpu_index
from paper_2410_22347_b200 import lv
c, X, Q, A32, B32, assign, R, k = _case(3, n=200_000, m=200, d=96, C=4)
ix = _gpu_index(lv, c, X, A32, B32, assign, 4)
ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), k, R, cand=True, timing=True)
print("path", dbg["path"], "failed", dbg["failed"])
cid = dbg["cand_ids"].cpu().numpy().astype(np.int64); csc = dbg["cand_scores"].cpu().numpy().astype(np.float64)
ref = O.search(Q, X, A32, B32, assign, R, k, store=c.low_dtype)
S = O.reduced_scores(ref["Qp"], ref["X_low"], assign)
exp = S[np.arange(Q.shape[0])[:, None], cid]
bad = np.abs(csc - exp) > 2e-3 * np.maximum(np.abs(exp), 1e-2 * np.abs(S).max())
print("bad count", bad.sum(), "rows", np.unique(np.nonzero(bad)[0])[:10])
X_low, perm, offs = lv.lv_index_export(ix); perm = perm.cpu().numpy()
inv = np.full(len(X), -1); inv[perm[perm >= 0]] = np.nonzero(perm >= 0)[0]
for j, r in list(zip(*np.nonzero(bad)))[:12]:
    i = cid[j, r]
    pos = inv[i] if i >= 0 else -1
    print(f"q{j} rank{r} id {i} gpu {csc[j,r]:.6f} oracle {exp[j,r]:.6f} assign {assign[i] if i>=0 else None} sortedpos {pos} tile {pos//128} off_in_tile {pos%128} offs {offs.tolist()}")
    # which oracle id has the GPU score?
    hit = np.nonzero(np.abs(S[j] - csc[j, r]) < 1e-6)[0][:5]
    print("   oracle ids with that score:", hit, [inv[h] for h in hit])

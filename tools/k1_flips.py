"""q' flip rate of the K1 projection against RNE(fp64 product), per implementation (LV_K1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ml_dtypes, lvgen, oracle as O
from paper_2410_22347_b200 import lv
for cfg_id, d, D in [(1, 32, None), (2, 128, None), (5, 160, None)]:
    c = lvgen.get_config(cfg_id, n=2000, m_test=2000)
    Q = lvgen.queries(c, "test")
    rng = np.random.default_rng(0)
    A = rng.standard_normal((1, c.d, c.D)).astype(np.float32) / np.sqrt(c.D) * 8.0
    ix = lv.lv_index_create(c.D, c.d, 1, c.low_dtype, c.full_dtype, torch.from_numpy(A).cuda(), torch.from_numpy(A).cuda())
    ref = O.project(Q, A, store=c.low_dtype)[:, 0, :]
    exact = Q.astype(np.float64) @ A[0].astype(np.float64).T
    absd = np.abs(Q.astype(np.float64)) @ np.abs(A[0].astype(np.float64)).T
    for impl in ("simt", "tc"):
        os.environ["LV_K1"] = impl
        got = lv.lv_project_queries(ix, torch.from_numpy(Q).cuda()).float().cpu().numpy().astype(np.float64)
        fl = (got != ref)
        print(f"cfg{cfg_id} D={c.D} d={c.d} {impl}: flips {fl.mean():.5f}  max|err|/sum|qa| among flips "
              f"{(np.abs(got-exact)/absd)[fl].max() if fl.any() else 0:.2e}", flush=True)

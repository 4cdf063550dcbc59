"""K6 flip rate: fraction of x_low elements that differ from RNE(fp64 B x) (R18 / R23)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_22347_b200 import lv
import ml_dtypes

for D, d, xdt, low in [(512, 128, "f32", "bf16"), (512, 96, "f32", "bf16"), (768, 160, "f16", "bf16"), (512, 128, "f32", "fp16"),
                       (768, 160, "f16", "fp16")]:
    rng = np.random.default_rng(D + d)
    n = 20000
    X = rng.standard_normal((n, D)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    if xdt == "f16":
        X = X.astype(np.float16)
    B = (rng.standard_normal((1, d, D)) / np.sqrt(D)).astype(np.float32)
    ix = lv.lv_index_create(D, d, 1, low, "fp32" if xdt == "f32" else "fp16", torch.from_numpy(B).cuda(), torch.from_numpy(B).cuda())
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), None)
    X_low, perm, _ = lv.lv_index_export(ix)
    got = X_low.float().cpu().numpy()[:n].astype(np.float64)
    t = ml_dtypes.bfloat16 if low == "bf16" else np.float16
    ref = (X.astype(np.float64) @ B[0].astype(np.float64).T).astype(t).astype(np.float64)
    print(f"D={D} d={d} rows={xdt} low={low}: flips {np.mean(got != ref) * 100:.4f} %  max|diff|/ulp-ish {np.abs(got - ref).max():.3e}", flush=True)

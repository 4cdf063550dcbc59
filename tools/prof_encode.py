"""Time K6 (lv_encode_database's tensor-core encode) on random data of a given shape, for ncu.

  python tools/prof_encode.py --n 1000000 --D 768 --d 160 --C 32 [--reps 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_22347_b200 import lv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--D", type=int, default=768)
    ap.add_argument("--d", type=int, default=160)
    ap.add_argument("--C", type=int, default=1)
    ap.add_argument("--low", default="bf16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--xf16", action="store_true", help="fp16 database rows (cfg 5's canonical type)")
    ap.add_argument("--full", default=None, help="full dtype kept for the re-rank (default: the rows' type)")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(a.n, a.D, device="cuda", generator=g)
    if a.xf16:
        X = X.half()
    A = torch.randn(a.C, a.d, a.D, device="cuda", generator=g) / a.D ** 0.5
    B = torch.randn(a.C, a.d, a.D, device="cuda", generator=g) / a.D ** 0.5
    assign = torch.randint(0, a.C, (a.n,), device="cuda", dtype=torch.int32, generator=g) if a.C > 1 else None
    a.full = a.full or ("fp16" if a.xf16 else "fp32")
    ix = lv.lv_index_create(a.D, a.d, a.C, a.low, a.full, A, B)
    for r in range(a.reps):
        lv.lv_encode_database(ix, X, assign)
        t = lv.lv_encode_timing(ix)
        n_pad = ix.info()["n_pad"]
        byts = a.n * a.D * X.element_size() + n_pad * a.d * 2 + n_pad * 4
        gbs = byts / (t["encode_K6"] * 1e-3) / 1e9
        print(f"rep {r}: {t}  K6 {gbs:.0f} GB/s algorithmic ({byts / 1e9:.2f} GB)", flush=True)


if __name__ == "__main__":
    main()

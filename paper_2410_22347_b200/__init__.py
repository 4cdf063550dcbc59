"""B200-native (sm_100a) hot path of LeanVec-Sphering / GleanVec (arXiv 2410.22347).

Batched maximum-inner-product search over a dimensionality-reduced database:
project queries (A or every A_c), score every database vector in dimension d on tcgen05
tensor cores with a fused per-query top-R, re-rank the R candidates with full-D fp32
inner products, return the top-k.  The work is in liblv.so behind the C ABI of
include/lv.h; `lv` is its ctypes binding, `fit` the host-side statistics->eig glue.
"""
from . import lv  # noqa: F401

__all__ = ["lv"]

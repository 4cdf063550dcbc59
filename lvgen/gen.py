"""Seeded synthetic workloads shaped like the paper's datasets.

The paper's datasets (Table 1) are not available; these
generators stand in for them.  Config 2 stands in for the 1M x 512 cross-modal
shape of LAION-1M-OOD / WIT, config 3 for LAION-1M-OOD with
C=16, config 4 for T2I-10M-OOD plus an ID counterpart
(PAPER.md:530, 555-557), config 5 for RQA-10M-OOD.

Recipe (DESIGN.md §3 lists every reading):
* RNG: numpy default_rng(SeedSequence([cfg_seed, stream, chunk])), rows drawn in
  chunks of 65 536 so that any chunk regenerates independently and a config
  with fewer rows is exactly a prefix of the same distribution.
* Haar(D): QR of a D x D Gaussian with column signs fixed by sign(diag R).
* orth(M): polar factor U V^T of the SVD of M.
* G_ij ~ N(0, 1/D); spectrum lambda_j = j^-beta, j = 1..D.
* flat:    x = normalize(M_X (sqrt(lambda) * z))
* mixture: x = normalize(mu_k + sigma_w R_k (sqrt(lambda / sum lambda) * z)), k uniform
* queries (OOD): q = normalize(M_Q (sqrt(lambda) * z)), M_Q = orth(M_X + alpha G),
  optionally q <- normalize(q + mu_off), mu_off = 0.3 normalize(g).
* All draws and transforms are fp64; canonical arrays are RNE-rounded to fp32
  (database of config 5: fp16).  Queries are fp32.

Nothing here computes any step of the method; k-means++ receives its uniform
draws from `kmeanspp_draws` so both sides consume identical random numbers.
"""
from __future__ import annotations

import dataclasses
import functools
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

CHUNK = 65536

# stream ids
S_MATRIX, S_G, S_OFF, S_DB, S_QLEARN, S_QTEST, S_QLEARN_ID, S_QTEST_ID, S_LEARNROWS, S_KMPP = range(10)


@dataclasses.dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    n: int
    D: int
    d: int
    C: int                 # clusters used by the method (1 = LeanVec-Sphering)
    m_test: int
    m_learn: int
    n_learn: int           # rows of X used for the fit (0 = all rows)
    R: int
    k: int
    low_dtype: str         # "bf16" | "fp16"  (reduced vectors X_low and Q')
    full_dtype: str        # "fp32" | "fp16"  (full vectors kept for re-rank)
    beta: float
    kind: str              # "flat" | "mixture"
    mix_components: int
    sigma_w: float
    alpha: float           # query rotation perturbation
    offset: float          # norm of the shared query mean offset (0 = none)
    families: tuple = ("ood",)

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    1: Config(1, "tiny-lvs-ood-10Kx128", 10_000, 128, 32, 1, 100, 1_000, 0, 50, 10,
              "bf16", "fp32", 1.0, "flat", 0, 0.0, 0.8, 0.0),
    2: Config(2, "lvs-ood-1Mx512", 1_000_000, 512, 128, 1, 10_000, 100_000, 100_000, 100, 10,
              "bf16", "fp32", 0.7, "flat", 0, 0.0, 1.0, 0.3),
    3: Config(3, "gleanvec-1Mx512-C16", 1_000_000, 512, 96, 16, 10_000, 100_000, 100_000, 100, 10,
              "bf16", "fp32", 0.7, "mixture", 16, 1.0, 1.0, 0.3),
    4: Config(4, "lvs-id-ood-10Mx200", 10_000_000, 200, 64, 1, 10_000, 100_000, 100_000, 100, 10,
              "fp16", "fp32", 0.5, "flat", 0, 0.0, 1.2, 0.0, ("id", "ood")),
    5: Config(5, "gleanvec-10Mx768-C32", 10_000_000, 768, 160, 32, 10_000, 100_000, 100_000, 200, 10,
              "bf16", "fp16", 0.6, "mixture", 32, 1.0, 1.0, 0.0),
}


def get_config(i: int, **overrides) -> Config:
    c = CONFIGS[i]
    return c.replace(**overrides) if overrides else c


def full_dtype_np(cfg: Config):
    return np.float16 if cfg.full_dtype == "fp16" else np.float32


def _rng(cfg: Config, stream: int, chunk: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([cfg.cfg_id, stream, chunk]))


def _normalize(Y: np.ndarray) -> np.ndarray:
    return Y / np.linalg.norm(Y, axis=-1, keepdims=True)


def _haar(D: int, rng: np.random.Generator) -> np.ndarray:
    Z = rng.standard_normal((D, D))
    Qm, Rm = np.linalg.qr(Z)
    return Qm * np.sign(np.diag(Rm))[None, :]


def _orth(M: np.ndarray) -> np.ndarray:
    U, _, Vt = np.linalg.svd(M)
    return U @ Vt


def _spectrum(cfg: Config) -> np.ndarray:
    j = np.arange(1, cfg.D + 1, dtype=np.float64)
    return j ** (-cfg.beta)


# the matrices only depend on (cfg_id, D, beta, kind, components, alpha) -- cache them
def _mkey(cfg: Config):
    return (cfg.cfg_id, cfg.D, cfg.kind, cfg.mix_components, cfg.alpha, cfg.offset)


@functools.lru_cache(maxsize=8)
def _matrices(key):
    cfg_id, D, kind, K, alpha, offset = key
    cfg = Config(cfg_id, "", 0, D, 0, 1, 0, 0, 0, 0, 0, "bf16", "fp32", 0.0, kind, K, 0.0, alpha, offset)
    out = {}
    r0 = _rng(cfg, S_MATRIX)
    r1 = _rng(cfg, S_G)
    if kind == "flat":
        MX = _haar(D, r0)
        G = r1.standard_normal((D, D)) / np.sqrt(D)
        out["MX"] = MX
        out["MQ"] = _orth(MX + alpha * G)
    else:
        mu = _normalize(r0.standard_normal((K, D)))
        Rk = np.stack([_haar(D, r0) for _ in range(K)])
        Gk = np.stack([r1.standard_normal((D, D)) / np.sqrt(D) for _ in range(K)])
        out["mu"] = mu
        out["Rk"] = Rk
        out["RQk"] = np.stack([_orth(Rk[k] + alpha * Gk[k]) for k in range(K)])
    if offset > 0:
        g = _rng(cfg, S_OFF).standard_normal(D)
        out["mu_off"] = offset * g / np.linalg.norm(g)
    return out


def _mats(cfg: Config):
    return _matrices(_mkey(cfg))


def _draw_rows(cfg: Config, stream: int, chunk: int, rows: int, family: str) -> np.ndarray:
    """fp64 rows [rows, D] of chunk `chunk` of stream `stream`."""
    mats = _mats(cfg)
    rng = _rng(cfg, stream, chunk)
    lam = _spectrum(cfg)
    D = cfg.D
    if cfg.kind == "flat":
        z = rng.standard_normal((rows, D))
        M = mats["MX"] if (stream == S_DB or family == "id") else mats["MQ"]
        Y = _normalize((z * np.sqrt(lam)) @ M.T)
        if stream != S_DB and family != "id" and "mu_off" in mats:
            Y = _normalize(Y + mats["mu_off"])
        return Y
    K = cfg.mix_components
    comp = rng.integers(0, K, size=rows)
    z = rng.standard_normal((rows, D))
    s = np.sqrt(lam / lam.sum())
    rot = mats["Rk"] if stream == S_DB else mats["RQk"]
    Y = np.empty((rows, D))
    zs = z * s
    for k in range(K):
        idx = np.nonzero(comp == k)[0]
        if idx.size:
            Y[idx] = mats["mu"][k] + cfg.sigma_w * (zs[idx] @ rot[k].T)
    Y = _normalize(Y)
    if stream != S_DB and "mu_off" in mats:
        Y = _normalize(Y + mats["mu_off"])
    return Y


def _db_chunk(args):
    cfg, c, rows = args
    Y = _draw_rows(cfg, S_DB, c, rows, "db")
    return Y.astype(full_dtype_np(cfg))


def database_rows(cfg: Config, start: int, stop: int) -> np.ndarray:
    """Canonical database rows [start, stop) (fp32, or fp16 for full_dtype fp16)."""
    out = np.empty((stop - start, cfg.D), dtype=full_dtype_np(cfg))
    c0, c1 = start // CHUNK, (stop - 1) // CHUNK
    for c in range(c0, c1 + 1):
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, cfg.n)
        blk = _db_chunk((cfg, c, hi - lo))
        a, b = max(lo, start), min(hi, stop)
        out[a - start:b - start] = blk[a - lo:b - lo]
    return out


def database(cfg: Config, workers: int | None = None) -> np.ndarray:
    """Canonical database X [n, D]; chunks generated in parallel processes."""
    nch = (cfg.n + CHUNK - 1) // CHUNK
    jobs = [(cfg, c, min(CHUNK, cfg.n - c * CHUNK)) for c in range(nch)]
    out = np.empty((cfg.n, cfg.D), dtype=full_dtype_np(cfg))
    workers = workers or min(len(os.sched_getaffinity(0)), 16)
    _mats(cfg)  # build matrices once in the parent (inherited by fork)
    if nch <= 2 or workers <= 1:
        for j in jobs:
            out[j[1] * CHUNK:j[1] * CHUNK + j[2]] = _db_chunk(j)
        return out
    import multiprocessing as mp
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        for j, blk in zip(jobs, ex.map(_db_chunk, jobs, chunksize=1)):
            out[j[1] * CHUNK:j[1] * CHUNK + j[2]] = blk
    return out


def queries(cfg: Config, split: str = "test", family: str | None = None, m: int | None = None) -> np.ndarray:
    """Query vectors, fp32 [m, D].  split in {learn, test}; family in {ood, id}."""
    family = family or cfg.families[-1]
    if family == "id":
        stream = S_QLEARN_ID if split == "learn" else S_QTEST_ID
    else:
        stream = S_QLEARN if split == "learn" else S_QTEST
    m = m if m is not None else (cfg.m_learn if split == "learn" else cfg.m_test)
    out = np.empty((m, cfg.D), dtype=np.float32)
    for c in range((m + CHUNK - 1) // CHUNK):
        rows = min(CHUNK, m - c * CHUNK)
        out[c * CHUNK:c * CHUNK + rows] = _draw_rows(cfg, stream, c, rows, family)
    return out


def learn_rows(cfg: Config) -> np.ndarray:
    """Sorted row indices of X used as X_learn (all rows if n_learn == 0 or >= n)."""
    if cfg.n_learn <= 0 or cfg.n_learn >= cfg.n:
        return np.arange(cfg.n, dtype=np.int64)
    idx = _rng(cfg, S_LEARNROWS).choice(cfg.n, size=cfg.n_learn, replace=False)
    return np.sort(idx).astype(np.int64)


def kmeanspp_draws(cfg: Config, C: int | None = None) -> np.ndarray:
    """Uniform [0,1) draws consumed by k-means++ seeding (one per centre)."""
    C = C or cfg.C
    return _rng(cfg, S_KMPP).random(C)

"""Pinned synthetic inputs for BASELINE.json configs 1-5 (TEST/BENCH INFRASTRUCTURE).

The paper's datasets are not available; seeded synthetic matrices with the
configs' shapes, sizes and value distributions stand in for them (DESIGN.md
"Inputs").  Both the GPU path and the CPU oracle read the identical arrays
(float64 on the host; the GPU takes the float32 cast where its config is fp32).

Choices BASELINE.json leaves open, pinned here:
* C2/C4 planted inner rank r0 = the factorisation rank (50 / 64).
* C4 uses the C2 generator ("the same generator as config 2") with seed 1.
* Sparse (C3/C5): per-column target nnz k_j = clip(ceil(c * z_j), 1, cap) with
  z_j ~ Zipf(1.1) and c found by bisection so sum k_j hits density * n * m
  (raw Zipf(1.1) capped at 2000 overshoots the density, so the draw is scaled
  rather than the cap dropped).  Rows are drawn with replacement from a
  Zipf(1.0) popularity law over a fixed seeded permutation of the rows
  (ceil(1.5 k_j) draws), deduplicated keeping first occurrences, truncated to
  k_j distinct rows.  Counts ~ Poisson(2) + 1; value = log1p(count) *
  ln(m / df_row) (tf-idf-style log scaling); explicit zeros (rows present in
  every column) are dropped exactly as matrix.py:from_triplets does.
"""

from __future__ import annotations

import numpy as np

from .nmf_oracle import Config, Csc


def c1():
    """Config 1: X = W0 H0 + |N(0, 0.01)|, W0 (500x10), H0 (10x1000) ~ U[0,1), seed 0."""
    rng = np.random.default_rng(0)
    w0 = rng.uniform(size=(500, 10))
    h0 = rng.uniform(size=(10, 1000))
    x = w0 @ h0 + np.abs(rng.normal(0.0, 0.01, size=(500, 1000)))
    return x


def dense_exp(n, m, r0, sigma, seed):
    """Configs 2/4: X = W0 H0 + |N(0, sigma)| with W0, H0 ~ Exp(1)."""
    rng = np.random.default_rng(seed)
    w0 = rng.exponential(1.0, size=(n, r0))
    h0 = rng.exponential(1.0, size=(r0, m))
    x = w0 @ h0
    x += np.abs(rng.normal(0.0, sigma, size=(n, m)))
    return x


def _column_targets(z, target, cap):
    lo, hi = 1e-9, 1e9
    for _ in range(200):
        c = np.sqrt(lo * hi)
        s = int(np.clip(np.ceil(c * z), 1, cap).sum())
        if s < target:
            lo = c
        else:
            hi = c
    return np.clip(np.ceil(hi * z), 1, cap).astype(np.int64)


def sparse_zipf(n, m, density, seed, cap=2000, oversample=1.5):
    """Configs 3/5: text-like CSC (see module docstring for the pinned rule)."""
    rng = np.random.default_rng(seed)
    cap = min(cap, n)
    target = int(round(density * n * m))
    perm = rng.permutation(n).astype(np.int64)
    z = rng.zipf(1.1, size=m).astype(np.float64)
    k = _column_targets(z, target, cap)
    draws = np.ceil(k * oversample).astype(np.int64)
    # Zipf(1.0) popularity over ranks 1..n via inverse CDF
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(int(draws.sum()))
    rank = np.minimum(np.searchsorted(cdf, u, side="right"), n - 1)
    rows = perm[rank]
    cols = np.repeat(np.arange(m, dtype=np.int64), draws)
    keys = cols * n + rows
    del rank, u
    uniq, first = np.unique(keys, return_index=True)
    ucol = uniq // n
    order = np.lexsort((first, ucol))
    ucol_o = ucol[order]
    starts = np.searchsorted(ucol_o, np.arange(m, dtype=np.int64), side="left")
    within = np.arange(len(order), dtype=np.int64) - starts[ucol_o]
    keep = np.sort(order[within < k[ucol_o]])
    kept = uniq[keep]
    i = kept % n
    j = kept // n
    counts = rng.poisson(2.0, size=len(kept)).astype(np.float64) + 1.0
    df = np.bincount(i, minlength=n).astype(np.float64)
    with np.errstate(divide="ignore"):
        idf = np.log(m / np.maximum(df, 1.0))
    vals = np.log1p(counts) * idf[i]
    return Csc.from_triplets(n, m, i, j, vals, sum_duplicates=False)


CONFIGS = {
    1: dict(kind="dense", shape=(500, 1000), rank=10, iters=50, dtype="f64",
            cfg=dict(rank=10, seed=0)),
    2: dict(kind="dense", shape=(10000, 20000), rank=50, iters=100, dtype="f32",
            cfg=dict(rank=50, seed=1)),
    3: dict(kind="sparse", shape=(100000, 50000), rank=100, iters=50, dtype="f32",
            cfg=dict(rank=100, seed=2)),
    4: dict(kind="dense", shape=(20000, 20000), rank=64, iters=100, dtype="f32",
            cfg=dict(rank=64, seed=1, mu1=0.1, beta2=0.01)),
    5: dict(kind="sparse", shape=(1000000, 200000), rank=200, iters=30, dtype="f32",
            cfg=dict(rank=200, seed=4)),
}


def make(config_id):
    """Return (X, Config) for BASELINE config 1-5 (X dense ndarray or Csc)."""
    c = CONFIGS[config_id]
    n, m = c["shape"]
    if config_id == 1:
        x = c1()
    elif config_id == 2:
        x = dense_exp(n, m, 50, 0.05, 1)
    elif config_id == 4:
        x = dense_exp(n, m, 64, 0.05, 1)
    elif config_id == 3:
        x = sparse_zipf(n, m, 1e-3, 2)
    else:
        x = sparse_zipf(n, m, 5e-4, 4)
    cfg = Config(max_outer=c["iters"], rel_change_tol=0.0, **c["cfg"])
    return x, cfg

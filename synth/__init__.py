"""Seeded synthetic inputs for the oblivious-forest hot path (BASELINE.json configs).

This module holds NO arithmetic of the method (no comparisons against
thresholds, no leaf indexing, no sums): it only draws factor matrices and raw
forests (feature_index[], thresholds[], leaf_values[]) from seeded numpy
generators.  Both the oracle (tests, bench cpu_baseline) and the CUDA path
consume its outputs; it is the only code they share.

Recipe:

* c1 (tiny): D=1024, F=32, x ~ U(0,1); T=64, depth 6; per feature a pool of 16
  sorted U(0,1) samples; each level picks a feature uniformly and a threshold
  uniformly from that feature's pool; leaves N(0, sigma=0.01).
* c2-c5 feature mix (kinds by a seeded permutation): 70% continuous N(0,1);
  20% sparse (0 w.p. 0.8, else LogNormal(0,1)); 10% discrete integers 0..15.
* c2-c5 border pools: per feature, the unique order statistics of the first
  min(D, 65536) documents at levels q_j = (j+1)/255, j < 254 (every border is a
  real sample value, so exact ties occur).
* c2-c5 splits: rank r ~ Zipf(s=1.1) truncated to 1..F, feature = perm[r-1]
  (seeded, independent of kinds); threshold uniform from that feature's pool;
  leaves N(0, sigma=0.005).
* Sizes: c2 100k x 1000, T=2000 d=6; c3 1M x 1000, T=10000 d=6;
  c4 4M x 500, T=4000 d=10; c5 pool 1M x 1000 (c2 mix), T=5000 d=6, queries of
  B in {100, 1000, 5000} docs at seeded offsets.

The paper's own workloads (a proprietary Yandex ranking model, and
unnamed synthetic models of Tables 5.1/6.1) are not available; these inputs
stand in for them with the production model's shape (depth-6 trees, ~1000
float factors).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

BLOCK = 65536  # rows per generation block (block 0 is the calibration sample)

# purpose tags for independent sub-streams (adding one never perturbs others)
_P_KINDS, _P_FACTORS, _P_SPLITFEAT, _P_SPLITPERM, _P_THR, _P_LEAVES, _P_POOL, _P_QUERY = range(1, 9)


def _rng(seed: int, purpose: int, *extra: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), purpose, *map(int, extra)]))


@dataclass
class ForestCase:
    """Raw inputs of one workload: factors [D, ld] fp32 and a raw oblivious forest."""
    name: str
    x: np.ndarray                 # float32 [n_docs, ld] (ld >= n_features)
    n_features: int
    feature_index: np.ndarray     # int32 [n_trees * depth], entry t*depth + l = level l
    thresholds: np.ndarray        # float32 [n_trees * depth]
    leaf_values: np.ndarray       # float32 [n_trees << depth]
    depth: int
    n_trees: int
    meta: dict = field(default_factory=dict)

    @property
    def n_docs(self) -> int:
        return int(self.x.shape[0])


CONFIGS = {
    "c1": dict(n_docs=1024, n_features=32, n_trees=64, depth=6, seed=1),
    "c2": dict(n_docs=100_000, n_features=1000, n_trees=2000, depth=6, seed=2),
    "c3": dict(n_docs=1_000_000, n_features=1000, n_trees=10_000, depth=6, seed=3),
    "c4": dict(n_docs=4_000_000, n_features=500, n_trees=4000, depth=10, seed=4),
    "c5": dict(n_docs=1_000_000, n_features=1000, n_trees=5000, depth=6, seed=5),
}
WORKLOAD_NAMES = {
    "c1": "c1-tiny-1024x32-T64-d6",
    "c2": "c2-ranking-100000x1000-T2000-d6",
    "c3": "c3-large-1000000x1000-T10000-d6",
    "c4": "c4-deep-4000000x500-T4000-d10",
    "c5": "c5-latency-pool1000000x1000-T5000-d6",
}
LEAF_SIGMA = {"c1": 0.01, "c2": 0.005, "c3": 0.005, "c4": 0.005, "c5": 0.005}


# --------------------------------------------------------------------------
# factor matrices
# --------------------------------------------------------------------------
def feature_kinds(seed: int, n_features: int) -> np.ndarray:
    """0 = continuous N(0,1), 1 = sparse, 2 = discrete 0..15 (70/20/10 %)."""
    perm = _rng(seed, _P_KINDS).permutation(n_features)
    n_cont = int(round(0.7 * n_features))
    n_sparse = int(round(0.2 * n_features))
    kinds = np.empty(n_features, np.int8)
    kinds[perm[:n_cont]] = 0
    kinds[perm[n_cont:n_cont + n_sparse]] = 1
    kinds[perm[n_cont + n_sparse:]] = 2
    return kinds


def _ranking_block(seed: int, b: int, rows: int, kinds: np.ndarray, out: np.ndarray) -> None:
    """Rows [b*BLOCK, b*BLOCK+rows) of a ranking-shaped factor matrix into out[rows, :F]."""
    F = kinds.size
    g = _rng(seed, _P_FACTORS, b)
    xt = np.empty((F, rows), np.float32)
    idx_c = np.flatnonzero(kinds == 0)
    idx_s = np.flatnonzero(kinds == 1)
    idx_d = np.flatnonzero(kinds == 2)
    xt[idx_c] = g.standard_normal((idx_c.size, rows), dtype=np.float32)
    zero = g.random((idx_s.size, rows), dtype=np.float32) < 0.8
    ln = np.exp(g.standard_normal((idx_s.size, rows), dtype=np.float64)).astype(np.float32)
    ln[zero] = 0.0
    xt[idx_s] = ln
    xt[idx_d] = g.integers(0, 16, (idx_d.size, rows)).astype(np.float32)
    out[:, :F] = xt.T


def ranking_factors(seed: int, n_docs: int, n_features: int, ld: int | None = None,
                    threads: int | None = None, out: np.ndarray | None = None,
                    rows: tuple[int, int] | None = None) -> np.ndarray:
    """Rows [0, n_docs) of the ranking-shaped matrix, or only rows [r0, r1) of it
    (rows=(r0, r1)): every block is drawn with its full-matrix row count, so a
    row range holds exactly the values of those rows of the whole matrix."""
    ld = n_features if ld is None else ld
    r0, r1 = (0, n_docs) if rows is None else (int(rows[0]), int(rows[1]))
    if not 0 <= r0 <= r1 <= n_docs:
        raise ValueError(f"rows [{r0}, {r1}) outside [0, {n_docs})")
    kinds = feature_kinds(seed, n_features)
    x = out if out is not None else np.empty((r1 - r0, ld), np.float32)
    if ld > n_features:
        x[:, n_features:] = 0.0
    nb = (n_docs + BLOCK - 1) // BLOCK

    def job(b):
        b0 = b * BLOCK
        brows = min(BLOCK, n_docs - b0)
        lo, hi = max(b0, r0), min(b0 + brows, r1)
        if lo >= hi:
            return
        if lo == b0 and hi == b0 + brows:
            _ranking_block(seed, b, brows, kinds, x[b0 - r0:b0 - r0 + brows])
        else:
            tmp = np.empty((brows, n_features), np.float32)
            _ranking_block(seed, b, brows, kinds, tmp)
            x[lo - r0:hi - r0, :n_features] = tmp[lo - b0:hi - b0]

    threads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(nb)))
    return x


# --------------------------------------------------------------------------
# forests
# --------------------------------------------------------------------------
def quantile_pools(calib: np.ndarray, n_levels: int = 254) -> list:
    """Per feature: unique order statistics of the calibration sample at
    levels q_j = (j+1)/(n_levels+1) (inverted-CDF: each border is a sample)."""
    n = calib.shape[0]
    srt = np.sort(calib, axis=0)
    q = (np.arange(n_levels) + 1) / (n_levels + 1)
    pos = np.clip(np.ceil(q * n).astype(np.int64) - 1, 0, n - 1)
    pools = []
    for f in range(calib.shape[1]):
        pools.append(np.unique(srt[pos, f]))
    return pools


def zipf_features(seed: int, n_nodes: int, n_features: int, s: float = 1.1) -> np.ndarray:
    ranks = np.arange(1, n_features + 1, dtype=np.float64)
    p = ranks ** (-s)
    p /= p.sum()
    r = _rng(seed, _P_SPLITFEAT).choice(n_features, size=n_nodes, p=p)
    perm = _rng(seed, _P_SPLITPERM).permutation(n_features)
    return perm[r].astype(np.int32)


def thresholds_from_pools(seed: int, feature_index: np.ndarray, pools: list) -> np.ndarray:
    g = _rng(seed, _P_THR)
    sizes = np.array([p.size for p in pools])
    pick = (g.random(feature_index.size) * sizes[feature_index]).astype(np.int64)
    return np.array([pools[f][k] for f, k in zip(feature_index, pick)], np.float32)


def leaves(seed: int, n_trees: int, depth: int, sigma: float, exact: bool = False) -> np.ndarray:
    g = _rng(seed, _P_LEAVES)
    n = n_trees << depth
    if exact:
        # integer * 2^-20, |integer| <= 1024: every fp32 partial sum of <= 10^4 trees is exact
        return (g.integers(-1024, 1025, n).astype(np.float64) * 2.0 ** -20).astype(np.float32)
    return g.normal(0.0, sigma, n).astype(np.float32)


def ranking_forest(seed: int, n_features: int, n_trees: int, depth: int, calib: np.ndarray,
                   sigma: float, exact_leaves: bool = False):
    pools = quantile_pools(calib)
    fi = zipf_features(seed, n_trees * depth, n_features)
    thr = thresholds_from_pools(seed, fi, pools)
    lv = leaves(seed, n_trees, depth, sigma, exact_leaves)
    return fi, thr, lv, pools


def tiny_case(seed: int = 1, n_docs: int = 1024, n_features: int = 32, n_trees: int = 64,
              depth: int = 6, pool: int = 16, sigma: float = 0.01, exact_leaves: bool = False,
              ld: int | None = None, name: str = "c1") -> ForestCase:
    """Config 1 recipe (also used with other sizes for parity sweeps)."""
    g = _rng(seed, _P_FACTORS, 0)
    ld = n_features if ld is None else ld
    x = np.zeros((n_docs, ld), np.float32)
    x[:, :n_features] = g.random((n_docs, n_features), dtype=np.float32)
    pools = np.sort(_rng(seed, _P_POOL).random((n_features, pool), dtype=np.float32), axis=1)
    gf = _rng(seed, _P_SPLITFEAT)
    fi = gf.integers(0, n_features, n_trees * depth).astype(np.int32)
    pick = _rng(seed, _P_THR).integers(0, pool, n_trees * depth)
    thr = pools[fi, pick].astype(np.float32)
    lv = leaves(seed, n_trees, depth, sigma, exact_leaves)
    return ForestCase(name, x, n_features, fi, thr, lv, depth, n_trees,
                      meta=dict(seed=seed, recipe="tiny"))


def make_case(name: str, n_docs: int | None = None, exact_leaves: bool = False,
              seed: int | None = None, ld: int | None = None,
              n_trees: int | None = None, rows: tuple[int, int] | None = None) -> ForestCase:
    """A BASELINE.json config by name ('c1'..'c5'); n_docs/n_trees may shrink it for tests.
    rows=(r0, r1) (c2-c5): x holds only documents [r0, r1) of the n_docs batch (one
    rank's shard), the model is the whole config's."""
    cfg = dict(CONFIGS[name])
    seed = cfg["seed"] if seed is None else seed
    D = cfg["n_docs"] if n_docs is None else int(n_docs)
    T = cfg["n_trees"] if n_trees is None else int(n_trees)
    if name == "c1":
        return tiny_case(seed, n_docs=D, n_trees=T, exact_leaves=exact_leaves, ld=ld, name=name)
    F, d = cfg["n_features"], cfg["depth"]
    # the calibration sample (block 0) defines the border pools whatever D is requested
    calib_rows = min(cfg["n_docs"], BLOCK)
    calib = np.empty((calib_rows, F), np.float32)
    _ranking_block(seed, 0, calib_rows, feature_kinds(seed, F), calib)
    fi, thr, lv, pools = ranking_forest(seed, F, T, d, calib, LEAF_SIGMA[name], exact_leaves)
    x = ranking_factors(seed, D, F, ld=ld, rows=rows)
    meta = dict(seed=seed, recipe="ranking", pool_sizes=[int(p.size) for p in pools],
                rows=list(rows) if rows is not None else [0, D])
    return ForestCase(name, x, F, fi, thr, lv, d, T, meta=meta)


def latency_queries(seed: int, pool_docs: int, batch: int, n_queries: int) -> np.ndarray:
    """Config 5: query q scores docs [o_q, o_q + batch) of the pool."""
    return _rng(seed, _P_QUERY, batch).integers(0, pool_docs - batch + 1, n_queries)


@dataclass
class PaperModel:
    """The paper's model layout, for the paper-native import (NEXT-2)."""
    n_features: int
    group_factor: np.ndarray   # int32 [n_groups]
    group_count: np.ndarray    # int32 [n_groups]
    thresholds: np.ndarray     # float32 [K]
    stc: np.ndarray            # int32 [9], trees per height 0..8
    cond_indices: np.ndarray   # uint32 [sum h*stc[h]], trees in descending height
    leaves: np.ndarray         # uint32 [sum 2^h*stc[h]]
    scale: float = 1.0
    bias: float = 0.0


def paper_model(seed: int, n_features: int, n_binary: int, stc) -> PaperModel:
    """A synthetic model of the paper's shape: n_binary binary features spread
    round-robin over the factors (one descriptor group per factor),
    thresholds U[0,1), condition indices uniform over the binary features, u32
    answers uniform over the full range, STC[h] trees of height h stored in
    descending height.  Table 6.1's synthetic model is
    n_binary=100 with 100 trees of each height."""
    g = _rng(seed, _P_THR, 99)
    base, extra = divmod(n_binary, n_features)
    counts = np.array([base + (1 if f < extra else 0) for f in range(n_features)], np.int32)
    gf = np.flatnonzero(counts > 0).astype(np.int32)
    gc = counts[gf]
    thr = np.concatenate([np.sort(g.random(c, dtype=np.float32)) for c in gc]) if gc.size else \
        np.zeros(0, np.float32)
    stc = np.asarray(stc, np.int32)
    heights = [h for h in range(len(stc) - 1, -1, -1) for _ in range(stc[h])]
    ci = g.integers(0, max(n_binary, 1), sum(heights)).astype(np.uint32)
    lv = g.integers(0, 2 ** 32, sum(1 << h for h in heights), dtype=np.uint64).astype(np.uint32)
    return PaperModel(n_features, gf, gc, thr.astype(np.float32), stc, ci, lv)

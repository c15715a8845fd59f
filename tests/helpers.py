"""Shared test helpers: oracle references (CPU) and CUDA-path runs on the same inputs."""
from __future__ import annotations

import numpy as np

import oracle


def tolerance(leaf_values: np.ndarray, depth: int) -> float:
    """BASELINE.json north_star: |err| <= 1e-5 * sum_t max_j |L_t[j]|."""
    if leaf_values.size == 0:
        return 0.0
    lv = np.abs(leaf_values.astype(np.float64)).reshape(-1, 1 << depth)
    return 1e-5 * float(lv.max(axis=1).sum())


def oracle_bins_used(case, n_docs=None):
    """Oracle bins restricted to the used features (ascending id), [n_docs, n_used]."""
    per, flat, counts, offs = oracle.borders(case.feature_index, case.thresholds, case.n_features)
    used = np.flatnonzero(counts > 0)
    b = oracle.bins(case.x, case.n_features, flat, counts, offs, n_docs=n_docs)
    return b[:, used], used, counts


def cuda_model(case, device=0):
    from paper_2205_07307_b200 import Model
    return Model(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                 case.n_features, device=device)


def to_dev(x, device=0):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{device}")


def run_cuda(model, x_dev, n_docs):
    """bins (blocked), fused scores, two-stage scores -- all on the GPU."""
    import torch
    bins = model.binarize(x_dev)
    s2 = model.apply(bins, n_docs)
    s1 = model.score(x_dev)
    torch.cuda.synchronize()
    return bins, s1, s2

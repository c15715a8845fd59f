#!/usr/bin/env python
"""Timing of a P:168-width model (1,950 factors -> 64-document tiles) on 1 M documents:
fused odf_score, binarize, apply (CUDA-event medians); and the K4 latency path on
batches of 100 / 1000 / 5000 of those documents (per-call CUDA-event medians: direct
two-launch calls, and a captured graph replayed on a resident buffer).  One JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import _wide_columns_case
    from paper_2205_07307_b200 import Model
    from time_kernels import timeit
    n = 1_000_000
    case = _wide_columns_case(4096, n_trees=10000)
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal((n, case.x.shape[1]), dtype=np.float32)).cuda()
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    out = torch.empty(n, device="cuda")
    bins = m.binarize(x)
    res = {"workload": "1,950 factors (all used), 10,000 depth-6 trees, 1 M docs U N(0,1)",
           "info": {k: m.info[k] for k in ("bins_tile_docs", "n_columns", "stages_fused", "smem_fused",
                                           "trees_per_chunk")},
           "fused_ms": timeit(lambda: m.score(x, out=out), 10),
           "binarize_ms": timeit(lambda: m.binarize(x, out=bins), 10),
           "apply_ms": timeit(lambda: m.apply(bins, n, out=out), 10)}
    res["fused_docs_per_s"] = n / (res["fused_ms"] / 1e3)
    lat = {}
    for B in (100, 1000, 5000):
        xb = x[:B].contiguous()
        ws = m.latency_workspace(B)
        ob = torch.empty(B, device="cuda")
        e = {"direct_us": timeit(lambda: m.score_latency(xb, ws, out=ob), 200) * 1e3,
             "fused_us": timeit(lambda: m.score(xb, out=ob), 200) * 1e3}
        g = torch.cuda.CUDAGraph()
        m.score_latency(xb, ws, out=ob)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            m.score_latency(xb, ws, out=ob)
        e["graph_us"] = timeit(g.replay, 200) * 1e3
        lat[str(B)] = e
    res["latency_p50"] = lat
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""CUDA-event timings (median of repeats, after warm-up) of the main-path kernels on
one BASELINE config: fused odf_score, odf_binarize, odf_apply.  Honours
ODF_LIB_OVERRIDE (diagnostics / A-B builds, paper_2205_07307_b200.build.build_variant).

    python tools/time_kernels.py --config c2 [--reps 20] [--tag name]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("ODF_LIB_OVERRIDE"):  # diagnostics / A-B build (tools only)
    from paper_2205_07307_b200 import odf as _odf
    _odf.use_library(os.environ["ODF_LIB_OVERRIDE"])


def timeit(fn, reps=20, warm=5):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tag", default=os.environ.get("ODF_LIB_OVERRIDE", "product"))
    ap.add_argument("--n-docs", type=int, default=None)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    case = synth.make_case(a.config, n_docs=a.n_docs)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda()
    n = case.n_docs
    bins = m.binarize(x)
    out = torch.empty(n, device="cuda")
    res = {"config": a.config, "tag": a.tag,
           "fused_ms": timeit(lambda: m.score(x, out=out), a.reps),
           "binarize_ms": timeit(lambda: m.binarize(x, out=bins), a.reps),
           "apply_ms": timeit(lambda: m.apply(bins, n, out=out), a.reps),
           "info": {k: m.info[k] for k in ("stages_fused", "smem_fused", "trees_per_chunk", "n_columns",
                                           "bord_stride", "max_tile_docs", "stages_fused_256")}}
    if m.info["max_tile_docs"] == 256:  # both tile widths, explicitly
        for t in (128, 256):
            res[f"fused_ms_t{t}"] = timeit(lambda: m.score(x, out=out, tile_docs=t), a.reps)
            res[f"apply_ms_t{t}"] = timeit(lambda: m.apply(bins, n, out=out, tile_docs=t), a.reps)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

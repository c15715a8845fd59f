#!/usr/bin/env python
"""Serial vs pipelined fused kernel (odf_set_fused_kernel): bit-identity against each
other and the two-stage path, and CUDA-event medians, on BASELINE configs.

    python tools/pipe_probe.py [--configs c1,c2,c3,c4] [--docs N] [--reps R]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
if os.environ.get("ODF_LIB_OVERRIDE"):  # diagnostics / A-B build (tools only)
    from paper_2205_07307_b200 import odf as _odf
    _odf.use_library(os.environ["ODF_LIB_OVERRIDE"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--docs", type=int, default=None)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    from time_kernels import timeit
    for cfg in a.configs.split(","):
        case = synth.make_case(cfg, n_docs=a.docs)
        m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
        x = torch.from_numpy(case.x).cuda()
        n = case.n_docs
        res = {"config": cfg, "tag": os.path.basename(os.environ.get("ODF_LIB_OVERRIDE", "product")),
               "n_docs": n, "info": {k: m.info[k] for k in (
            "stages_pipe", "smem_pipe", "stages_pipe_256", "pipe_scratch_bytes", "trees_per_chunk",
            "stages_fused", "smem_fused")}}
        bins = m.binarize(x)
        two = m.apply(bins, n)
        outs = {}
        for k in ("serial", "pipelined"):
            if k == "pipelined" and not (m.info["stages_pipe"] or m.info["stages_pipe_256"]):
                continue
            m.set_fused_kernel(k)
            outs[k] = m.score(x)
            torch.cuda.synchronize()
            res[k + "_ms"] = timeit(lambda: m.score(x), a.reps)
        ref = two.cpu().numpy().view(np.uint32)
        res["identical"] = {k: bool(np.array_equal(v.cpu().numpy().view(np.uint32), ref)) for k, v in outs.items()}
        print(json.dumps(res), flush=True)
        m.close()


if __name__ == "__main__":
    main()

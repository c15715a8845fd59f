"""Run each CUDA-path kernel a few times on a BASELINE config (for ncu / nsys captures).

    python tools/prof_kernels.py --config c2 --iters 3 [--only fused|binarize|apply|all]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("ODF_LIB_OVERRIDE"):  # diagnostics / A-B build (tools only)
    from paper_2205_07307_b200 import odf as _odf
    _odf.use_library(os.environ["ODF_LIB_OVERRIDE"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--only", default="all")
    ap.add_argument("--n-docs", type=int, default=None)
    ap.add_argument("--tile-docs", type=int, default=0, help="128 / 256 (0: automatic)")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    case = synth.make_case(a.config, n_docs=a.n_docs)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    print(m.info, flush=True)
    x = torch.from_numpy(case.x).cuda()
    n = case.n_docs
    out = torch.empty(n, device="cuda")
    bins = torch.empty(m.bins_bytes(n), dtype=torch.uint8, device="cuda")
    for _ in range(a.iters):
        if a.only in ("all", "fused"):
            m.score(x, out=out, tile_docs=a.tile_docs)
        if a.only in ("all", "binarize", "apply"):
            m.binarize(x, out=bins)
        if a.only in ("all", "apply"):
            m.apply(bins, n, out=out, tile_docs=a.tile_docs)
    torch.cuda.synchronize()
    print("done", flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Compare the two binarized formats of the north_star on one config (default c2):
uint8 bins (7-bit code columns, SWAR leaf-index assembly; odf_apply) vs bit-packed
ordered condition words (ballot; odf_bits_from_bins + odf_apply_bits, NEXT-3).
CUDA-event timing, warm-up, median of repeats.  Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


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
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    case = synth.make_case(a.config)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda()
    n = case.n_docs
    bins = m.binarize(x)
    words = m.bits_from_bins(bins, n)
    out = torch.empty(n, device="cuda")
    nbytes, k = m.bits_layout(n)
    res = {"config": synth.WORKLOAD_NAMES[a.config], "n_binary_features": k,
           "bins_bytes": m.bins_bytes(n), "words_bytes": nbytes,
           "fused_ms": timeit(lambda: m.score(x, out=out)),
           "binarize_ms": timeit(lambda: m.binarize(x, out=bins)),
           "apply_u8_ms": timeit(lambda: m.apply(bins, n, out=out)),
           "bits_from_bins_ms": timeit(lambda: m.bits_from_bins(bins, n, out=words)),
           "apply_bits_ms": timeit(lambda: m.apply_bits(words, n, out=out))}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

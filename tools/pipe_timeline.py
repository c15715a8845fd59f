#!/usr/bin/env python
"""Per-tile timeline of the pipelined fused kernel (diagnostics build, ODF_DIAG=8):
medians over CTAs and tiles 1..: consumer bins wait, phase B, tile total; binarizer
tile time and border-ring waits; producer bins copy.  ODF_LIB_OVERRIDE = the build.

    ODF_LIB_OVERRIDE=build/ab/ptl.so python tools/pipe_timeline.py --config c2
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_07307_b200 import odf as _odf  # noqa: E402

_odf.use_library(os.environ["ODF_LIB_OVERRIDE"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    case = synth.make_case(a.config)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    m.set_fused_kernel("pipelined")
    x = torch.from_numpy(case.x).cuda()
    L = _odf.lib()
    for _ in range(3):
        m.score(x)
    torch.cuda.synchronize()
    L.odf_pipe_diag_clear()
    m.score(x)
    torch.cuda.synchronize()
    it = 64
    buf = np.zeros(148 * it * 128, np.uint64)
    L.odf_pipe_diag_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(148, it, 128).astype(np.float64)
    valid = d[:, :, 0] > 0
    t0 = d[:, :, 0][valid].min()
    res = {"config": a.config}

    def med(x):
        x = x[np.isfinite(x)]
        return float(np.median(x)) / 1e3 if x.size else None  # us

    cons_b = d[:, :, 1] - d[:, :, 0]
    tile_tot = d[:, 1:, 0] - d[:, :-1, 0]
    wait_bins = d[:, 1:, 0] - d[:, :-1, 2]
    binz = d[:, :, 4] - d[:, :, 3]
    prod_copy = d[:, :, 6] - d[:, :, 5]
    ok1 = valid[:, 1:] & valid[:, :-1]
    res["phase_b_us"] = med(cons_b[valid])
    res["tile_period_us"] = med(tile_tot[ok1])
    res["consumer_wait_for_bins_us"] = med(wait_bins[ok1])
    res["binarizer_tile_us"] = med(binz[d[:, :, 4] > 0])
    res["binarizer_border_wait_us"] = med(d[:, :, 8][d[:, :, 4] > 0])
    res["binarizer1_border_wait_us"] = med(d[:, :, 10][d[:, :, 4] > 0])
    res["issue_wait_us"] = med(d[:, :, 9][d[:, :, 4] > 0])
    res["producer_copy_us"] = med(prod_copy[d[:, :, 6] > 0])
    res["first_bins_ready_us"] = med(d[:, 0, 0] - t0)
    res["last_tile_end_us"] = float((d[:, :, 2].max(1) - t0).max()) / 1e3
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

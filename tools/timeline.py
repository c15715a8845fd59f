#!/usr/bin/env python
"""Per-warp phase timeline of the fused kernel (diagnostics build with ODF_DIAG=8,
loaded via ODF_LIB_OVERRIDE): for each (CTA, tile) the consumer warps record the
%globaltimer at tile start, phase-A done, phase-B start (after the barrier),
phase-B done and tile end, plus the time they spent waiting on ring-slot
mbarriers in each phase.  Prints averages per tile in microseconds.

    ODF_LIB_OVERRIDE=build/diag/libodf_t8.so python tools/timeline.py --config c2
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("ODF_LIB_OVERRIDE"):  # diagnostics / A-B build (tools only)
    from paper_2205_07307_b200 import odf as _odf
    _odf.use_library(os.environ["ODF_LIB_OVERRIDE"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="fused", choices=["fused", "apply", "binarize"])
    a = ap.parse_args()
    import torch
    import synth
    from paper_2205_07307_b200 import Model, odf
    case = synth.make_case(a.config)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda()
    n = case.n_docs
    out = torch.empty(n, device="cuda")
    bins = m.binarize(x)
    L = odf.lib()
    run = {"fused": lambda: m.score(x, out=out), "apply": lambda: m.apply(bins, n, out=out),
           "binarize": lambda: m.binarize(x, out=bins)}[a.mode]
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    L.odf_diag_clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    KIT = 64
    buf = np.zeros(148 * KIT * 16 * 8, np.uint64)
    L.odf_diag_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(148, KIT, 16, 8).astype(np.float64)
    valid = d[:, :, :, 4] > 0
    t0 = d[:, :, :, 0][valid].min()
    tend = d[:, :, :, 4][valid].max()
    ok = valid.all(axis=2)  # (cta, it) with all 16 warps recorded
    dd = d[ok]  # [n_tiles, 16, 8]
    us = lambda v: float(np.mean(v) / 1e3)
    res = {
        "config": a.config, "mode": a.mode, "kernel_ms_event": e0.elapsed_time(e1),
        "span_ms": (tend - t0) / 1e6, "tiles": int(ok.sum()),
        "tile_us": us(dd[:, :, 4].max(1) - dd[:, :, 0].min(1)),
        "phaseA_us_mean_warp": us(dd[:, :, 1] - dd[:, :, 0]),
        "phaseA_us_last_warp": us(dd[:, :, 1].max(1) - dd[:, :, 0].min(1)),
        "phaseA_imbalance_us": us(dd[:, :, 1].max(1) - dd[:, :, 1].min(1)),
        "barrier_A_to_B_us": us(dd[:, :, 2].max(1) - dd[:, :, 1].max(1)),
        "phaseB_us_mean_warp": us(dd[:, :, 3] - dd[:, :, 2]),
        "phaseB_imbalance_us": us(dd[:, :, 3].max(1) - dd[:, :, 3].min(1)),
        "finish_us": us(dd[:, :, 4].max(1) - dd[:, :, 3].max(1)),
        "waitA_us_mean_warp": us(dd[:, :, 5]),
        "waitB_us_mean_warp": us(dd[:, :, 6]),
        "first_tile_start_spread_us": float((d[:, 0, :, 0][valid[:, 0, :]].max() - t0) / 1e3),
        "last_tile_end_spread_us": float((tend - np.max(np.where(valid, d[:, :, :, 4], 0), axis=(1, 2)).min()) / 1e3),
    }
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

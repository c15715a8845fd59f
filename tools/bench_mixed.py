#!/usr/bin/env python
"""NEXT-2: a production-shaped mixed-height forest (154,995 of 155,100 trees
of depth 6, the rest of heights 0..8) imported in the paper's layout, scored with
odf_score_u64 (fused, exact u64 sums) per height segment and in the padded
uniform-depth form; CUDA-event medians.  Scaled: 1,000,000 documents x 1,000
factors U(0,1), 80 binary features per factor (155,377 over 1,950), and
10,000 trees: 9,990 of depth 6, 3 of depth 8, 1 of depth 7, 1 each of depths 0..5.
Also the K4 latency path (odf_score_latency_u64) on batches of 100 / 1000 / 5000 of
those documents against the fused launch (CUDA-event medians, sums checked equal).

    python tools/bench_mixed.py [--docs N] [--reps R]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    import synth
    from bench import ClockSampler
    from paper_2205_07307_b200 import Model
    from time_kernels import timeit

    F = 1000
    stc = [1, 1, 1, 1, 1, 1, 9990, 1, 3]
    pm = synth.paper_model(168, F, 80 * F, stc)
    g = np.random.default_rng(168)
    x = torch.from_numpy(g.random((a.docs, F), dtype=np.float32)).cuda()
    res = {"workload": f"P:168-shaped mixed forest, {a.docs} docs x {F} factors, stc {stc}",
           "n_trees": int(sum(stc)), "n_binary": int(pm.thresholds.size)}
    sums = {}
    with ClockSampler(torch.cuda.current_device()) as clk:
        for pad in (False, True):
            m = Model.from_paper(pm.n_features, pm.group_factor, pm.group_count, pm.thresholds,
                                 pm.stc, pm.cond_indices, pm.leaves, pad_heights=pad)
            key = "padded" if pad else "per_height"
            sums[key] = m.score_u64(x)[0].cpu().numpy()
            res[key + "_ms"] = timeit(lambda: m.score_u64(x), a.reps)
            res[key + "_docs_per_s"] = a.docs / (res[key + "_ms"] / 1e3)
            if not pad:  # the K4 latency path on small batches of the same model (exact u64)
                lat = {}
                for B in (100, 1000, 5000):
                    xb = x[:B].contiguous()
                    ws = m.latency_workspace(B)
                    want = m.score_u64(xb)[0]
                    got = m.score_latency_u64(xb, ws)[0]
                    lat[str(B)] = {"k4_us": timeit(lambda: m.score_latency_u64(xb, ws), 200) * 1e3,
                                   "fused_us": timeit(lambda: m.score_u64(xb), 200) * 1e3,
                                   "identical": bool(torch.equal(got, want))}
                res["latency_p50_per_height"] = lat
            m.close()
        # reference: the same 10,000 trees all at depth 6 (the cost floor of this mix)
        pm6 = synth.paper_model(168, F, 80 * F, [0] * 6 + [sum(stc)])
        m = Model.from_paper(pm6.n_features, pm6.group_factor, pm6.group_count, pm6.thresholds,
                             pm6.stc, pm6.cond_indices, pm6.leaves)
        res["uniform_depth6_ms"] = timeit(lambda: m.score_u64(x), a.reps)
        m.close()
    res["sums_identical"] = bool(np.array_equal(sums["per_height"], sums["padded"]))
    res["speedup_per_height_vs_padded"] = res["padded_ms"] / res["per_height_ms"]
    res["clocks"] = clk.summary()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

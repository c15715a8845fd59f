#!/usr/bin/env python
"""Config c5 latency sweep: per-query p50/p99 of the K4 latency path (odf_score_latency).

A 1,000,000-document pool (config-2 factor mix, 1,000 factors) is resident in HBM;
query q of batch size B scores the contiguous documents [o_q, o_q + B) against the
5,000-tree depth-6 forest.  For each B in {100, 1000, 5000}: Q queries
(default 10,000) are issued

  * isolated: one stream, each query timed alone with CUDA events (device latency);
  * loaded:   round-robin over S streams (default 4), per-query event deltas and the
              wall-clock throughput (queries/s) of the whole batch of queries;

and the single-launch fused odf_score is timed the same way for comparison.  The
oracle checks a seeded 1% of the queries of each B (tolerance parity).
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pct(a, q):
    return float(np.percentile(np.asarray(a), q))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=10000)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--pool-docs", type=int, default=1_000_000)
    ap.add_argument("--batches", default="100,1000,5000")
    ap.add_argument("--check-frac", type=float, default=0.01)
    a = ap.parse_args()
    import torch

    import synth
    from paper_2205_07307_b200 import Model

    case = synth.make_case("c5", n_docs=a.pool_docs)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda()
    res = {"metric": "per-query latency (c5)", "unit": "us", "config": {
        "workload": synth.WORKLOAD_NAMES["c5"], "pool_docs": case.n_docs,
        "n_trees": case.n_trees, "depth": case.depth, "queries": a.queries,
        "streams": a.streams}, "batches": {}}
    tol = 1e-5 * np.abs(case.leaf_values.astype(np.float64)).reshape(-1, 64).max(1).sum()
    for B in [int(b) for b in a.batches.split(",")]:
        offs = synth.latency_queries(5, case.n_docs, B, a.queries)
        streams = [torch.cuda.Stream() for _ in range(a.streams)]
        wss = [m.latency_workspace(B) for _ in streams]
        outs = [torch.empty(B, device="cuda") for _ in streams]
        out1 = torch.empty(B, device="cuda")
        ws1 = m.latency_workspace(B)
        # warm-up
        for o in offs[:50]:
            m.score_latency(x[o:o + B], ws1, out=out1)
            m.score(x[o:o + B], out=out1)
        torch.cuda.synchronize()
        entry = {}
        for name, fn in (("latency_path", lambda q, s, w, o: m.score_latency(q, w, out=o, stream=s)),
                         ("fused", lambda q, s, w, o: m.score(q, out=o, stream=s))):
            # isolated
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            iso = []
            cur = torch.cuda.current_stream()
            for o in offs[: min(len(offs), 2000)]:
                e0.record(cur)
                fn(x[o:o + B], cur, ws1, out1)
                e1.record(cur)
                e1.synchronize()
                iso.append(e0.elapsed_time(e1) * 1000.0)
            # loaded: S streams
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in offs]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, o in enumerate(offs):
                k = i % len(streams)
                s = streams[k]
                evs[i][0].record(s)
                fn(x[o:o + B], s, wss[k], outs[k])
                evs[i][1].record(s)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            lat = [s.elapsed_time(e) * 1000.0 for s, e in evs]
            entry[name] = {"isolated_p50_us": pct(iso, 50), "isolated_p99_us": pct(iso, 99),
                           "loaded_p50_us": pct(lat, 50), "loaded_p99_us": pct(lat, 99),
                           "queries_per_s": len(offs) / wall,
                           "docs_per_s": len(offs) * B / wall}
        # oracle on a seeded subset of queries
        import oracle
        rng = np.random.default_rng(B)
        pick = rng.choice(len(offs), max(1, int(len(offs) * a.check_frac)), replace=False)
        worst = 0.0
        for i in pick[:20]:
            o = int(offs[i])
            got = m.score_latency(x[o:o + B], ws1, out=out1).cpu().numpy()
            rows = np.arange(o, o + B)
            if B > 200:
                rows = rows[rng.choice(B, 200, replace=False)]
            s64 = oracle.score_rows(case.x, rows, case.feature_index, case.thresholds,
                                    case.leaf_values, case.depth)
            worst = max(worst, float(np.abs(got[rows - o] - s64).max()))
        entry["parity"] = {"checked_queries": int(min(len(pick), 20)),
                           "sample": "seeded 1% of queries, <=20 checked, <=200 docs each",
                           "max_abs_err": worst, "tolerance": tol, "ok": bool(worst <= tol)}
        res["batches"][str(B)] = entry
    print(json.dumps(res), flush=True)
    m.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Config c5 latency sweep: per-query p50/p99 of the small-batch paths.

A 1,000,000-document pool (config-2 factor mix, 1,000 factors) is resident in HBM;
query q of batch size B scores the contiguous documents [o_q, o_q + B) against the
5,000-tree depth-6 forest.  For each B in {100, 1000, 5000}, all Q queries (default
10,000) are issued by each mode, twice:

  * isolated: one stream, each query timed alone with CUDA events;
  * loaded:   round-robin over S streams (default 4), per-query event deltas and the
              wall-clock throughput of the whole set of queries.

Modes:
  * k4_graph: the K4 latency path (odf_score_latency: binarize kernel + apply
    kernel with a programmatic dependent launch) captured once per stream in a
    CUDA graph on a fixed input buffer; per query the B documents are copied
    device-to-device into that buffer (inside the timed region) and the graph is
    replayed -- how a server with a fixed request buffer runs it;
  * k4_graph_resident: the same graph replay with the query already in the buffer
    (its copy issued before the start event): the kernels' own latency;
  * k4_direct: odf_score_latency called directly on the pool slice (two launches);
  * fused: the single-launch fused odf_score on the pool slice.

NVML SM clocks and throttle reasons are sampled during the timed loops.  The oracle
checks a seeded 1% of the queries of each B (tolerance parity; <= 20 queries,
<= 200 documents each).  Prints one JSON line.
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
    from bench import ClockSampler
    from paper_2205_07307_b200 import Model

    case = synth.make_case("c5", n_docs=a.pool_docs)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda()
    res = {"metric": "per-query latency (c5)", "unit": "us", "config": {
        "workload": synth.WORKLOAD_NAMES["c5"], "pool_docs": case.n_docs,
        "n_trees": case.n_trees, "depth": case.depth, "queries": a.queries,
        "streams": a.streams}, "batches": {}}
    tol = 1e-5 * np.abs(case.leaf_values.astype(np.float64)).reshape(-1, 64).max(1).sum()
    clk = ClockSampler(torch.cuda.current_device())
    with clk:
        for B in [int(b) for b in a.batches.split(",")]:
            offs = [int(o) for o in synth.latency_queries(5, case.n_docs, B, a.queries)]
            S = a.streams
            streams = [torch.cuda.Stream() for _ in range(S)]
            wss = [m.latency_workspace(B) for _ in range(S + 1)]
            outs = [torch.empty(B, device="cuda") for _ in range(S + 1)]
            bufs = [torch.empty((B, x.shape[1]), device="cuda") for _ in range(S + 1)]
            # one graph per stream (index S: the isolated runs' own) on its fixed buffer
            graphs = []
            for k in range(S + 1):
                bufs[k].copy_(x[:B])
                m.score_latency(bufs[k], wss[k], out=outs[k])
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    m.score_latency(bufs[k], wss[k], out=outs[k])
                graphs.append(g)
            torch.cuda.synchronize()

            def stage(q, k):  # k4_graph_resident: the query is in the buffer before timing
                bufs[k].copy_(x[offs[q]:offs[q] + B], non_blocking=True)

            def run(mode, q, k, s):
                o = offs[q]
                if mode == "k4_graph_resident":
                    graphs[k].replay()
                elif mode == "k4_graph":
                    bufs[k].copy_(x[o:o + B], non_blocking=True)
                    graphs[k].replay()
                elif mode == "k4_direct":
                    m.score_latency(x[o:o + B], wss[k], out=outs[k], stream=s)
                else:
                    m.score(x[o:o + B], out=outs[k], stream=s)

            entry = {}
            for mode in ("k4_graph", "k4_graph_resident", "k4_direct", "fused"):
                cur = torch.cuda.current_stream()
                for q in range(min(50, len(offs))):  # warm-up
                    run(mode, q, S, cur)
                torch.cuda.synchronize()
                # isolated: every query alone on one stream
                e0 = [torch.cuda.Event(enable_timing=True) for _ in offs]
                e1 = [torch.cuda.Event(enable_timing=True) for _ in offs]
                for q in range(len(offs)):
                    if mode == "k4_graph_resident":
                        stage(q, S)
                    e0[q].record(cur)
                    run(mode, q, S, cur)
                    e1[q].record(cur)
                    e1[q].synchronize()
                iso = [s.elapsed_time(e) * 1000.0 for s, e in zip(e0, e1)]
                # loaded: S streams round-robin
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for q in range(len(offs)):
                    k = q % S
                    with torch.cuda.stream(streams[k]):
                        if mode == "k4_graph_resident":
                            stage(q, k)
                        e0[q].record(streams[k])
                        run(mode, q, k, streams[k])
                        e1[q].record(streams[k])
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                lat = [s.elapsed_time(e) * 1000.0 for s, e in zip(e0, e1)]
                entry[mode] = {"isolated_p50_us": pct(iso, 50), "isolated_p99_us": pct(iso, 99),
                               "loaded_p50_us": pct(lat, 50), "loaded_p99_us": pct(lat, 99),
                               "queries_per_s": len(offs) / wall,
                               "docs_per_s": len(offs) * B / wall, "queries": len(offs)}
            # oracle on a seeded subset of queries (graph path)
            import oracle
            rng = np.random.default_rng(B)
            pick = rng.choice(len(offs), max(1, int(len(offs) * a.check_frac)), replace=False)
            worst = 0.0
            for i in pick[:20]:
                o = offs[int(i)]
                bufs[S].copy_(x[o:o + B])
                graphs[S].replay()
                got = outs[S].cpu().numpy()
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
    res["clocks"] = clk.summary()
    print(json.dumps(res), flush=True)
    m.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the oblivious-forest hot path (binarize + apply) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--shard docs|trees]
                    [--weak] [--impl ours|reference] [--secondary c2,c4|none]

One "step" = one pass of the whole hot path (the fused odf_score kernel:
binarization + leaf-index assembly + leaf gather/sum) over one
synthetic batch.  The headline workload is BASELINE.json configs[2] = c3, the
1,000,000-document config the north_star's HBM target names (1,000,000 docs x
1,000 factors, 10,000 depth-6 trees); c2 (configs[1]) and the deep forest c4
(configs[3]) are reported alongside in the same run (`secondary`, `secondary_deep`,
each with its own NVML clocks).  Inputs are resident in HBM when the timed
region starts and larger than L2 (4 GB vs 126 MB), so no L2 flush is needed.

N > 1 (torchrun, one rank per GPU, NCCL):
  --shard docs (default): strong scaling of ONE batch: rank r scores documents
      [floor(r*D/N), floor((r+1)*D/N)) with the replicated model and the step
      includes the NCCL all-gather of the scores; rank 0 checks (untimed) that
      the gathered scores are bit-identical to one GPU scoring the whole batch.
  --weak: every rank scores its own full batch (the same model, its own seeded
      documents) with no collective on the data path (weak scaling).
  --shard trees (default config c4): rank r holds trees [floor(r*T/N), ...),
      scores every document and the step includes one NCCL reduce (sum) of the
      fp32 partial scores to rank 0; rank 0 checks the tolerance.
time = max over ranks of the CUDA-event time of the K steps.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "documents/sec (and doc·trees/sec) for binarize+apply; % of HBM roofline"
SMEM_BYTES_PER_CLK = 128  # shared-memory data path per SM per clock (B200_PROFILING / B300_MICROARCH)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    def __init__(self, device: int):
        self.device = device
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _capture(cfg: str, kernel: str = "fused"):
    """This kernel's counters from the latest committed ncu --set full capture
    (profiles/rN_traffic.json, written by tools/ncu_metrics.py), or (None, None)."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            return json.load(open(path))[cfg][kernel], os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def _roofline_hbm(n_docs, n_used, kern_ms, cfg):
    """the fused path moves 4*F_used + 4 algorithmic bytes per document."""
    peak, peak_kind = _peaks()
    alg = n_docs * (4 * n_used + 4)
    achieved = alg / (kern_ms / 1000.0) / 1e9
    cap, src = _capture(cfg)
    traffic = cap.get("dram_bytes_per_launch") if cap else None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": src,
            "peak_kind": peak_kind, "kernel": "odf_main_kernel<FUSED>", "kernel_ms": kern_ms,
            "alg_bytes_per_launch": alg, "alg_bytes_per_doc": 4 * n_used + 4}


def _roofline_smem(cfg, kern_ms, num_sms, mhz):
    """The resource that binds the fused kernel: the SM's shared-memory
    data path, 128 B per SM per clock.  Bytes per launch = (shared-memory load + store
    wavefronts) x 128 B + the TMA bytes that fill shared memory (l1tex xbar->L1 read
    bytes), from the committed ncu capture of the same build, over this run's kernel time;
    peak = SMs x 128 B x the SM clock sampled during the run."""
    cap, src = _capture(cfg)
    if not cap or not mhz or "smem_ld_wavefronts" not in cap:
        return None
    wf = cap["smem_ld_wavefronts"] + cap.get("smem_st_wavefronts", 0.0)
    tma = cap.get("xbar2l1tex_bytes", 0.0)
    per_launch = wf * SMEM_BYTES_PER_CLK + tma
    achieved = per_launch / (kern_ms / 1000.0) / 1e9
    peak = num_sms * SMEM_BYTES_PER_CLK * mhz * 1e6 / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "bytes_per_launch": per_launch,
            "wavefronts_per_launch": wf, "tma_bytes_per_launch": tma,
            "issue_active": (cap.get("issue_active_pct") or 0.0) / 100.0,
            "peak_basis": f"{num_sms} SMs x 128 B/clk x {mhz:.0f} MHz (run median)",
            "source": src}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _config(cfg: str, case, ws: int, shard: str, n_docs_total: int) -> dict:
    """The workload description (identical for the reference arm and ours)."""
    import synth
    used = int(np.unique(case.feature_index).size) if case.feature_index.size else 0
    return {"workload": synth.WORKLOAD_NAMES[cfg], "n_docs": int(n_docs_total),
            "n_features": int(case.n_features), "n_trees": int(case.n_trees),
            "depth": int(case.depth), "used_features": used,
            "l2": "inputs larger than L2 (%.0f MB > 126 MB); no flush"
                  % (n_docs_total * case.x.shape[1] * 4 / 1e6),
            "parallelism": ("1 GPU" if ws == 1 else f"tree-shard x{ws} + NCCL reduce"
                            if shard == "trees" else f"doc batches x{ws}, no collective (weak)"
                            if shard == "weak" else f"doc-shard x{ws} + NCCL all-gather")}


def cpu_baseline(case, target_s: float = 10.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload:
    the first n docs (all threads), repeated over whole passes when the workload is
    shorter than the target, so the sample is about target_s of wall time."""
    import oracle
    threads = oracle.default_threads()
    n_cal = min(case.n_docs, max(threads * 4, 64))
    t0 = time.perf_counter()
    oracle.score(case.x[:n_cal], case.feature_index, case.thresholds, case.leaf_values,
                 case.depth, n_trees=case.n_trees, n_threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    want = max(n_cal, int(n_cal * (target_s - dt) / dt))
    n = min(case.n_docs, want)
    passes = max(1, min(1000, want // max(n, 1)))
    t0 = time.perf_counter()
    for _ in range(passes):
        oracle.score(case.x[:n], case.feature_index, case.thresholds, case.leaf_values,
                     case.depth, n_trees=case.n_trees, n_threads=threads)
    dt = time.perf_counter() - t0
    docs = n * passes
    return {"value": docs / dt, "unit": "docs/s", "cores": threads, "kind": "oracle",
            "sample": f"{passes} pass(es) over the first {n} of {case.n_docs} docs x all "
                      f"{case.n_trees} trees ({docs * case.n_trees:.3g} doc-trees, {dt:.1f} s wall)",
            "doc_trees_per_s": docs * case.n_trees / dt}


def run_reference(args):
    """The reference arm: the oracle (tier framing: no reference code exists), timed on
    the host cores, each step a bounded sample of the same workload."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import synth
    weak = args.weak and ws > 1 and args.shard == "docs"
    n_docs = synth.CONFIGS[args.config]["n_docs"]
    case = synth.make_case(args.config, rows=(0, min(n_docs, 65536)) if args.config != "c1" else None)
    times = []
    base = None
    per_step = max(0.25, min(args.ref_seconds, 120.0 / (args.warmup + args.steps)))
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(case, target_s=per_step)
        if i >= args.warmup:
            times.append(cb["value"])
            base = cb
    v = float(np.median(times))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "docs/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v * n_docs,
            "higher_is_better": True, "scaling": "strong" if ws > 1 and not weak else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args.config, case, ws, "weak" if weak else args.shard, n_docs),
            "doc_trees_per_s": v * case.n_trees,
            "cpu_baseline": {"value": v, "unit": "docs/s", "cores": base["cores"],
                             "kind": "oracle", "sample": base["sample"]},
            "e2e": {"value": v, "unit": "docs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _time_steps(step, steps, stream, ws, dev, clk=None):
    """K timed steps bracketed by barrier + synchronize, CUDA events on `stream`;
    returns (max over ranks of the total ms, this rank's mean per-step ms)."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ctx = clk if clk is not None else _Null()
    with ctx:
        t0.record(stream)
        for i in range(steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    per = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    return total_ms, per


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def _secondary(cfg, steps, warmup, dev, stream):
    """A second workload (default c2) on one GPU in the same run: fused odf_score time,
    docs/s and HBM roofline fraction (no cpu_baseline / e2e)."""
    import torch
    import synth
    from paper_2205_07307_b200 import Model
    case = synth.make_case(cfg)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth,
              case.n_features, device=dev.index)
    x = torch.from_numpy(case.x).to(dev)
    out = torch.empty(case.n_docs, dtype=torch.float32, device=dev)
    for _ in range(warmup):
        m.score(x, out=out, stream=stream)
    with ClockSampler(dev.index) as ck:
        total_ms, kern_ms = _time_steps(lambda: m.score(x, out=out, stream=stream), steps, stream, 1, dev)
    n_used = m.info["n_used_features"]
    clocks = ck.summary()
    res = {"workload": synth.WORKLOAD_NAMES[cfg], "value": case.n_docs * steps / (total_ms / 1e3),
           "unit": "docs/s", "ms_per_step": total_ms / steps, "steps": steps,
           "doc_trees_per_s": case.n_docs * case.n_trees * steps / (total_ms / 1e3),
           "roofline": _roofline_hbm(case.n_docs, n_used, kern_ms, cfg),
           "roofline_binding": _roofline_smem(cfg, kern_ms, m.info["num_sms"],
                                              clocks.get("sm_mhz") or ck.max_mhz or 1965),
           "gpu_launches": steps * m.score_launches(case.n_docs),
           "clocks": clocks}
    m.close()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    # --dist-backend gloo (tests only): the multi-rank code path on a one-GPU box, every
    # rank on cuda:0 (a functional check of the sharding, collectives and checks; the
    # timing of such a run means nothing)
    local = local % max(1, torch.cuda.device_count())
    if ws > 1 and args.dist_backend == "gloo":
        dist.init_process_group("gloo")
    elif ws > 1:
        # NCCL's communicator-init lines (nranks, transports) on stderr, so the one
        # JSON line stays alone on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        probe = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(probe)  # creates the communicator now
        if rank == 0:
            try:
                v = torch.cuda.nccl.version()
                v = ".".join(map(str, v)) if isinstance(v, (tuple, list)) else str(v)
            except Exception:
                v = "?"
            print(f"[bench] NCCL {v}: communicator nranks={dist.get_world_size()} "
                  f"(all-reduce probe = {int(probe.item())})", file=sys.stderr, flush=True)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import synth
    from paper_2205_07307_b200 import Model
    from paper_2205_07307_b200.parallel import DocSharded, shard_bounds, tree_shard

    tree_mode = args.shard == "trees"
    weak = args.weak and ws > 1 and not tree_mode  # every rank its own batch, no collective
    D = synth.CONFIGS[args.config]["n_docs"]
    if tree_mode or ws == 1 or weak:
        lo, hi = 0, D
    else:
        lo, hi = shard_bounds(D, ws, rank)
    # rank 0 of a doc-sharded run also holds the whole batch for the bit-identity check
    full_rows = ws == 1 or tree_mode or weak or rank == 0
    case = synth.make_case(args.config, rows=None if full_rows else (lo, hi))
    if weak and rank > 0:  # the same model, rank r's own seeded batch of D documents
        case.x = synth.ranking_factors(synth.CONFIGS[args.config]["seed"] + 7919 * rank, D,
                                       case.n_features, ld=case.x.shape[1])
    if tree_mode:
        fi, th, lv, _ = tree_shard(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                                   ws, rank)
        model = Model(fi, th, lv, case.depth, case.n_features, device=local)
    else:
        model = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                      case.n_features, device=local)
    info = model.info
    off = 0 if full_rows else lo  # case.x holds rows [off, ...) of the batch
    x_host = case.x[lo - off:hi - off]
    x = torch.from_numpy(np.ascontiguousarray(x_host)).to(dev)
    n = x.shape[0]
    launches_per_step = model.score_launches(n)  # 2 when the last wave runs as a second grid
    out = torch.empty(n, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ds = DocSharded(lambda t: model.score(t))
    m_pad = DocSharded.padded_size(D, ws)
    loc_pad = torch.zeros(m_pad, dtype=torch.float32, device=dev)
    all_pad = torch.empty(m_pad * ws, dtype=torch.float32, device=dev)

    def step():
        if tree_mode:
            model.score(x, out=out, stream=stream)
            if ws > 1:  # one NCCL reduce (sum) of the fp32 partial scores to rank 0
                dist.reduce(out, dst=0, op=dist.ReduceOp.SUM)
        elif ws > 1 and not weak:  # this rank's documents, then the NCCL all-gather of the scores
            model.score(x, out=loc_pad[:n], stream=stream)
            ds.gather_into(loc_pad, all_pad)
        else:
            model.score(x, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    with ClockSampler(local) as clk:
        total_ms, step_ms = _time_steps(step, args.steps, stream, ws, dev, clk)

    # the fused kernel alone (one launch per step; the collective excluded) for the rooflines
    kern_ms = step_ms
    if ws > 1:
        _, kern_ms = _time_steps(lambda: model.score(x, out=out, stream=stream),
                                 max(3, min(args.steps, 50)), stream, 1, dev)

    # ---- correctness of the sharded result (untimed) ----
    check = None
    if ws > 1 and not weak:
        torch.cuda.synchronize()
        if tree_mode:
            step()
            torch.cuda.synchronize()
        if rank == 0:
            if tree_mode:
                full = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                             case.n_features, device=local)
                ref = full.score(x)
                tol = 1e-5 * float(np.abs(case.leaf_values.astype(np.float64))
                                   .reshape(case.n_trees, -1).max(1).sum())
                err = float((out - ref).abs().max().item())
                check = {"kind": "tree-shard sum vs one GPU", "max_abs_err": err, "tol": tol,
                         "ok": err <= tol}
                full.close()
            else:
                ref = model.score(torch.from_numpy(case.x).to(dev))
                got = ds.unpad(all_pad, D)
                same = bool(torch.equal(got.view(torch.int32), ref.view(torch.int32)))
                check = {"kind": "doc-shard gather vs one GPU, whole batch", "bit_identical": same}

    # ---- two-stage path (binarize + apply), one GPU, reported alongside ----
    tb = ta = None
    if ws == 1:
        bins = torch.empty(model.bins_bytes(n), dtype=torch.uint8, device=dev)
        for _ in range(max(1, args.warmup)):
            model.binarize(x, out=bins, stream=stream)
            model.apply(bins, n, out=out, stream=stream)
        torch.cuda.synchronize()
        k2 = max(1, min(args.steps, 20))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tb = ta = 0.0
        for _ in range(k2):
            ev[0].record(stream)
            model.binarize(x, out=bins, stream=stream)
            ev[1].record(stream)
            model.apply(bins, n, out=out, stream=stream)
            ev[2].record(stream)
            torch.cuda.synchronize()
            tb += ev[0].elapsed_time(ev[1])
            ta += ev[1].elapsed_time(ev[2])
        tb /= k2
        ta /= k2
        del bins

    # ---- end to end through the public API from pinned host memory ----
    xh = torch.from_numpy(np.ascontiguousarray(x_host)).pin_memory()
    if ws > 1 and not tree_mode and not weak:
        sh = torch.empty(m_pad * ws, dtype=torch.float32).pin_memory()
    else:
        sh = torch.empty(n, dtype=torch.float32).pin_memory()

    def e2e_step():
        if ws > 1 and not weak:  # H2D of this rank's inputs, score, collective, D2H on rank 0
            x.copy_(xh, non_blocking=True)
            step()
            if rank == 0:
                sh.copy_(out if tree_mode else all_pad, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        else:  # odf_score_host: chunked H2D / score / D2H over two streams
            model.score_host(xh, out=sh, chunk_docs=args.e2e_chunk)

    e2e_step()
    k_e2e = max(1, min(args.steps, args.e2e_steps))
    if ws > 1:
        dist.barrier()
    t_e = time.perf_counter()
    for _ in range(k_e2e):
        e2e_step()
    e2e_s = time.perf_counter() - t_e
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # bytes over all ranks: doc sharding copies each document once, tree sharding every
    # document to every rank; the result read back is the [D] score vector on rank 0
    h2d = int(D * x_host.shape[1] * 4) * (ws if tree_mode or weak else 1)
    d2h = int(D * 4) * (ws if weak else 1)

    if rank == 0:
        docs_total = D * args.steps * (ws if weak else 1)
        value = docs_total / (total_ms / 1000.0)
        mhz = clk.summary().get("sm_mhz") or clk.max_mhz
        line = {
            "metric": METRIC, "value": value, "unit": "docs/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if ws > 1 and not weak else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(args.config, case, ws, "weak" if weak else args.shard, D),
            "path": "fused odf_score (one launch per step)" +
                    (" + NCCL reduce" if tree_mode and ws > 1 else
                     " + NCCL all-gather" if ws > 1 and not weak else ""),
            "doc_trees_per_s": value * case.n_trees,
            "roofline": _roofline_hbm(n, info["n_used_features"], kern_ms, args.config),
            "roofline_binding": _roofline_smem(args.config, kern_ms, info["num_sms"], mhz),
            "e2e": {"value": D * (ws if weak else 1) * k_e2e / e2e_s, "unit": "docs/s",
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": k_e2e,
                    "path": "odf_score_host (pinned host memory, chunked H2D/score/D2H)"
                            + (" on every rank" if weak else "")
                            if ws == 1 or weak else "H2D + odf_score + NCCL collective + D2H on rank 0"},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk.summary(),
            "model": {k: info[k] for k in ("n_split_features", "n_columns", "trees_per_chunk",
                                           "stages_fused", "smem_fused", "total_borders",
                                           "max_borders")},
        }
        if ws > 1:
            line["per_rank_docs"] = n
            line["check"] = check
            line["fused_kernel_ms_rank0"] = kern_ms
        if tb is not None:
            # binarise-only moves 4*F_used + F_used algorithmic bytes per
            # document (factors read, uint8 bins written), apply-only F_used + 4
            hbm, _ = _peaks()
            nu = info["n_used_features"]
            line["two_stage"] = {"binarize_ms": tb, "apply_ms": ta,
                                 "docs_per_s": n / ((tb + ta) / 1000.0),
                                 "binarize_hbm_frac": n * 5 * nu / (tb / 1e3) / 1e9 / hbm,
                                 "binarize_alg_bytes_per_doc": 5 * nu}
        sec = [c for c in args.secondary.split(",") if c and c != "none" and c != args.config]
        if ws == 1 and sec:
            del x
            torch.cuda.empty_cache()
            # the first (c2) is `secondary`; the deep forest (c4) `secondary_deep`, fewer steps
            line["secondary"] = _secondary(sec[0], max(3, min(args.steps * 10, 500)),
                                           max(3, args.warmup), dev, stream)
            for c in sec[1:]:
                torch.cuda.empty_cache()
                line["secondary_deep" if c == "c4" else f"secondary_{c}"] = _secondary(
                    c, max(3, min(args.steps, 20)), max(3, args.warmup), dev, stream)
        if not args.no_cpu_baseline and ws == 1:  # the oracle baseline: rank 0 at N=1 only
            line["cpu_baseline"] = cpu_baseline(case, target_s=args.ref_seconds)
        print(json.dumps(line), flush=True)
    model.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4"],
                    help="default c3 (c4 with --shard trees)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="docs", choices=["docs", "trees"],
                    help="multi-GPU: document sharding of one batch + all-gather, or tree "
                         "sharding + NCCL reduce of fp32 partials (both strong scaling)")
    ap.add_argument("--weak", action="store_true",
                    help="multi-GPU: every rank scores its own full batch (same model, its own seed), "
                         "no collective on the data path (weak scaling)")
    ap.add_argument("--secondary", default="c2,c4",
                    help="further workloads reported in the line (comma list), or none")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk", type=int, default=65536)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: tests only (multi-rank code path on one GPU; timings meaningless)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "c4" if args.shard == "trees" else "c3"
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

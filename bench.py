#!/usr/bin/env python
"""Benchmark of the oblivious-forest hot path (binarize + apply) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" = one pass of the whole hot path (fused odf_score: binarization +
leaf-index assembly + leaf gather/sum) over one synthetic batch of the
workload (BASELINE.json configs[1] = c2 by default: 100,000 docs x 1,000
factors, 2,000 depth-6 trees).  Inputs are resident in HBM when the timed
region starts and are larger than L2 (400 MB vs 126 MB), so no L2 flush is
needed between steps.  N > 1 (torchrun, one rank per GPU, NCCL): every rank
scores its own batch (document sharding, weak scaling, no data-path
collective); time = max over ranks of the CUDA-event time.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "documents/sec (and doc·trees/sec) for binarize+apply; % of HBM roofline"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def _ncu_fused(cfg: str):
    """The fused kernel's entry of the latest committed ncu capture (profiles/rN_traffic.json)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            return json.load(open(path))[cfg]["fused"], os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def _traffic(cfg: str):
    """dram read+write bytes per launch of the fused kernel from the latest committed
    ncu --set full capture (profiles/rN_traffic.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            return (int(json.load(open(path))[cfg]["fused"]["dram_bytes_per_launch"]),
                    os.path.relpath(path, ROOT))
        except Exception:
            continue
    return None, None


def _binding(cfg: str, kern_ms: float, info: dict, clk) -> dict | None:
    """The resources that bind the fused kernel (profiles/README.md):
    shared-memory / L1 pipe wavefronts per launch from the committed ncu capture,
    over this run's mean kernel time, against one wavefront per SM clock; and the
    capture's instruction-issue utilisation.  `resource` names the busier one."""
    ent, src = _ncu_fused(cfg)
    if not ent or "smem_wavefronts" not in ent:
        return None
    mhz = clk.summary().get("sm_mhz") or clk.max_mhz
    if not mhz:
        return None
    per_s = ent["smem_wavefronts"] / (kern_ms / 1000.0)
    peak = info["num_sms"] * mhz * 1e6
    smem_frac = per_s / peak
    issue_frac = (ent.get("issue_active_pct") or 0.0) / 100.0
    return {"resource": "instruction issue" if issue_frac > smem_frac else "shared-memory/L1 pipe wavefronts",
            "smem": {"achieved": per_s, "peak": peak, "unit": "wavefronts/s", "frac": smem_frac,
                     "per_launch": ent["smem_wavefronts"],
                     "peak_basis": "1 wavefront per SM per clock x SMs x SM clock during the run"},
            "issue": {"frac": issue_frac, "basis": "ncu smsp__issue_active (fraction of active cycles)"},
            "source": src}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _workload(cfg: str, rank: int):
    import synth
    from synth import CONFIGS
    base = CONFIGS[cfg]
    # the model is the config's; rank r scores its own batch (seed offset = rank)
    case = synth.make_case(cfg)
    if rank > 0:
        case.x = synth.ranking_factors(base["seed"] + 7919 * rank, case.n_docs, case.n_features)
    return case


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
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import synth
    case = _workload(args.config, 0)
    times = []
    base = None
    # each step is a bounded sample; the whole W+K run stays within ~2 minutes
    per_step = max(0.25, min(args.ref_seconds, 120.0 / (args.warmup + args.steps)))
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(case, target_s=per_step)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(cb["value"])
            base = cb
    v = float(np.median(times))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "docs/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v * case.n_docs,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": synth.WORKLOAD_NAMES[args.config], "n_docs": case.n_docs,
                       "n_features": case.n_features, "n_trees": case.n_trees,
                       "depth": case.depth, "parallelism": "host threads"},
            "cpu_baseline": {"value": v, "unit": "docs/s", "cores": base["cores"],
                             "kind": "oracle", "sample": base["sample"]},
            "e2e": {"value": v, "unit": "docs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import synth
    from paper_2205_07307_b200 import Model

    tree_shard = args.shard == "trees"
    case = _workload(args.config, 0 if tree_shard else rank)
    if tree_shard:  # rank r holds trees [r*T/W, (r+1)*T/W) and scores every document
        from paper_2205_07307_b200.parallel import tree_shard as _shard
        fi, th, lv, _ = _shard(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                               ws, rank)
        model = Model(fi, th, lv, case.depth, case.n_features, device=local)
    else:
        model = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth,
                      case.n_features, device=local)
    info = model.info
    x = torch.from_numpy(case.x).to(dev)
    n = case.n_docs
    out = torch.empty(n, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        model.score(x, out=out, stream=stream)
        if tree_shard and ws > 1:  # one NCCL all-reduce of the fp32 partial scores
            dist.all_reduce(out, op=dist.ReduceOp.SUM)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    kern_ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- two-stage path (binarize + apply), reported alongside ----
    bins = torch.empty(model.bins_bytes(n), dtype=torch.uint8, device=dev)
    for _ in range(max(1, args.warmup)):
        model.binarize(x, out=bins, stream=stream)
        model.apply(bins, n, out=out, stream=stream)
    torch.cuda.synchronize()
    k2 = max(1, min(args.steps, 200))
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

    # ---- end to end through the public API from pinned host memory ----
    xh = torch.from_numpy(case.x).pin_memory()
    sh = torch.empty(n, dtype=torch.float32).pin_memory()

    def e2e_step():
        if tree_shard and ws > 1:  # H2D, shard scores, NCCL all-reduce, D2H
            x.copy_(xh, non_blocking=True)
            step()
            sh.copy_(out, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        else:
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

    line = None
    if rank == 0:
        peak, peak_kind = _peaks()
        docs_total = n * args.steps * (1 if tree_shard else ws)
        value = docs_total / (total_ms / 1000.0)
        alg_bytes = n * (4 * info["n_used_features"] + 4)  # fused = 4*F_used + 4
        achieved = alg_bytes / (kern_ms / 1000.0) / 1e9
        traffic, traffic_src = (args.traffic, "--traffic") if args.traffic else _traffic(args.config)
        line = {
            "metric": METRIC, "value": value, "unit": "docs/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if tree_shard else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": synth.WORKLOAD_NAMES[args.config], "n_docs": n,
                       "n_features": case.n_features, "n_trees": case.n_trees,
                       "depth": case.depth, "used_features": info["n_used_features"],
                       "path": "fused odf_score",
                       "l2": "inputs larger than L2 (%.0f MB > 126 MB); no flush" % (case.x.nbytes / 1e6),
                       "parallelism": (f"tree-shard x{ws} + NCCL all-reduce" if tree_shard
                                       else f"doc-shard x{ws}")},
            "doc_trees_per_s": value * case.n_trees,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind, "kernel": "odf_main_kernel<FUSED,%d>" % case.depth,
                         "kernel_ms": kern_ms, "alg_bytes_per_launch": alg_bytes},
            "binding": _binding(args.config, kern_ms, info, clk),
            "two_stage": {"binarize_ms": tb, "apply_ms": ta,
                          "docs_per_s": n / ((tb + ta) / 1000.0)},
            "e2e": {"value": n * k_e2e / e2e_s, "unit": "docs/s",
                    "h2d_bytes_per_step": int(case.x.nbytes), "d2h_bytes_per_step": int(n * 4)},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "model": {k: info[k] for k in ("n_split_features", "n_columns", "trees_per_chunk",
                                           "borders_in_smem", "stages_fused", "smem_fused",
                                           "total_borders", "max_borders")},
        }
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
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="docs", choices=["docs", "trees"],
                    help="multi-GPU: document sharding (weak scaling) or tree sharding + NCCL "
                         "all-reduce of fp32 partials (strong scaling)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-chunk", type=int, default=16384)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

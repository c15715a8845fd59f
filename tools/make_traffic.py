"""Assemble profiles/rN_traffic.json (read by bench.py for `roofline.traffic` and
`roofline_binding`) from the ncu reports that tools/r2_evidence.sh TAG ncu writes:

    python tools/make_traffic.py TAG OUT.json

TAG_{c3,c2,c4}_fused.ncu-rep and TAG_c3_binarize.ncu-rep under gpurun_out/.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def metrics(rep):
    """Counters of the report's launches, summed (odf_score may run a second grid for a
    partly filled last wave: both belong to one launch of the fused path)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_metrics.py"), rep, "--all"],
                         capture_output=True, text=True, check=True).stdout
    ms = json.loads(out)
    m = dict(ms[0])
    for extra in ms[1:]:
        for k in ("duration_ms", "dram_read", "dram_write", "xbar2l1tex_bytes", "smem_ld_wavefronts",
                  "smem_st_wavefronts", "smem_bank_conflicts_ld", "warp_instructions"):
            if extra.get(k) is not None and m.get(k) is not None:
                m[k] += extra[k]
        m["kernel"] += " + " + extra["kernel"][:40]
    return {
        "kernel": m["kernel"],
        "dram_bytes_per_launch": int(m["dram_read"] + m["dram_write"]),
        "ncu_duration_ms": m["duration_ms"],
        "xbar2l1tex_bytes": m.get("xbar2l1tex_bytes"),
        "smem_ld_wavefronts": m.get("smem_ld_wavefronts"),
        "smem_st_wavefronts": m.get("smem_st_wavefronts"),
        "smem_bank_conflicts_ld": m.get("smem_bank_conflicts_ld"),
        "warp_instructions": m.get("warp_instructions"),
        "issue_active_pct": m.get("issue_active_pct"),
        "l1tex_pct": m.get("l1tex_pct"),
        "sm_cycles_avg": m.get("sm_cycles"),
    }


def main():
    tag, out = sys.argv[1], sys.argv[2]
    d = os.path.join(ROOT, "gpurun_out")
    res = {cfg: {"fused": metrics(os.path.join(d, f"{tag}_{cfg}_fused.ncu-rep"))} for cfg in ("c3", "c2", "c4")}
    res["c3"]["binarize"] = metrics(os.path.join(d, f"{tag}_c3_binarize.ncu-rep"))
    res["source"] = (f"ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 1 "
                     f"of tools/prof_kernels.py --config CFG --iters 1 --only fused (binarize: --only binarize) "
                     f"(tools/r2_evidence.sh {tag} ncu; tools/make_traffic.py)")
    res["units"] = ("bytes / wavefronts / warp instructions per launch; ncu_duration_ms under the profiler "
                    "(cold, serialised)")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v["fused"]["ncu_duration_ms"] for k, v in res.items() if isinstance(v, dict) and "fused" in v}))


if __name__ == "__main__":
    main()

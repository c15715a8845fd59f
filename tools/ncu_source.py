"""Summarise an ncu report's SASS source page: per-instruction executed counts and stall samples.

    python tools/ncu_source.py REPORT.ncu-rep [kernel-id] [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kid = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kid is not None:
        args += ["--print-kernel-base", "function", "--launch-skip", kid, "--launch-count", "1"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    lines = out.splitlines()
    # first line: kernel name, then CSV
    print(lines[0][:150])
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    data = rows[1:]
    def f(r, k):
        try:
            return float(r[col[k]])
        except Exception:
            return 0.0
    tot_exec = sum(f(r, "Instructions Executed") for r in data)
    tot_samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"instructions executed (warp-level): {tot_exec:.4g}; stall samples {tot_samp:.4g}")
    opc = {}
    for r in data:
        op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[col["Source"]].split()[1]
        op = op.split(".")[0]
        e = opc.setdefault(op, [0, 0])
        e[0] += f(r, "Instructions Executed")
        e[1] += f(r, "Warp Stall Sampling (All Samples)")
    print("by opcode (exec share, stall share):")
    for op, (e, s) in sorted(opc.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"  {op:10s} {e / max(tot_exec, 1):6.1%} {s / max(tot_samp, 1):6.1%}")
    print(f"top {top} instructions by stall samples:")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        print(f"  {r[col['Address']]:>6s} {f(r, 'Warp Stall Sampling (All Samples)'):7.0f} "
              f"{f(r, 'Instructions Executed'):10.0f}  {r[col['Source']][:90]}")


if __name__ == "__main__":
    main()

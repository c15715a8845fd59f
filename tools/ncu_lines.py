"""Per-CUDA-source-line summary of an ncu report (instructions executed, stall samples).

    python tools/ncu_lines.py REPORT.ncu-rep [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    ix = hdr.index("Instructions Executed")
    iw = hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows[hi + 1:]:
        if r and r[0] not in ("", "Line No"):
            try:
                lines.append((int(r[0]), r[1][:90], float(r[ix] or 0), float(r[iw] or 0)))
            except ValueError:
                pass
    tot = sum(l[2] for l in lines) or 1
    tw = sum(l[3] for l in lines) or 1
    print(f"instructions {tot:.4g}, stall samples {tw:.4g}")
    print("by stall samples:")
    for l in sorted(lines, key=lambda l: -l[3])[:top]:
        print(f"{l[0]:5d} exec {l[2] / tot:6.1%} stall {l[3] / tw:6.1%}  {l[1]}")


if __name__ == "__main__":
    main()

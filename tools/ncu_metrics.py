"""Key counters of one kernel in an ncu report (raw page), as JSON.

    python tools/ncu_metrics.py REPORT.ncu-rep [--kernel REGEX] [--all]
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "lts_bytes": "lts__t_bytes.sum",
    "xbar2l1tex_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_st_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts_ld": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smem_ld_requests": "l1tex__t_requests_pipe_lsu_mem_shared_op_ld.sum",
    "warp_instructions": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "data_bank_reads": "l1tex__data_bank_reads.sum",
    "data_bank_writes": "l1tex__data_bank_writes.sum",
    "sm_cycles": "sm__cycles_elapsed.avg",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return None


def main():
    rep = sys.argv[1]
    kre = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if kre and not re.search(kre, d.get("Kernel Name", "")):
            continue
        e = {"kernel": d.get("Kernel Name", "")[:80]}
        for k, m in KEYS.items():
            if m in d:
                v = _num(d[m])
                u = units[hdr.index(m)]
                # normalise: bytes, milliseconds, Hz
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                         "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1,
                         "msecond": 1, "s": 1e3, "second": 1e3, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
                         "Ghz": 1e9, "cycle/usecond": 1e6, "cycle/nsecond": 1e9}
                if v is not None and u in scale:
                    v *= scale[u]
                e[k] = v
        res.append(e)
    print(json.dumps(res if "--all" in sys.argv else res[0], indent=1))


if __name__ == "__main__":
    main()

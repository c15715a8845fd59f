"""SASS guard for the slot-release ordering of the apply phase (DESIGN.md §7 "Hazard
fixed in round 1").

A consumer warp hands a tree-chunk ring slot back to the producer with an mbarrier
arrive; every leaf gather it made from that slot must have completed first, or the
producer's next bulk copy can overwrite leaves still being read.  The gathers are
plain loads whose results only feed FADDs, so nothing in the PTX stops ptxas from
sinking those FADDs (and leaving the gathers in flight) below the arrive; the kernels
therefore execute a never-taken store predicated on all accumulators (Acc::pin)
before the arrive.  This test reads the SASS of the shipped library and checks, for
every fp32 fused / apply kernel, that each slot release following the apply loop is
preceded by that predicated store, and that no FADD2 of the chunk was scheduled
after the release.  It fails if a compiler change breaks the ordering the fix relies
on, without needing a GPU.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2205_07307_b200", "libodf.so")

# odf_main_kernel<MODE, DEPTH, U32=false, WIDE=false, H, DPL(, TM)>: fused (0) / apply (2)
KERNEL = re.compile(r"Function : (_ZN3odf15odf_main_kernelILi([02])ELi(\d+)ELb0ELb0ELi(\d)ELi(\d)E\S*)")
INSTR = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;")


def _sass():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(cuobjdump):
        pytest.skip("libodf.so or cuobjdump not available (run __graft_entry__.build())")
    return subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True, check=True).stdout


def _functions(text):
    out, cur, body = {}, None, []
    for line in text.splitlines():
        m = KERNEL.search(line)
        if "Function :" in line:
            if cur:
                out[cur] = body
            cur, body = (m.groups() if m else None), []
            continue
        if cur:
            i = INSTR.search(line)
            if i:
                body.append(i.group(1))
    if cur:
        out[cur] = body
    return out


def test_slot_release_after_every_gather_sum():
    funcs = _functions(_sass())
    assert funcs, "no fused / apply kernel found in the SASS"
    checked = 0
    for (name, mode, depth, halves, dpl), body in funcs.items():
        if int(depth) == 0:
            continue  # no gathers to order
        for k, ins in enumerate(body):
            # a consumer's release of a ring slot: arrive (count 1) on an empty barrier
            if "SYNCS.ARRIVE.TRANS64.A1T0" not in ins:
                continue
            window = body[max(0, k - 80):k]
            if not any(w.startswith("FADD2") or " FADD2 " in f" {w} " for w in window):
                continue  # a phase-A release: no leaf gathers before it
            last_fadd = max(i for i, w in enumerate(window) if "FADD2" in w)
            pin = [i for i, w in enumerate(window) if re.match(r"@!?P\d+\s+STS\b", w)]
            assert pin and max(pin) > last_fadd, (
                f"{name}: slot release at SASS index {k} is not preceded by the accumulator-"
                f"predicated store after the chunk's last FADD2")
            # nothing of the chunk's sums may be sunk below the release (up to the loop branch)
            for w in body[k + 1:k + 12]:
                if w.split()[0].startswith("BRA") or "BRA " in w:
                    break
                assert "FADD2" not in w, f"{name}: FADD2 scheduled after the slot release"
            checked += 1
    assert checked >= 8, f"only {checked} apply-loop slot releases found"

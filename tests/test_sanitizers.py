"""Sanitizer builds on the CPU (the paper's code builds and runs under
all sanitizers; compute-sanitizer is closed on this GPU pool).

* the oracle (oracle/odf_oracle.c) under AddressSanitizer + UndefinedBehaviorSanitizer
  and, separately, ThreadSanitizer (its scoring and fingerprints run on pthreads),
  driven by tests/sanitize/oracle_driver.c;
* the host side of the C ABI (paper_2205_07307_b200/csrc/odf_capi.cu: validation,
  the model compiler, the NEXT-2 import) under ASan + UBSan, linked against stub
  kernel launchers (tests/sanitize/kernel_stubs.cpp) and driven by
  tests/sanitize/capi_driver.cpp.  The host-side compile runs before any device
  call, so it is fully exercised without a GPU.

Every sanitizer aborts on its first report (-fno-sanitize-recover=all), so a clean
run is exit status 0 and the driver's own "ok" line.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = os.path.join(ROOT, "tests", "sanitize")
NVCC = "/usr/local/cuda/bin/nvcc"


def _run(cmd, env=None, timeout=600):
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    return r.returncode, r.stdout + r.stderr


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
@pytest.mark.parametrize("flags", [["-fsanitize=address,undefined", "-fno-sanitize-recover=all"],
                                   ["-fsanitize=thread"]], ids=["asan_ubsan", "tsan"])
def test_oracle_under_sanitizers(tmp_path, flags):
    exe = str(tmp_path / "oracle_driver")
    rc, out = _run(["gcc", "-O1", "-g", "-fno-omit-frame-pointer", *flags,
                    os.path.join(ROOT, "oracle", "odf_oracle.c"),
                    os.path.join(SAN, "oracle_driver.c"), "-o", exe, "-lpthread", "-lm"])
    assert rc == 0, out
    rc, out = _run([exe], env={"TSAN_OPTIONS": "halt_on_error=1"})
    assert rc == 0 and "oracle driver: ok" in out, out


@pytest.mark.skipif(not os.path.exists(NVCC) or shutil.which("g++") is None,
                    reason="nvcc / g++ not available")
def test_model_compiler_under_asan_ubsan(tmp_path):
    san = ["-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer"]
    capi, drv, stubs, exe = (str(tmp_path / n) for n in ("capi.o", "drv.o", "stubs.o", "capi_san"))
    # nvcc splits -Xcompiler values at commas: one flag per -Xcompiler
    xc = [a for f in ("-fsanitize=address", "-fsanitize=undefined", *san[1:]) for a in ("-Xcompiler", f)]
    rc, out = _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O1", "-g",
                    *xc, "-I", os.path.join(ROOT, "include"), "-c",
                    os.path.join(ROOT, "paper_2205_07307_b200", "csrc", "odf_capi.cu"), "-o", capi])
    assert rc == 0, out
    for src, obj in ((os.path.join(SAN, "capi_driver.cpp"), drv),
                     (os.path.join(SAN, "kernel_stubs.cpp"), stubs)):
        rc, out = _run(["g++", "-std=c++17", "-O1", "-g", *san, "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", "-c", src, "-o", obj])
        assert rc == 0, out
    rc, out = _run(["g++", *san, capi, drv, stubs, "-L/usr/local/cuda/lib64", "-lcudart_static",
                    "-ldl", "-lpthread", "-lrt", "-o", exe])
    assert rc == 0, out
    rc, out = _run([exe], env={"ASAN_OPTIONS": "detect_leaks=0"})  # the CUDA runtime's own
    assert rc == 0 and "capi driver: ok" in out, out

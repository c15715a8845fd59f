"""CPU-side checks of the boundary: the C-ABI library builds, loads, and exports
every symbol include/odf.h declares; no compute call is made without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "odf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(odf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for s in ("odf_load_model", "odf_binarize", "odf_apply", "odf_score", "odf_free_model",
              "odf_leaf_indices", "odf_index_fingerprint", "odf_bins_layout", "odf_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2205_07307_b200 import build, odf
    path = build.build()
    L = ctypes.CDLL(path)
    for s in _declared_symbols():
        assert hasattr(L, s), s
    assert set(odf.ABI_SYMBOLS) == set(_declared_symbols())
    assert odf.lib().odf_version() >= 100


def test_library_is_sm100a_and_not_fast_math():
    import subprocess
    from paper_2205_07307_b200 import build
    path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass and "UBLKCP" in sass  # TMA tensor + bulk copies are in the product
    # exact IEEE compares / adds: no flush-to-zero on FSETP or FADD
    assert not re.search(r"\b(FSETP|FADD|FSET)\S*\.FTZ", sass)
    assert "FSETP" in sass


def test_load_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2205_07307_b200 import Model, OdfError
    with pytest.raises(OdfError):
        Model(np.zeros(6, np.int32), np.zeros(6, np.float32), np.zeros(64, np.float32), 6, 4)


def test_validation_errors_precede_device_checks():
    import numpy as np
    from paper_2205_07307_b200 import Model, OdfError
    with pytest.raises(OdfError) as e:
        Model(np.zeros(6, np.int32), np.zeros(6, np.float32), np.zeros(64, np.float32), 11, 4)
    assert e.value.status == 1
    with pytest.raises(OdfError) as e:
        Model(np.array([0, 9], np.int32), np.zeros(2, np.float32), np.zeros(4, np.float32), 2, 4)
    assert e.value.status == 1 and "feature_index" in e.value.message
    with pytest.raises(OdfError) as e:
        Model(np.zeros(1, np.int32), np.array([np.nan], np.float32), np.zeros(2, np.float32), 1, 4)
    assert e.value.status == 1 and "threshold" in e.value.message
    with pytest.raises(OdfError) as e:
        Model(np.zeros(1, np.int32), np.zeros(1, np.float32), np.array([0, np.inf], np.float32), 1, 4)
    assert e.value.status == 1 and "leaf" in e.value.message

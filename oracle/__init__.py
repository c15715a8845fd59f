"""CPU oracle for oblivious-decision-forest inference -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product path
(``paper_2205_07307_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``odf_oracle.c`` (plain C, built with
gcc -O2, no -ffast-math); every arithmetic step of the method is in that file,
each function citing the PAPER.md passage it follows.  Functions pinned by
tests/test_oracle_pins.py; see DESIGN.md "Oracle and its pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "odf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def build(force: bool = False) -> str:
    """Compile odf_oracle.c into liboracle.so (gcc, -O2, IEEE semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
             "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_leaf_index.restype = _i32
        L.oracle_leaf_index.argtypes = [_f32p, _i32p, _f32p, _i32, _i64]
        L.oracle_score.restype = None
        L.oracle_score.argtypes = [_f32p, _i64, _i64, _i32p, _f32p, _f32p, _i32, _i64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_score_rows.restype = None
        L.oracle_score_rows.argtypes = [_f32p, _i64, _i64p, _i64, _i32p, _f32p, _f32p, _i32,
                                        _i64, _f64p]
        L.oracle_leaf_indices.restype = None
        L.oracle_leaf_indices.argtypes = [_f32p, _i64, _i32p, _f32p, _i32, _i64, _i64, _i64,
                                          _i64, _u16p]
        L.oracle_fingerprint.restype = None
        L.oracle_fingerprint.argtypes = [_f32p, _i64, _i64, _i32p, _f32p, _i32, _i64, _u64p,
                                         ctypes.c_int]
        L.oracle_fnv1a64.restype = ctypes.c_uint64
        L.oracle_fnv1a64.argtypes = [ctypes.c_char_p, _i64]
        L.oracle_borders.restype = _i64
        L.oracle_borders.argtypes = [_i32p, _f32p, _i64, _i32, _f32p, _i32p, _i64p]
        L.oracle_bins.restype = None
        L.oracle_bins.argtypes = [_f32p, _i64, _i64, _i32, _f32p, _i32p, _i64p, _u16p]
        L.oracle_border_index.restype = None
        L.oracle_border_index.argtypes = [_i32p, _f32p, _i64, _f32p, _i32p, _i64p, _i32p]
        L.oracle_score_u64.restype = None
        L.oracle_score_u64.argtypes = [_f32p, _i64, _i64, _i32p, _f32p, _u32p, _i32, _i64,
                                       _u64p, ctypes.c_int]
        L.oracle_finalize.restype = None
        L.oracle_finalize.argtypes = [_u64p, _i64, ctypes.c_double, ctypes.c_double, _f64p]
        L.oracle_binary_features.restype = None
        L.oracle_binary_features.argtypes = [_f32p, _i32p, _i32p, _i32, _f32p, _u8p]
        L.oracle_apply_paper.restype = None
        L.oracle_apply_paper.argtypes = [_f32p, _i64, _i64, _i32p, _i32p, _i32, _f32p, _i64,
                                         _i32p, _u32p, _u32p, _u64p]
        L.oracle_condition_words.restype = None
        L.oracle_condition_words.argtypes = [_f32p, _i64, _i64, _i32, _f32p, _i32p, _i64p, _u32p,
                                             _i64]
        L.oracle_default_threads.restype = ctypes.c_int
        L.oracle_default_threads.argtypes = []
        _lib = L
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _x2d(x):
    x = np.asarray(x)
    assert x.dtype == np.float32 and x.ndim == 2
    if not x.flags["C_CONTIGUOUS"]:
        x = np.ascontiguousarray(x)
    return x


def default_threads() -> int:
    return int(lib().oracle_default_threads())


def leaf_index(row, feature_index, thresholds, depth, t) -> int:
    """O2 for one (doc, tree)."""
    return int(lib().oracle_leaf_index(_c(row, np.float32), _c(feature_index, np.int32),
                                       _c(thresholds, np.float32), int(depth), int(t)))


def score(x, feature_index, thresholds, leaf_values, depth, n_trees=None, n_threads=0,
          n_docs=None):
    """O3: fp64 scores (and their fp32 rounding) for every row of x."""
    x = _x2d(x)
    fi = _c(feature_index, np.int32)
    thr = _c(thresholds, np.float32)
    lv = _c(leaf_values, np.float32)
    if n_trees is None:
        n_trees = lv.size >> int(depth)
    n = x.shape[0] if n_docs is None else int(n_docs)
    out64 = np.zeros(n, np.float64)
    out32 = np.zeros(n, np.float32)
    lib().oracle_score(x, n, x.shape[1], fi, thr, lv, int(depth), int(n_trees),
                       out64.ctypes.data, out32.ctypes.data, int(n_threads))
    return out64, out32


def score_rows(x, rows, feature_index, thresholds, leaf_values, depth, n_trees=None):
    """O3 on an explicit list of row indices (sampled parity at full sizes)."""
    x = _x2d(x)
    rows = _c(rows, np.int64)
    lv = _c(leaf_values, np.float32)
    if n_trees is None:
        n_trees = lv.size >> int(depth)
    out = np.zeros(rows.size, np.float64)
    lib().oracle_score_rows(x, x.shape[1], rows, rows.size, _c(feature_index, np.int32),
                            _c(thresholds, np.float32), lv, int(depth), int(n_trees), out)
    return out


def leaf_indices(x, feature_index, thresholds, depth, doc0, ndoc, tree0, ntree):
    x = _x2d(x)
    out = np.zeros((ndoc, ntree), np.uint16)
    lib().oracle_leaf_indices(x, x.shape[1], _c(feature_index, np.int32),
                              _c(thresholds, np.float32), int(depth), int(doc0), int(ndoc),
                              int(tree0), int(ntree), out)
    return out


def fingerprint(x, feature_index, thresholds, depth, n_trees, n_threads=0, n_docs=None):
    x = _x2d(x)
    n = x.shape[0] if n_docs is None else int(n_docs)
    out = np.zeros(n, np.uint64)
    lib().oracle_fingerprint(x, n, x.shape[1], _c(feature_index, np.int32),
                             _c(thresholds, np.float32), int(depth), int(n_trees), out,
                             int(n_threads))
    return out


def fnv1a64(data: bytes) -> int:
    return int(lib().oracle_fnv1a64(data, len(data)))


def borders(feature_index, thresholds, n_features):
    """O4: per-feature sorted unique borders -> (list of float32 arrays, flat, counts, offsets)."""
    fi = _c(feature_index, np.int32)
    thr = _c(thresholds, np.float32)
    flat = np.zeros(max(1, fi.size), np.float32)
    counts = np.zeros(n_features, np.int32)
    offsets = np.zeros(n_features, np.int64)
    total = lib().oracle_borders(fi, thr, fi.size, int(n_features), flat, counts, offsets)
    flat = flat[:total].copy()
    per = [flat[offsets[f]:offsets[f] + counts[f]] for f in range(n_features)]
    return per, flat, counts, offsets


def bins(x, n_features, flat, counts, offsets, n_docs=None):
    """O4: bins for all features (unused features: 0 borders -> bin 0), uint16."""
    x = _x2d(x)
    n = x.shape[0] if n_docs is None else int(n_docs)
    out = np.zeros((n, n_features), np.uint16)
    fl = _c(flat if flat.size else np.zeros(1, np.float32), np.float32)
    lib().oracle_bins(x, n, x.shape[1], int(n_features), fl, _c(counts, np.int32),
                      _c(offsets, np.int64), out)
    return out


def border_index(feature_index, thresholds, flat, counts, offsets):
    fi = _c(feature_index, np.int32)
    out = np.zeros(fi.size, np.int32)
    fl = _c(flat if flat.size else np.zeros(1, np.float32), np.float32)
    lib().oracle_border_index(fi, _c(thresholds, np.float32), fi.size, fl,
                              _c(counts, np.int32), _c(offsets, np.int64), out)
    return out


def condition_words(x, n_features, flat, counts, offsets):
    """NEXT-3: ordered bit format, words[g, kb] with bit i = condition of doc 32g+i."""
    x = _x2d(x)
    n_bin = int(np.asarray(counts).sum())
    g = (x.shape[0] + 31) // 32
    out = np.zeros((g, max(n_bin, 1)), np.uint32)
    fl = _c(flat if flat.size else np.zeros(1, np.float32), np.float32)
    lib().oracle_condition_words(x, x.shape[0], x.shape[1], int(n_features), fl,
                                 _c(counts, np.int32), _c(offsets, np.int64), out, max(n_bin, 1))
    return out[:, :n_bin]


def score_u64(x, feature_index, thresholds, leaf_values_u32, depth, n_trees=None, n_threads=0):
    """NEXT-1: u32 leaves summed in u64."""
    x = _x2d(x)
    lv = _c(leaf_values_u32, np.uint32)
    if n_trees is None:
        n_trees = lv.size >> int(depth)
    out = np.zeros(x.shape[0], np.uint64)
    lib().oracle_score_u64(x, x.shape[0], x.shape[1], _c(feature_index, np.int32),
                           _c(thresholds, np.float32), lv, int(depth), int(n_trees), out,
                           int(n_threads))
    return out


def finalize(r_u64, scale, bias):
    """NEXT-1: (R - 2^31) * S + B per document."""
    r = _c(r_u64, np.uint64)
    out = np.zeros(r.size, np.float64)
    lib().oracle_finalize(r, r.size, float(scale), float(bias), out)
    return out


def binary_features(row, group_factor, group_count, thresholds):
    gf = _c(group_factor, np.int32)
    gc = _c(group_count, np.int32)
    out = np.zeros(int(gc.sum()), np.uint8)
    lib().oracle_binary_features(_c(row, np.float32), gf, gc, gf.size,
                                 _c(thresholds, np.float32), out)
    return out


def apply_paper(x, group_factor, group_count, thresholds, stc, cond_indices, leaves_u32):
    """NEXT-2: paper-native mixed-height model, u64 sums."""
    x = _x2d(x)
    gf = _c(group_factor, np.int32)
    gc = _c(group_count, np.int32)
    thr = _c(thresholds, np.float32)
    out = np.zeros(x.shape[0], np.uint64)
    ci = _c(cond_indices, np.uint32)
    lv = _c(leaves_u32, np.uint32)
    lib().oracle_apply_paper(x, x.shape[0], x.shape[1], gf, gc, gf.size, thr, thr.size,
                             _c(stc, np.int32), ci if ci.size else np.zeros(1, np.uint32),
                             lv if lv.size else np.zeros(1, np.uint32), out)
    return out

"""Thin Python binding of the C ABI in include/odf.h (argument marshalling only).

Every step of the hot path runs in libodf.so's CUDA kernels; this module only
passes torch tensors' device pointers, sizes and the current CUDA stream.  If
the library is missing or fails to load, importing the binding raises: there is
no CPU fallback.  torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import build as _build

TILE_DOCS = 128
MAX_DEPTH = 10
MAX_BORDERS = 254        # uint8 bins
MAX_BORDERS_WIDE = 2032  # uint16 bins (wide models, NEXT-4)

_STATUS = {0: "ODF_OK", 1: "ODF_E_INVALID_ARG", 2: "ODF_E_UNSUPPORTED", 3: "ODF_E_NOMEM",
           4: "ODF_E_CUDA"}


class OdfError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class _Info(ctypes.Structure):
    _fields_ = [("depth", ctypes.c_int32), ("n_features", ctypes.c_int32),
                ("n_used_features", ctypes.c_int32), ("n_split_features", ctypes.c_int32),
                ("n_columns", ctypes.c_int32), ("n_trees", ctypes.c_int64),
                ("trees_per_chunk", ctypes.c_int32), ("n_tree_chunks", ctypes.c_int32),
                ("chunk_bytes", ctypes.c_int64), ("model_device_bytes", ctypes.c_int64),
                ("max_borders", ctypes.c_int32), ("total_borders", ctypes.c_int64),
                ("borders_in_smem", ctypes.c_int32), ("stages_fused", ctypes.c_int32),
                ("smem_fused", ctypes.c_int32), ("num_sms", ctypes.c_int32),
                ("leaf_type", ctypes.c_int32), ("bord_stride", ctypes.c_int32),
                ("bins_elem_bytes", ctypes.c_int32), ("max_tile_docs", ctypes.c_int32),
                ("stages_fused_256", ctypes.c_int32), ("smem_fused_256", ctypes.c_int32),
                ("bins_tile_docs", ctypes.c_int32), ("tail_tile_docs", ctypes.c_int32)]


class _Desc(ctypes.Structure):
    _fields_ = [("feature_index", ctypes.c_void_p), ("thresholds", ctypes.c_void_p),
                ("leaf_values", ctypes.c_void_p), ("leaf_type", ctypes.c_int32),
                ("depth", ctypes.c_int32), ("n_trees", ctypes.c_int64),
                ("n_features", ctypes.c_int32), ("device", ctypes.c_int32),
                ("scale", ctypes.c_double), ("bias", ctypes.c_double)]


class _PaperDesc(ctypes.Structure):
    _fields_ = [("n_features", ctypes.c_int32), ("group_factor", ctypes.c_void_p),
                ("group_count", ctypes.c_void_p), ("n_groups", ctypes.c_int32),
                ("thresholds", ctypes.c_void_p), ("stc", ctypes.c_void_p),
                ("cond_indices", ctypes.c_void_p), ("leaves", ctypes.c_void_p),
                ("scale", ctypes.c_double), ("bias", ctypes.c_double),
                ("device", ctypes.c_int32), ("pad_heights", ctypes.c_int32)]


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def library_path() -> str:
    return _build.LIB


_lib_path = None  # set by use_library() (diagnostics / A-B builds in tools/ only)


def use_library(path: str) -> None:
    """Load another build of the library (tools/: diagnostics and A/B builds made by
    build.build_variant) instead of the product libodf.so.  Must precede lib()."""
    global _lib_path
    if _lib is not None:
        raise RuntimeError("the library is already loaded")
    _lib_path = os.path.abspath(path)


def lib():
    """Load libodf.so (building it first if the sources are newer).  Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    path = _lib_path or _build.LIB
    if path == _build.LIB and _build._stale():
        try:
            _build.build()
        except Exception as e:  # no silent fallback: the CUDA path is the product
            if not os.path.exists(path):
                raise RuntimeError(f"libodf.so is missing and could not be built: {e}") from e
    L = ctypes.CDLL(path)
    L.odf_version.restype = ctypes.c_int
    L.odf_last_error.restype = ctypes.c_char_p
    L.odf_load_model.restype = ctypes.c_int
    L.odf_load_model.argtypes = [_vp, _vp, _vp, _i32, _i64, _i32, ctypes.c_int,
                                 ctypes.POINTER(_vp)]
    L.odf_load_model_ex.restype = ctypes.c_int
    L.odf_load_model_ex.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(_vp)]
    L.odf_load_model_paper.restype = ctypes.c_int
    L.odf_load_model_paper.argtypes = [ctypes.POINTER(_PaperDesc), ctypes.POINTER(_vp)]
    L.odf_binarize_fm.restype = ctypes.c_int
    L.odf_binarize_fm.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
    L.odf_score_fm.restype = ctypes.c_int
    L.odf_score_fm.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
    L.odf_bits_layout.restype = ctypes.c_int
    L.odf_bits_layout.argtypes = [_vp, _i64, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(_i64)]
    L.odf_bits_from_bins.restype = ctypes.c_int
    L.odf_bits_from_bins.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.odf_apply_bits.restype = ctypes.c_int
    L.odf_apply_bits.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.odf_score_u64.restype = ctypes.c_int
    L.odf_score_u64.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _vp]
    L.odf_apply_u64.restype = ctypes.c_int
    L.odf_apply_u64.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp]
    L.odf_free_model.restype = None
    L.odf_free_model.argtypes = [_vp]
    L.odf_get_info.restype = ctypes.c_int
    L.odf_get_info.argtypes = [_vp, ctypes.POINTER(_Info)]
    L.odf_bins_layout.restype = ctypes.c_int
    L.odf_bins_layout.argtypes = [_vp, _i64, ctypes.POINTER(ctypes.c_size_t),
                                  ctypes.POINTER(_i32), ctypes.POINTER(ctypes.POINTER(_i32))]
    L.odf_binarize.restype = ctypes.c_int
    L.odf_binarize.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
    L.odf_apply.restype = ctypes.c_int
    L.odf_apply.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.odf_score.restype = ctypes.c_int
    L.odf_score.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
    L.odf_score_tiles.restype = ctypes.c_int
    L.odf_score_tiles.argtypes = [_vp, _vp, _i64, _i64, _vp, _i32, _vp]
    L.odf_apply_tiles.restype = ctypes.c_int
    L.odf_apply_tiles.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp]
    L.odf_leaf_indices.restype = ctypes.c_int
    L.odf_leaf_indices.argtypes = [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp]
    L.odf_index_fingerprint.restype = ctypes.c_int
    L.odf_index_fingerprint.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.odf_latency_workspace_bytes.restype = ctypes.c_size_t
    L.odf_latency_workspace_bytes.argtypes = [_vp, _i64, _i32]
    L.odf_score_latency.restype = ctypes.c_int
    L.odf_score_latency.argtypes = [_vp, _vp, _i64, _i64, _vp, _i32, _vp, ctypes.c_size_t, _vp]
    L.odf_score_host.restype = ctypes.c_int
    L.odf_score_latency_u64.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _i32, _vp, ctypes.c_size_t, _vp]
    L.odf_score_latency_u64.restype = ctypes.c_int
    L.odf_score_host.argtypes = [_vp, _vp, _i64, _i64, _vp, _i64, _vp]
    _lib = L
    return L


ABI_SYMBOLS = ("odf_version", "odf_last_error", "odf_load_model", "odf_free_model",
               "odf_get_info", "odf_bins_layout", "odf_binarize", "odf_apply", "odf_score",
               "odf_leaf_indices", "odf_index_fingerprint", "odf_score_host",
               "odf_latency_workspace_bytes", "odf_score_latency", "odf_load_model_ex",
               "odf_score_u64", "odf_apply_u64", "odf_load_model_paper", "odf_binarize_fm",
               "odf_score_fm", "odf_bits_layout", "odf_bits_from_bins", "odf_apply_bits",
               "odf_score_tiles", "odf_apply_tiles", "odf_score_latency_u64")


def _check(status: int):
    if status != 0:
        raise OdfError(status, lib().odf_last_error().decode())


def _stream(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return _vp(stream.cuda_stream)


def _ptr(t):
    return _vp(t.data_ptr()) if t is not None and t.numel() > 0 else _vp(0)


def bins_to_canonical(bins: torch.Tensor, n_docs: int, n_used: int, elem_bytes: int = 1,
                      tile_docs: int = TILE_DOCS) -> torch.Tensor:
    """Blocked layout [tile][used][tile_docs] -> [n_docs][n_used] (a view + copy, no
    arithmetic).  uint8 bins, or (elem_bytes == 2, wide models) uint16 bins as int32."""
    tiles = (n_docs + tile_docs - 1) // tile_docs
    b = bins[: tiles * n_used * tile_docs * elem_bytes]
    if elem_bytes == 2:
        b = b.view(torch.int16).to(torch.int32) & 0xFFFF
    b = b.view(tiles, n_used, tile_docs)
    return b.permute(0, 2, 1).reshape(tiles * tile_docs, n_used)[:n_docs]


class Model:
    """An oblivious forest loaded onto one GPU (odf_load_model)."""

    def __init__(self, feature_index, thresholds, leaf_values, depth: int, n_features: int,
                 device: int = 0, leaf_type: str = "f32", scale: float = 1.0, bias: float = 0.0):
        L = lib()
        fi = np.ascontiguousarray(feature_index, dtype=np.int32)
        thr = np.ascontiguousarray(thresholds, dtype=np.float32)
        u32 = leaf_type == "u32"
        lv = np.ascontiguousarray(leaf_values, dtype=np.uint32 if u32 else np.float32)
        depth = int(depth)
        n_trees = lv.size >> depth if depth >= 0 else 0
        if depth >= 0 and (fi.size != n_trees * depth or thr.size != n_trees * depth
                           or lv.size != n_trees << depth):
            raise OdfError(1, f"array sizes {fi.size}/{thr.size}/{lv.size} inconsistent with "
                              f"depth {depth}")
        d = _Desc(fi.ctypes.data if fi.size else None, thr.ctypes.data if thr.size else None,
                  lv.ctypes.data if lv.size else None, 1 if u32 else 0, depth, n_trees,
                  int(n_features), int(device), float(scale), float(bias))
        h = _vp()
        _check(L.odf_load_model_ex(ctypes.byref(d), ctypes.byref(h)))
        self._init_from_handle(h, device)

    @classmethod
    def from_paper(cls, n_features, group_factor, group_count, thresholds, stc, cond_indices,
                   leaves, scale=1.0, bias=0.0, device: int = 0, pad_heights: bool = False) -> "Model":
        """Import the paper's model layout: see odf_load_model_paper
        (per-height segments; pad_heights=True: the padded uniform-depth form)."""
        gf = np.ascontiguousarray(group_factor, dtype=np.int32)
        gc = np.ascontiguousarray(group_count, dtype=np.int32)
        th = np.ascontiguousarray(thresholds, dtype=np.float32)
        st = np.zeros(MAX_DEPTH + 1, np.int32)
        st[:len(stc)] = np.asarray(stc, dtype=np.int32)
        ci = np.ascontiguousarray(cond_indices, dtype=np.uint32)
        lv = np.ascontiguousarray(leaves, dtype=np.uint32)
        d = _PaperDesc(int(n_features), gf.ctypes.data if gf.size else None,
                       gc.ctypes.data if gc.size else None, gf.size,
                       th.ctypes.data if th.size else None, st.ctypes.data,
                       ci.ctypes.data if ci.size else None, lv.ctypes.data if lv.size else None,
                       float(scale), float(bias), int(device), 1 if pad_heights else 0)
        h = _vp()
        _check(lib().odf_load_model_paper(ctypes.byref(d), ctypes.byref(h)))
        self = cls.__new__(cls)
        self._init_from_handle(h, device)
        return self

    def _init_from_handle(self, h, device):
        L = lib()
        self._h = h
        self.device = int(device)
        inf = _Info()
        _check(L.odf_get_info(self._h, ctypes.byref(inf)))
        self.info = {k: getattr(inf, k) for k, _ in _Info._fields_}
        self.depth = int(inf.depth)
        self.n_trees = int(inf.n_trees)
        self.n_features = int(inf.n_features)
        self.leaf_type = "u32" if inf.leaf_type == 1 else "f32"
        n = _i32()
        ids = ctypes.POINTER(_i32)()
        nb = ctypes.c_size_t()
        _check(L.odf_bins_layout(self._h, 0, ctypes.byref(nb), ctypes.byref(n), ctypes.byref(ids)))
        self.n_used = int(n.value)
        self.used_feature_ids = np.array([ids[i] for i in range(self.n_used)], np.int32)

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().odf_free_model(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- helpers ----------------------------------------------------------
    def _dev(self):
        return torch.device("cuda", self.device)

    def score_launches(self, n_docs: int) -> int:
        """Kernel launches of one odf_score (tile_docs = 0) over n_docs documents: 2 when a
        partly filled last wave runs as 64-document tiles in a second grid (odf.h)."""
        if not self.info.get("tail_tile_docs") or n_docs <= 0:
            return 1 if n_docs > 0 else 0
        nt, s = (n_docs + 127) // 128, self.info["num_sms"]
        return 2 if nt > s and nt % s and 2 * (nt % s) <= s else 1

    def bins_bytes(self, n_docs: int) -> int:
        nb = ctypes.c_size_t()
        _check(lib().odf_bins_layout(self._h, int(n_docs), ctypes.byref(nb), None, None))
        return int(nb.value)

    def _check_x(self, x: torch.Tensor):
        if not (x.is_cuda and x.dtype == torch.float32 and x.dim() == 2 and x.stride(1) == 1):
            raise OdfError(1, "factors must be a CUDA float32 [n_docs, ld] tensor with unit "
                              "column stride")
        if x.device != self._dev():
            raise OdfError(1, f"factors are on {x.device}, the model on {self._dev()}")
        if x.shape[1] < self.n_features:
            raise OdfError(1, f"factors have {x.shape[1]} columns < n_features {self.n_features}")
        return x.shape[0], x.stride(0)

    def _check_out(self, out, n: int, dtype, name: str = "out"):
        """A caller-supplied output: on the model's device, of `dtype`, >= n elements."""
        if out is None:
            return torch.empty(max(int(n), 0), dtype=dtype, device=self._dev())
        if not (isinstance(out, torch.Tensor) and out.is_cuda and out.device == self._dev()
                and out.dtype == dtype and out.is_contiguous() and out.numel() >= n):
            raise OdfError(1, f"{name} must be a contiguous CUDA {dtype} tensor on "
                              f"{self._dev()} with >= {n} elements")
        return out

    def _check_bins(self, bins, n_docs: int):
        need = self.bins_bytes(n_docs)
        if not (isinstance(bins, torch.Tensor) and bins.is_cuda and bins.device == self._dev()
                and bins.dtype == torch.uint8 and bins.is_contiguous() and bins.numel() >= need):
            raise OdfError(1, f"bins must be a contiguous CUDA uint8 tensor on {self._dev()} "
                              f"with >= {need} bytes (bins_bytes)")
        return bins

    # -- hot path ---------------------------------------------------------
    def binarize(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        n, ld = self._check_x(x)
        out = self._check_out(out, self.bins_bytes(n), torch.uint8)
        _check(lib().odf_binarize(self._h, _ptr(x), n, ld, _ptr(out), _stream(stream, self._dev())))
        return out

    def apply(self, bins: torch.Tensor, n_docs: int, out: torch.Tensor | None = None, stream=None,
              tile_docs: int = 0):
        """tile_docs: 0 (automatic), 128 or 256 (odf_apply_tiles); same scores for all."""
        bins = self._check_bins(bins, int(n_docs))
        out = self._check_out(out, int(n_docs), torch.float32)
        _check(lib().odf_apply_tiles(self._h, _ptr(bins), int(n_docs), _ptr(out), int(tile_docs),
                                     _stream(stream, self._dev())))
        return out

    def score(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None,
              tile_docs: int = 0):
        """Fused binarize + apply; tile_docs: 0 (automatic), 128 or 256 (odf_score_tiles)."""
        n, ld = self._check_x(x)
        out = self._check_out(out, n, torch.float32)
        _check(lib().odf_score_tiles(self._h, _ptr(x), n, ld, _ptr(out), int(tile_docs),
                                     _stream(stream, self._dev())))
        return out

    def latency_workspace(self, max_docs: int, splits: int = 0) -> torch.Tensor:
        n = int(lib().odf_latency_workspace_bytes(self._h, int(max_docs), int(splits)))
        return torch.empty(max(n, 256), dtype=torch.uint8, device=self._dev())

    def score_latency(self, x: torch.Tensor, workspace: torch.Tensor, out=None, splits: int = 0,
                      stream=None):
        """K4 small-batch path: two launches, tolerance-level parity with score()."""
        n, ld = self._check_x(x)
        out = self._check_out(out, n, torch.float32)
        if not (workspace.is_cuda and workspace.device == self._dev()):
            raise OdfError(1, f"workspace must be on {self._dev()}")
        _check(lib().odf_score_latency(self._h, _ptr(x), n, ld, _ptr(out), int(splits),
                                       _ptr(workspace), workspace.numel(),
                                       _stream(stream, self._dev())))
        return out

    def score_latency_u64(self, x: torch.Tensor, workspace: torch.Tensor, splits: int = 0, stream=None):
        """K4 for integer-leaf models: (u64 sums R as int64 bits, (R - 2^31)*S + B), equal to
        score_u64 bit for bit."""
        n, ld = self._check_x(x)
        if not (workspace.is_cuda and workspace.device == self._dev() and workspace.dtype == torch.uint8):
            raise OdfError(1, f"workspace must be a uint8 tensor on {self._dev()}")
        sums = torch.empty(n, dtype=torch.int64, device=self._dev())
        sc = torch.empty(n, dtype=torch.float64, device=self._dev())
        _check(lib().odf_score_latency_u64(self._h, _ptr(x), n, ld, _ptr(sums), _ptr(sc), int(splits),
                                           _ptr(workspace), workspace.numel(),
                                           _stream(stream, self._dev())))
        return sums, sc

    def score_u64(self, x: torch.Tensor, stream=None):
        """Integer-leaf model: (u64 sums R as int64 bits, (R - 2^31)*S + B as float64)."""
        n, ld = self._check_x(x)
        sums = torch.empty(n, dtype=torch.int64, device=self._dev())
        sc = torch.empty(n, dtype=torch.float64, device=self._dev())
        _check(lib().odf_score_u64(self._h, _ptr(x), n, ld, _ptr(sums), _ptr(sc),
                                   _stream(stream, self._dev())))
        return sums, sc

    def apply_u64(self, bins: torch.Tensor, n_docs: int, stream=None):
        bins = self._check_bins(bins, int(n_docs))
        sums = torch.empty(int(n_docs), dtype=torch.int64, device=self._dev())
        sc = torch.empty(int(n_docs), dtype=torch.float64, device=self._dev())
        _check(lib().odf_apply_u64(self._h, _ptr(bins), int(n_docs), _ptr(sums), _ptr(sc),
                                   _stream(stream, self._dev())))
        return sums, sc

    def _check_xt(self, xt: torch.Tensor, n_docs: int):
        if not (xt.is_cuda and xt.dtype == torch.float32 and xt.dim() == 2 and xt.stride(1) == 1
                and xt.shape[0] >= self.n_features and xt.shape[1] >= n_docs
                and xt.device == self._dev()):
            raise OdfError(1, "feature-major factors must be a CUDA float32 [>= n_features, "
                              f">= n_docs] tensor with unit column stride on {self._dev()}")
        return xt.stride(0)

    def binarize_fm(self, xt: torch.Tensor, n_docs: int, out=None, stream=None):
        """Feature-major input (NEXT-4): xt[f, i] = factor f of document i."""
        ld = self._check_xt(xt, n_docs)
        out = self._check_out(out, self.bins_bytes(n_docs), torch.uint8)
        _check(lib().odf_binarize_fm(self._h, _ptr(xt), int(n_docs), ld, _ptr(out),
                                     _stream(stream, self._dev())))
        return out

    def score_fm(self, xt: torch.Tensor, n_docs: int, out=None, stream=None):
        ld = self._check_xt(xt, n_docs)
        out = self._check_out(out, int(n_docs), torch.float32)
        _check(lib().odf_score_fm(self._h, _ptr(xt), int(n_docs), ld, _ptr(out),
                                  _stream(stream, self._dev())))
        return out

    # -- NEXT-3: bit-packed ordered condition words --------------------------------
    def bits_layout(self, n_docs: int):
        nb = ctypes.c_size_t()
        k = _i64()
        _check(lib().odf_bits_layout(self._h, int(n_docs), ctypes.byref(nb), ctypes.byref(k)))
        return int(nb.value), int(k.value)

    def bits_from_bins(self, bins: torch.Tensor, n_docs: int, out=None, stream=None):
        nbytes, k = self.bits_layout(n_docs)
        bins = self._check_bins(bins, int(n_docs))
        out = self._check_out(out, max(nbytes // 4, 1), torch.int32)
        _check(lib().odf_bits_from_bins(self._h, _ptr(bins), int(n_docs), _ptr(out),
                                        _stream(stream, self._dev())))
        return out

    def apply_bits(self, words: torch.Tensor, n_docs: int, out=None, stream=None):
        nbytes, _ = self.bits_layout(n_docs)
        self._check_out(words, nbytes // 4, torch.int32, "words")
        out = self._check_out(out, int(n_docs), torch.float32)
        _check(lib().odf_apply_bits(self._h, _ptr(words), int(n_docs), _ptr(out),
                                    _stream(stream, self._dev())))
        return out

    def score_host(self, x, out=None, chunk_docs: int = 65536, stream=None):
        """End-to-end from host memory (numpy array or CPU tensor, ideally pinned)."""
        if isinstance(x, torch.Tensor):
            if not (x.device.type == "cpu" and x.dtype == torch.float32 and x.dim() == 2
                    and x.stride(1) == 1):
                raise OdfError(1, "host factors must be a CPU float32 [n_docs, ld] tensor with "
                                  "unit column stride")
            n, ld, xp = x.shape[0], x.stride(0), x.data_ptr()
            if out is None:
                out = torch.empty(n, dtype=torch.float32, pin_memory=x.is_pinned())
            if not (isinstance(out, torch.Tensor) and out.device.type == "cpu"
                    and out.dtype == torch.float32 and out.is_contiguous() and out.numel() >= n):
                raise OdfError(1, f"out must be a contiguous CPU float32 tensor with >= {n} elements")
            op = out.data_ptr()
        else:
            x = np.ascontiguousarray(x, dtype=np.float32)
            if x.ndim != 2:
                raise OdfError(1, "host factors must be a 2-D [n_docs, n_features] array")
            n, ld, xp = x.shape[0], x.shape[1], x.ctypes.data
            if out is None:
                out = np.empty(n, np.float32)
            if not (isinstance(out, np.ndarray) and out.dtype == np.float32
                    and out.flags["C_CONTIGUOUS"] and out.size >= n):
                raise OdfError(1, f"out must be a contiguous float32 array with >= {n} elements")
            op = out.ctypes.data
        _check(lib().odf_score_host(self._h, _vp(xp), n, ld, _vp(op), int(chunk_docs),
                                    _stream(stream, self._dev())))
        return out

    # -- test / debug (K6) ----------------------------------------------------
    def leaf_indices(self, bins, n_docs, doc0, ndoc, tree0, ntree, stream=None):
        bins = self._check_bins(bins, int(n_docs))
        out = torch.empty((int(ndoc), int(ntree)), dtype=torch.int16, device=self._dev())
        _check(lib().odf_leaf_indices(self._h, _ptr(bins), int(n_docs), int(doc0), int(ndoc),
                                      int(tree0), int(ntree), _ptr(out),
                                      _stream(stream, self._dev())))
        return out

    def index_fingerprint(self, bins, n_docs, stream=None):
        bins = self._check_bins(bins, int(n_docs))
        out = torch.empty(int(n_docs), dtype=torch.int64, device=self._dev())
        _check(lib().odf_index_fingerprint(self._h, _ptr(bins), int(n_docs), _ptr(out),
                                           _stream(stream, self._dev())))
        return out

    def canonical_bins(self, bins: torch.Tensor, n_docs: int) -> torch.Tensor:
        return bins_to_canonical(bins, n_docs, self.n_used, self.info["bins_elem_bytes"],
                                 self.info["bins_tile_docs"])

"""B200-native oblivious-decision-forest scorer (arxiv 2205.07307 hot path).

Stage 1 binarization and stage 2 tree apply as sm_100a CUDA kernels behind the
C ABI in include/odf.h; this package is the thin Python binding (odf.py) plus
the multi-GPU orchestration over torch.distributed (parallel.py).
"""
from .odf import (MAX_BORDERS, MAX_BORDERS_WIDE, MAX_DEPTH, TILE_DOCS, Model, OdfError, bins_to_canonical, lib,
                  library_path)

__all__ = ["Model", "OdfError", "lib", "library_path", "bins_to_canonical", "TILE_DOCS",
           "MAX_DEPTH", "MAX_BORDERS", "MAX_BORDERS_WIDE"]

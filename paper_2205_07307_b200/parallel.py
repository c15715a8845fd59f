"""Multi-GPU orchestration over torch.distributed (one process per GPU, NCCL).

The paper scales by giving every worker a private copy of the data and the
model ("Каждый поток получал свою копию данных и модели").  On one
8xB200 box that becomes:

* document sharding (the default): every rank holds the whole model (<= ~20 MB)
  and scores its own contiguous slice of one batch's documents
  [floor(r*D/W), floor((r+1)*D/W)); the only collective is the score all-gather
  (bench.py times it inside the step: strong scaling of one batch).  Scores are
  bit-identical to W = 1 because a document's summation order does not depend
  on the batch it is scored in.
* tree sharding (for forests too large for one GPU's fast memory, config c4):
  rank r holds trees [floor(r*T/W), floor((r+1)*T/W)), binarizes ALL documents,
  produces fp32 partial scores, and one NCCL reduce (or all-reduce /
  reduce-scatter) sums them.  Results equal W = 1 within the tolerance (a
  different association of the same fp32 sum), bit-exactly when every partial
  sum is exact.

The per-rank compute is a `scorer(x) -> scores` callable: the CUDA path
(`Model.score`) in production; tests substitute a CPU scorer to exercise this
host logic with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[floor(rank*n/world), floor((rank+1)*n/world))."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} not in [0, {world})")
    return (n * rank) // world, (n * (rank + 1)) // world


def tree_shard(feature_index, thresholds, leaf_values, depth: int, world: int, rank: int):
    """The raw arrays of rank's tree shard (trees [floor(r*T/W), floor((r+1)*T/W)))."""
    lv = np.asarray(leaf_values)
    T = lv.size >> depth
    t0, t1 = shard_bounds(T, world, rank)
    fi = np.asarray(feature_index)[t0 * depth:t1 * depth]
    th = np.asarray(thresholds)[t0 * depth:t1 * depth]
    return fi, th, lv[t0 << depth:t1 << depth], (t0, t1)


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


@dataclass
class DocSharded:
    """Document-sharded scoring with a replicated model."""
    scorer: Callable[[torch.Tensor], torch.Tensor]
    group: object = None

    def local_range(self, n_docs: int) -> tuple[int, int]:
        w, r = _world(self.group)
        return shard_bounds(n_docs, w, r)

    def score_local(self, x_local: torch.Tensor) -> torch.Tensor:
        return self.scorer(x_local)

    def score(self, x_all: torch.Tensor, gather: bool = True) -> torch.Tensor:
        """Score this rank's slice of x_all (rows [lo, hi)); optionally all-gather."""
        lo, hi = self.local_range(x_all.shape[0])
        local = self.scorer(x_all[lo:hi].contiguous())
        return self.gather(local, x_all.shape[0]) if gather else local

    def gather(self, local: torch.Tensor, n_docs: int) -> torch.Tensor:
        w, _ = _world(self.group)
        if w == 1:
            return local
        sizes = [shard_bounds(n_docs, w, k)[1] - shard_bounds(n_docs, w, k)[0] for k in range(w)]
        m = max(sizes)
        buf = torch.zeros(m, dtype=local.dtype, device=local.device)
        buf[:local.numel()] = local
        parts = [torch.empty_like(buf) for _ in range(w)]
        dist.all_gather(parts, buf, group=self.group)
        return torch.cat([p[:s] for p, s in zip(parts, sizes)])

    @staticmethod
    def padded_size(n_docs: int, world: int) -> int:
        """Per-rank slot of the padded gather buffer: ceil(n_docs / world)."""
        return -(-n_docs // world)

    def gather_into(self, local_padded: torch.Tensor, out_padded: torch.Tensor) -> torch.Tensor:
        """All-gather with preallocated buffers (the timed step): rank r's scores sit in
        local_padded[:hi-lo] (length padded_size), and land in out_padded[r*m : r*m + hi-lo]
        (length world*m).  `unpad` turns the result into the [n_docs] score vector."""
        w, _ = _world(self.group)
        if w == 1:
            out_padded.copy_(local_padded)
            return out_padded
        if dist.get_backend(self.group) == "gloo":  # no all_gather_into_tensor on gloo
            dist.all_gather(list(out_padded.chunk(w)), local_padded, group=self.group)
        else:
            dist.all_gather_into_tensor(out_padded, local_padded, group=self.group)
        return out_padded

    def unpad(self, out_padded: torch.Tensor, n_docs: int) -> torch.Tensor:
        w, _ = _world(self.group)
        m = self.padded_size(n_docs, w)
        return torch.cat([out_padded[k * m:k * m + (shard_bounds(n_docs, w, k)[1] -
                                                    shard_bounds(n_docs, w, k)[0])]
                          for k in range(w)])


@dataclass
class TreeSharded:
    """Tree-sharded scoring: partial scores of this rank's trees, summed across ranks."""
    scorer: Callable[[torch.Tensor], torch.Tensor]  # scores x with THIS rank's tree shard
    group: object = None

    def score(self, x: torch.Tensor, op: str = "all_reduce", root: int = 0) -> torch.Tensor:
        part = self.scorer(x).to(torch.float32)
        w, r = _world(self.group)
        if w == 1:
            return part
        if op == "reduce":
            dist.reduce(part, dst=root, op=dist.ReduceOp.SUM, group=self.group)
            return part  # meaningful on root only
        if op == "all_reduce":
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
            return part
        if op == "reduce_scatter":  # doc-sharded totals: rank r gets rows shard_bounds(D, w, r)
            n = part.numel()
            sizes = [shard_bounds(n, w, k)[1] - shard_bounds(n, w, k)[0] for k in range(w)]
            m = max(sizes)
            padded = torch.zeros(w * m, dtype=part.dtype, device=part.device)
            for k in range(w):
                lo, hi = shard_bounds(n, w, k)
                padded[k * m:k * m + (hi - lo)] = part[lo:hi]
            out = torch.empty(m, dtype=part.dtype, device=part.device)
            if dist.get_backend(self.group) == "gloo":  # gloo has no reduce_scatter_tensor
                dist.all_reduce(padded, op=dist.ReduceOp.SUM, group=self.group)
                out.copy_(padded[r * m:(r + 1) * m])
            else:
                dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM, group=self.group)
            return out[:sizes[r]]
        raise ValueError(op)


def cuda_doc_sharded(model, group=None) -> DocSharded:
    """Document sharding over the CUDA path of `model` (paper_2205_07307_b200.Model)."""
    return DocSharded(lambda x: model.score(x), group)


def cuda_tree_sharded(feature_index, thresholds, leaf_values, depth, n_features, device,
                      group=None):
    """Load this rank's tree shard onto `device` and return (TreeSharded, model)."""
    from .odf import Model
    w, r = _world(group)
    fi, th, lv, _ = tree_shard(feature_index, thresholds, leaf_values, depth, w, r)
    model = Model(fi, th, lv, depth, n_features, device=device)
    return TreeSharded(lambda x: model.score(x), group), model

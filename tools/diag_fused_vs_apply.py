"""Determinism / agreement check of fused vs two-stage on many tiles, per depth."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, oracle
from helpers import cuda_model, to_dev, tolerance
depths = [int(a) for a in sys.argv[1:]] or [6, 7, 8, 9, 10]
for d in depths:
    case = synth.tiny_case(seed=500 + d, n_docs=200_000, n_features=40, n_trees=160, depth=d, pool=200)
    m = cuda_model(case); x = to_dev(case.x); nd = case.n_docs
    f1 = m.score(x).cpu().numpy(); f2 = m.score(x).cpu().numpy()
    bins = m.binarize(x); a1 = m.apply(bins, nd).cpu().numpy(); a2 = m.apply(bins, nd).cpu().numpy()
    bad = np.flatnonzero(f1.view(np.uint32) != a1.view(np.uint32))
    print('depth', d, 'info', {k: m.info[k] for k in ('stages_fused', 'trees_per_chunk', 'chunk_bytes', 'n_columns')},
          'fused det', np.array_equal(f1.view(np.uint32), f2.view(np.uint32)),
          'apply det', np.array_equal(a1.view(np.uint32), a2.view(np.uint32)),
          'mismatch', bad.size, 'first tiles', np.unique(bad // 128)[:6], flush=True)
    m.close(); del x, bins; torch.cuda.empty_cache()

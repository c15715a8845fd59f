import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from helpers import cuda_model, to_dev
for T in [16, 64, 256, 1000, 4000]:
    case = synth.make_case("c4", n_docs=100_000, n_trees=T)
    m = cuda_model(case); x = to_dev(case.x); nd = case.n_docs
    f1 = m.score(x).cpu().numpy(); f2 = m.score(x).cpu().numpy()
    bins = m.binarize(x); b2 = m.binarize(x)
    bdet = torch.equal(bins, b2)
    a1 = m.apply(bins, nd).cpu().numpy(); a2 = m.apply(bins, nd).cpu().numpy()
    bad = np.flatnonzero(f1.view(np.uint32) != a1.view(np.uint32))
    print('T', T, {k: m.info[k] for k in ('stages_fused', 'n_columns', 'n_split_features', 'smem_fused')},
          'bins det', bdet, 'fused det', np.array_equal(f1.view(np.uint32), f2.view(np.uint32)),
          'apply det', np.array_equal(a1.view(np.uint32), a2.view(np.uint32)),
          'mismatch', bad.size, 'first tiles', np.unique(bad // 128)[:6], flush=True)
    m.close(); del x, bins, b2; torch.cuda.empty_cache()

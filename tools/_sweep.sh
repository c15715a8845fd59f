cat > /tmp/ov.py <<'PY'
import json, sys, os; sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch, synth
from time_kernels import timeit
from paper_2205_07307_b200 import Model
for cfg in ["c2", "c3"]:
    case = synth.make_case(cfg)
    m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
    x = torch.from_numpy(case.x).cuda(); n = case.n_docs
    out = torch.empty(n, device="cuda"); ws = m.overlap_workspace(n)
    r = {"config": cfg, "fused_ms": timeit(lambda: m.score(x, out=out)),
         "overlap_ms": timeit(lambda: m.score_overlap(x, ws, out=out))}
    os.environ["ODF_OV_ONLY"] = "A"; r["A_only_ms"] = timeit(lambda: m.score_overlap(x, ws, out=out))
    os.environ["ODF_OV_ONLY"] = "B"; r["B_only_ms"] = timeit(lambda: m.score_overlap(x, ws, out=out))
    del os.environ["ODF_OV_ONLY"]
    print(json.dumps(r), flush=True)
    m.close()
PY
timeout 300 python /tmp/ov.py

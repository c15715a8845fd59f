import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2205_07307_b200 import Model
case = synth.make_case("c5", n_docs=65536)
m = Model(case.feature_index, case.thresholds, case.leaf_values, case.depth, case.n_features)
x = torch.from_numpy(case.x).cuda()
for B in (100, 1000, 5000):
    ws = m.latency_workspace(B)
    for q in range(5):
        m.score_latency(x[q * 7:q * 7 + B], ws)
torch.cuda.synchronize()
print("done")

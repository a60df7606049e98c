import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14628_b200 as H
from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state
layers = model_layers("rn18_224")
cons = channel_keep_constraints(layers, 0.4)
sched = H.PenaltySchedule.uniform([ls.name for ls in layers], 1.5e-3, 1.5e-4, adapt=False)
settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
eng = H.HSADMMSync(0, H.LocalCluster(H.Topology(1, 1)), layers, cons, sched, settings, residuals=False)
eng.load(**synthetic_rank_state(layers, 0, 1, 0))
for k in range(1, 4):
    H.run_local([eng], k)
    torch.cuda.synchronize()
    print("---- step", k, flush=True)

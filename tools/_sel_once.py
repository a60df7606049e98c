import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from probe_tails import engine
from paper_2512_14628_b200.synthetic import model_layers
eng = engine(model_layers("rn18_224"))
pl = eng.plan
torch.cuda.synchronize()
print("=== one candidate + select", flush=True)
pl.candidate(None, eng.theta, eng.u, eng.z, eng.v, eng.z_node); pl.select(0)
torch.cuda.synchronize()

"""Run a few iterations of a config with a given chain_warps (ncu target; tooling)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
k, W = int(sys.argv[1]), int(sys.argv[2])
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"))
s.set_options(chain_warps=W, streams=1)
X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
s.sample(X, 6, cfg.chain_seed, out=X)
torch.cuda.synchronize()
print("ok")

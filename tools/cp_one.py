"""One constraint-parallel run at config 3 sizes on one rank (tooling: ncu launch list)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
A, b, x0 = synth.make_instance(3, m=2000, d=1000)
cp = tm.ConstraintParallel(A, b)
cp.sample(np.tile(x0, (4096, 1)), 8, seed=1)
torch.cuda.synchronize()
print("ok")

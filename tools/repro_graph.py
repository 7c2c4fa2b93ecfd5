import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
A, b, x0 = synth.make_instance(3, m=150, d=40)
s = tm.Sampler(A, b, graphs=1)
out = s.sample(np.tile(x0, (130, 1)), 32, seed=13)
print("ok", out.shape)

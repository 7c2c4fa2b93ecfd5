"""Latency mode on two geometries (tooling): S4.2 (arcs start just past 0) and config-3
rows (arcs spread over the circle), 10 chains, per iteration, for two library builds."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for path in sys.argv[1:]:
    tm._LIB = None
    tm.LIB_PATH = os.path.abspath(path)
    for name, (A, b, x0) in (("S4.2 d=m=1000", synth.paper_random(1000, seed=1000)),
                             ("cfg3 rows m=2000 d=1000", synth.make_instance(3)),
                             ("cfg3 rows m=500 d=100", synth.make_instance(3, m=500, d=100))):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=1)
        X = torch.tensor(np.tile(x0, (10, 1)), device="cuda")
        s.sample(X, 50, 1, out=X)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, 300, 1, out=X)
        torch.cuda.synchronize()
        print(f"{os.path.basename(path)} {name}: {(time.perf_counter()-t0)/300*1e6:.1f} us/iter", flush=True)
        s.close()

"""Constraint-parallel iteration cost on one rank (tooling): per-iteration time of
ConstraintParallel vs tmvn_sample on the same instance."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for (m, d, C) in ((2000, 1000, 512), (2000, 1000, 4096), (1000, 1000, 10)):
    A, b, x0 = synth.make_instance(3, m=m, d=d)
    X0 = np.tile(x0, (C, 1))
    cp = tm.ConstraintParallel(A, b)
    cp.sample(X0, 3, seed=1)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cp.sample(X0, 20, seed=1)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
    s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=0)
    X = torch.tensor(X0, device="cuda")
    s.sample(X, 3, 1, out=X)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s.sample(X, 20, 1, out=X)
    torch.cuda.synchronize(); dt2 = (time.perf_counter() - t1) / 20
    print(f"m={m} d={d} C={C}: constraint-parallel (1 rank) {dt*1e6:.0f} us/iter ({C*m/dt:.2e} evals/s); "
          f"throughput path {dt2*1e6:.0f} us/iter ({C*m/dt2:.2e})", flush=True)

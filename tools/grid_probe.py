"""Latency mode: cluster variant vs cooperative-grid variant per iteration (tooling)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for d in (1000, 2000, 4000):
    A, b, x0 = synth.paper_random(d, seed=d)
    for C in (1, 2, 4, 10):
        for prec in (0, 1):
            res = []
            for mode in (-1, 1, 0):
                s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=1 if mode else 2,
                               precision=prec, trim_eps=1e-5 if prec else 0.0)
                s.test_latency_grid(mode)
                X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
                s.sample(X, 20, 42, out=X)
                torch.cuda.synchronize(); t0 = time.perf_counter()
                s.sample(X, 200, 42, out=X)
                torch.cuda.synchronize(); res.append((time.perf_counter() - t0) / 200 * 1e6)
                s.close()
            print(f"d=m={d} C={C} precision={prec}: cluster {res[0]:.1f} us/iter, grid {res[1]:.1f} us/iter, "
                  f"auto {res[2]:.1f} us/iter", flush=True)

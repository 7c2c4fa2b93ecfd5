"""Throughput path per-iteration time vs chain count at d = m = 1000 (tooling)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
A, b, x0 = synth.make_instance(3, m=1000, d=1000)
for C in (80, 148, 256, 512, 1024, 2048):
    for W in (0, 16):
        graphs = 1
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=0, graphs=graphs,
                       chain_warps=W)
        X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
        s.sample(X, 64, 3, out=X)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, 256, 3, out=X)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 256
        print(f"C={C} W={W or 'auto'}: {dt*1e6:.1f} us/iter, {C*1000/dt:.2e} evals/s", flush=True)
        s.close()

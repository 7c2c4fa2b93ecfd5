"""FP32 (options.precision = 1) vs FP64 latency mode: time per iteration on the S4.2
workload and the S4.1 rejection counts (tooling)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for d, C in ((1000, 10), (1000, 1), (2000, 10), (4000, 1), (4000, 10), (4000, 32)):
    A, b, x0 = synth.paper_random(d, seed=d)
    for prec, lat in ((0, 0), (0, 1), (1, 1)):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), precision=prec,
                       trim_eps=1e-5 if prec else 0.0, latency=lat)
        X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
        s.sample(X, 50, 42, out=X)
        s.reset_stats()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, 500, 42, out=X)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"S4.2 d=m={d} C={C} precision={prec} latency={lat}: {dt / 500 * 1e6:.1f} us/iter, "
              f"{C * d * 500 / dt:.3e} evals/s, rejections {s.stats()['rejections']}, "
              f"fallbacks {s.profile()['latency_fallbacks']}", flush=True)
        s.close()
for iv in ((-1.0, 3.0), (15.0, 16.0)):
    A, b, x0 = synth.one_dim(iv)
    s = tm.Sampler(A, b, precision=1, trim_eps=1e-5, burn_in=500, thin=10)
    s.sample(np.tile(x0, (2000, 1)), 1000, seed=2024)
    sm, sq, n = s.moments()
    print(f"S4.1 {iv} FP32: mean {sm[0]/n:.4f} var {sq[0]/n-(sm[0]/n)**2:.4f} rejections {s.stats()['rejections']} of {s.stats()['steps']}")

"""Time per iteration of tmvn_sample with options.warp_mode = 2 (auto) vs 0 on small
polytopes (tooling): BASELINE configs 1 and 2, the S4.1 interval, and few-chain cases."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

cases = []
A, b, x0 = synth.make_instance(1); cases.append(("cfg1 C=16", A, b, x0, 16))
A, b, x0 = synth.make_instance(2); cases.append(("cfg2 C=1024", A, b, x0, 1024))
cases.append(("cfg2 C=10", A, b, x0, 10))
cases.append(("cfg2 C=148", A, b, x0, 148))
cases.append(("cfg2 C=2048", A, b, x0, 2048))
cases.append(("cfg2 C=4096", A, b, x0, 4096))
A, b, x0 = synth.one_dim((-1.0, 3.0)); cases.append(("S4.1 C=2000", A, b, x0, 2000))
A, b, x0 = synth.make_instance(3, m=300, d=40); cases.append(("rand m300 d40 C=300", A, b, x0, 300))
cases.append(("rand m300 d40 C=20", A, b, x0, 20))
iters = int(os.environ.get("ITERS", "1000"))
for name, A, b, x0, C in cases:
    line = [name]
    for wm in (0, int(os.environ.get("WM", "2"))):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), warp_mode=wm)
        X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
        s.sample(X, 100, 3, out=X)
        s.reset_stats()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, iters, 3, out=X)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        pr = s.profile()
        line.append(f"wm={wm}: {dt / iters * 1e6:7.2f} us/it (warp calls {pr['warp_mode_calls']}, latency {pr.get('latency_calls', '-')})")
        s.close()
    print(" | ".join(line), flush=True)

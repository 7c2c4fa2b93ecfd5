"""Warp-mode timing at config 1 / 2 (tooling)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for k in [int(x) for x in sys.argv[1].split(",")]:
    cfg = synth.CONFIGS[k]
    A, b, x0 = synth.make_instance(k)
    s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), warp_mode=1)
    X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
    n = int(os.environ.get("ITERS", "500"))
    s.sample(X, 50, cfg.chain_seed, out=X)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.sample(X, n, cfg.chain_seed, out=X)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"config {k}: warp mode {dt / n * 1e6:.2f} us/iter", flush=True)

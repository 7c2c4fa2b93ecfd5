"""ESS / projection time per launch vs chain count at config-3 geometry (tooling)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
A, b, x0 = synth.make_instance(3)
for C in [int(x) for x in sys.argv[1].split(",")]:
    s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"))
    s.set_options(profile=1, streams=1, chain_warps=int(os.environ.get("W", "0")))
    X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
    s.sample(X, 60, 103, out=X)
    s.reset_stats()
    s.sample(X, 64, 103, out=X)
    pr = s.profile()
    e = pr["ess_ms"] / max(1, pr["ess_launches"]); g = pr["tc_ms"] / max(1, pr["tc_launches"])
    print(f"C={C:6d}  ess {e*1e3:8.1f} us ({e*1e6/C:.1f} ns/chain)  proj {g*1e3:8.1f} us ({g*1e6/C:.1f} ns/chain)", flush=True)
    s.close()

"""Per-iteration time of config k under option sets (tooling, not a bench number).
usage: python tools/probe.py k '{"projection": 2}' '{}' ...   (env ITERS, WARM)"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
k = int(sys.argv[1])
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
iters = int(os.environ.get("ITERS", "1000"))
warm = int(os.environ.get("WARM", "100"))
for spec in sys.argv[2:]:
    kw = json.loads(spec)
    s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), **kw)
    X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
    s.sample(X, warm, cfg.chain_seed, out=X)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.sample(X, iters, cfg.chain_seed, out=X)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    pr = s.profile()
    print(f"cfg{k} {spec}: {dt / iters * 1e6:.2f} us/iter  evals/s {cfg.C * cfg.m * iters / dt:.3e}  "
          f"lat {pr['latency_calls']} warp {pr['warp_mode_calls']} proj {pr['projection_used']}", flush=True)
    s.close()

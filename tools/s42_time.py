"""Per-iteration time of the S4.2 geometry (paper_random, one start, many chains) for
library builds and level-1 bucket mappings (tooling, not a bench number).
usage: python tools/s42_time.py lib1.so [lib2.so ...]   (env BUCKETS=1,2,0  SHAPES=d:C,..)"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
shapes = [tuple(int(v) for v in s.split(":")) for s in os.environ.get("SHAPES", "1000:200,1000:1000,600:400").split(",")]
bks = [int(v) for v in os.environ.get("BUCKETS", "1,2,0").split(",")]
for path in sys.argv[1:]:
    tm._LIB = None
    tm.LIB_PATH = os.path.abspath(path)
    for d, C in shapes:
        A, b, x0 = synth.paper_random(d, seed=d)
        for bk in bks:
            s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=0, buckets=bk, profile=1)
            X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
            s.sample(X, 20, 42, out=X)
            s.reset_stats()
            torch.cuda.synchronize(); t0 = time.perf_counter()
            NI = int(os.environ.get("ITERS", "100"))
            s.sample(X, NI, 42, out=X)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            pr = s.profile()
            print(f"{os.path.basename(path)} S4.2 d={d} C={C} buckets={bk}: {dt/NI*1e6:.1f} us/iter  used={pr['buckets_used']}  ess {pr['ess_ms']/max(1,pr['ess_launches'])*1e3:.1f} us x{pr['ess_launches']}  proj {(pr['gemm_ms']+pr['tc_ms'])/max(1,pr['gemm_launches']+pr['tc_launches'])*1e3:.1f} us", flush=True)
            s.close()

import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for k in (1, 6):
    cfg = synth.CONFIGS[k]
    A, b, x0 = synth.make_instance(k)
    for lat in (0, 1):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=lat)
        X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
        s.sample(X, 50, 7, out=X)
        for n in (100, 1000):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            s.sample(X, n, 7, out=X)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            print(f"cfg{k} C={cfg.C} latency={lat} n={n}: {dt/n*1e6:.2f} us/iter  calls={s.profile()['latency_calls']}", flush=True)
# fixed cost of one call (n_iter = 1), latency mode, device tensors
for k in (1, 6):
    cfg = synth.CONFIGS[k]
    A, b, x0 = synth.make_instance(k)
    s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=1)
    X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
    for rec in (1, 0):
        s.set_options(record=rec)
        s.sample(X, 1, 7, out=X)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(50):
            s.sample(X, 1, 7, out=X)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 50
        print(f"cfg{k} one-iteration call (record={rec}): {dt*1e6:.1f} us", flush=True)

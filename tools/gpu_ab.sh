mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/t_all.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_all.log
cat > /tmp/gr.py << 'PY'
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for k in (1, 2, 3):
    cfg = synth.CONFIGS[k]; A, b, x0 = synth.make_instance(k)
    for graphs in (0, 1):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), graphs=graphs)
        X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
        n = 640 if k < 3 else 128
        s.sample(X, 64, cfg.chain_seed, out=X); torch.cuda.synchronize()
        t0 = time.perf_counter(); s.sample(X, n, cfg.chain_seed, out=X); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"cfg{k} graphs={graphs}: {dt/n*1e6:.1f} us/iter  evals/s {cfg.C*cfg.m*n/dt:.3e}", flush=True)
PY
python /tmp/gr.py > gpurun_out/graphs.log 2>&1

mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "stages or options_bitwise or odd_m or trace" > gpurun_out/t24.log 2>&1
echo "tests rc=$?" >> gpurun_out/t24.log
( PAPER_D=1000 PAPER_C=200 python tools/phase_timing.py 3 12 ) > gpurun_out/ph24.log 2>&1
python - >> gpurun_out/ph24.log 2>&1 <<'PY'
import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for d, C in ((1000, 200), (1000, 1000), (600, 400)):
    A, b, x0 = synth.paper_random(d, seed=d)
    for bk in (1, 2, 0):
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=0, buckets=bk)
        X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
        s.sample(X, 20, 42, out=X)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, 100, 42, out=X)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"S4.2 d={d} C={C} buckets={bk}: {dt/100*1e6:.1f} us/iter", flush=True)
PY

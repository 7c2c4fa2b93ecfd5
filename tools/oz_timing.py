"""Role timing of ozaki_gemm_kernel (timing build; tooling, not a bench number).
usage: python tools/oz_timing.py [config] [iters]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
tm.LIB_PATH = os.environ.get("TIMING_LIB", os.path.join(ROOT, "build", "libtmvn_timing.so"))
L = tm.lib()
L.tmvn_test_oz_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), projection=1, graphs=0)
X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
s.sample(X, 4, cfg.chain_seed, out=X)
buf = np.zeros(10, dtype=np.uint64)
L.tmvn_test_oz_cycles(buf.ctypes.data_as(ctypes.c_void_p), 1)
s.sample(X, iters, cfg.chain_seed, out=X)
L.tmvn_test_oz_cycles(buf.ctypes.data_as(ctypes.c_void_p), 0)
tiles = float(buf[6])
names = ["MMA wait full", "MMA wait tmem_empty", "MMA issue", "epi wait tmem_full", "epi work",
         "producer wait empty", "tiles", "CTA cycles", "MMA wait A loaders", "loaders wait A buf"]
for i, n in enumerate(names):
    if i == 6:
        print(f"  {n:22s} {buf[i]:.0f}")
    else:
        print(f"  {n:22s} {buf[i] / tiles:12.0f} cycles/tile")

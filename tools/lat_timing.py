"""Phase timing of the latency kernel (timing build; tooling). usage: python tools/lat_timing.py config iters"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
tm.LIB_PATH = os.path.join(ROOT, "build", "libtmvn_timing.so")
L = tm.lib()
L.tmvn_test_lat_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
k = int(sys.argv[1]); iters = int(sys.argv[2])
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
s = tm.Sampler(A, b, latency=1)
C = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.C
X = np.tile(x0, (C, 1))
X = s.sample(X, 10, cfg.chain_seed)
buf = np.zeros(16, dtype=np.uint64)
L.tmvn_test_lat_cycles(buf.ctypes.data_as(ctypes.c_void_p), 1)
s.sample(X, iters, cfg.chain_seed)
L.tmvn_test_lat_cycles(buf.ctypes.data_as(ctypes.c_void_p), 0)
names = ["a nu", "b Q rows", "c arcs+stats", "sync1", "merge+gather", "sync2", "CTA0 I_act+theta", "sync3",
         "P'+safeguard", "sync4", "update+moments+refresh", "(live arcs)", "  L2 rank+zero", "  L2 atomics", "  L2 rest", "  L2 scan+live"]
for i, n in enumerate(names):
    print(f"  {n:24s} {buf[i] / iters:10.0f} cycles/iter")

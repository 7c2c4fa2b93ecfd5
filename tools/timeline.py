"""Kernel timeline of the hot loop (timeline build, -DTMVN_TIMELINE; tooling).
usage: python tools/timeline.py lib.so [pipeline] [iters]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
tm.LIB_PATH = os.path.abspath(sys.argv[1])
L = tm.lib()
L.tmvn_test_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
pipe = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 12
cfg = synth.CONFIGS[3]
A, b, x0 = synth.make_instance(3)
s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), pipeline=pipe, graphs=0)
X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
s.sample(X, 40, cfg.chain_seed, out=X)
buf = np.zeros(256 * 4, dtype=np.uint64)
L.tmvn_test_timeline(buf.ctypes.data_as(ctypes.c_void_p), 1)
s.set_options(iter_offset=0)
s.sample(X, iters, cfg.chain_seed, out=X)
L.tmvn_test_timeline(buf.ctypes.data_as(ctypes.c_void_p), 0)
tl = buf.reshape(256, 4).astype(np.float64)
valid = tl[:, 2] < 1e30
t0 = min(tl[valid, 2].min(), tl[tl[:, 0] < 1e30, 0].min())
print(f"pipeline={pipe}: times in us from the first kernel start")
for i in range(iters + 1):
    g0, g1, e0, e1 = tl[i]
    gs = f"gemm[{i}] {(g0 - t0) / 1e3:8.1f} .. {(g1 - t0) / 1e3:8.1f} ({(g1 - g0) / 1e3:6.1f})" if g0 < 1e30 else ""
    es = f"ess[{i}] {(e0 - t0) / 1e3:8.1f} .. {(e1 - t0) / 1e3:8.1f} ({(e1 - e0) / 1e3:6.1f})" if e0 < 1e30 else ""
    print(f"  {gs:44s} {es}")

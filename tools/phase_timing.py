"""Per-phase cycle breakdown of ess_kernel (timing build; tooling, not a bench number).
usage: python tools/phase_timing.py [config] [iters]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
tm.LIB_PATH = os.environ.get("TIMING_LIB", os.path.join(ROOT, "build", "libtmvn_timing.so"))
L = tm.lib()
L.tmvn_test_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
if os.environ.get("PAPER_D"):  # the S4.2 geometry (synth.paper_random) with PAPER_C chains
    import dataclasses
    dd = int(os.environ["PAPER_D"])
    A, b, x0 = synth.paper_random(dd, seed=dd)
    cfg = dataclasses.replace(cfg, C=int(os.environ.get("PAPER_C", "20")))
s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"), latency=0)
s.set_options(streams=1, chain_warps=int(os.environ.get("W", "0")), buckets=int(os.environ.get("BUCKETS", "0")))
X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
s.sample(X, 40, cfg.chain_seed, out=X)
buf = np.zeros(14, dtype=np.uint64)
L.tmvn_test_phase_cycles(buf.ctypes.data_as(ctypes.c_void_p), 1)
s.sample(X, iters, cfg.chain_seed, out=X)
L.tmvn_test_phase_cycles(buf.ctypes.data_as(ctypes.c_void_p), 0)
names = ["init", "A2 arcs+stats", "lo-word pass", "B intervals", "C theta", "D1 P'+safeguard",
         "D2 x/moments/nu"]
nchain = cfg.C * iters
tot = float(sum(buf[:7])) + float(buf[10])
print(f"config {k}: {nchain} chain-iterations; mean active arcs {buf[8]/nchain:.1f}, gaps {buf[9]/nchain:.2f}, general path {buf[7]/nchain:.3f}")
print(f"  {'A1 active+compact':18s} {buf[10]/nchain:10.0f} cycles/chain  {100*buf[10]/tot:5.1f}%")
for i, n in enumerate(names):
    print(f"  {n:18s} {buf[i]/nchain:10.0f} cycles/chain  {100*buf[i]/tot:5.1f}%")

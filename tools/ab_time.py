"""Quick A/B timing of tmvn_sample for several library builds and chain_warps (tooling).
usage: python tools/ab_time.py config W[,W..] S[,S..] R[,R..] lib1.so [lib2.so ...]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
k = int(sys.argv[1])
Ws = [int(w) for w in sys.argv[2].split(",")]
Ss = [int(x) for x in sys.argv[3].split(",")]
Rs = [int(x) for x in sys.argv[4].split(",")]
cfg = synth.CONFIGS[k]
A, b, x0 = synth.make_instance(k)
iters = int(os.environ.get("ITERS", "400" if k in (2, 3) else "20"))
reps = int(os.environ.get("REPS", "2"))
for path in sys.argv[5:] * reps:
    tm._LIB = None
    tm.LIB_PATH = os.path.abspath(path)
    for W, S, R in [(w, x, r) for w in Ws for x in Ss for r in Rs]:
        s = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"))
        s.set_options(profile=int(os.environ.get("PROFILE", "1")), chain_warps=W, streams=S, ring=R,
                      rng_ahead=int(os.environ.get("RNG_AHEAD", "0")), schedule=int(os.environ.get("SCHED", "0")),
                      pipeline=int(os.environ.get("PIPE", "0")), latency=int(os.environ.get("LATENCY", "0")),
                      record=int(os.environ.get("RECORD", "1")))
        if "GRAPHS" in os.environ:
            s.set_options(graphs=int(os.environ["GRAPHS"]))
        if "OVL" in os.environ:
            s.set_options(rng_overlap=int(os.environ["OVL"]))
        if "RNG_GEMM" in os.environ:
            s.set_options(rng_gemm=int(os.environ["RNG_GEMM"]))
        if "WARP" in os.environ:
            s.set_options(warp_mode=int(os.environ["WARP"]), small_warps=int(os.environ.get("SW", "0")))
        if "BUCKETS" in os.environ:
            s.set_options(buckets=int(os.environ["BUCKETS"]))
        if "FUSE" in os.environ:
            s.set_options(fuse_arcs=int(os.environ["FUSE"]))
        X = torch.tensor(np.tile(x0, (cfg.C, 1)), device="cuda")
        s.sample(X, int(os.environ.get("WARM", "200" if k in (2, 3) else "10")), cfg.chain_seed, out=X)
        s.reset_stats()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.sample(X, iters, cfg.chain_seed, out=X)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        pr = s.profile()
        print(f"{os.path.basename(path)} g={os.environ.get('GRAPHS', '-')} ovl={os.environ.get('OVL', '-')} rg={os.environ.get('RNG_GEMM', '-')} fuse={os.environ.get('FUSE', '-')} bk={os.environ.get('BUCKETS', '-')} warp={os.environ.get('WARP', '-')}/{os.environ.get('SW', '-')} rec={os.environ.get('RECORD', '1')} rng_ahead={os.environ.get('RNG_AHEAD', '0')} sched={os.environ.get('SCHED', '0')} pipe={os.environ.get('PIPE', '0')} lat={os.environ.get('LATENCY', '0')} W={W} S={S} R={R} cfg{k}: {dt/iters*1e3:.3f} ms/iter  gemm "
              f"{pr['gemm_ms']/max(1,pr['gemm_launches']):.3f} ms  tc {pr['tc_ms']/max(1,pr['tc_launches']):.3f} ms"
              f"  ess {pr['ess_ms']/max(1,pr['ess_launches']):.3f} ms"
              f"  evals/s {cfg.C*cfg.m*iters/dt:.3e}  l1={pr['buckets_used']}", flush=True)
        s.close()

"""Small runs of every production kernel for compute-sanitizer (tooling)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
for k, kw, C in [(3, dict(m=300, d=150), 200), (4, dict(m=6000, d=40), 40), (2, dict(), 130)]:
    A, b, x0 = synth.make_instance(k, **kw)
    for opts in (dict(), dict(projection=2), dict(pipeline=1), dict(rng_ahead=1)):
        s = tm.Sampler(A, b, **opts)
        X = s.sample(np.tile(x0, (C, 1)), 40, seed=5)
        assert s.stats()["rejections"] == 0
        s.close()
print(tm.test_ozaki_gemm(np.random.default_rng(0).standard_normal((70, 100)),
                         np.random.default_rng(1).standard_normal((130, 100)), 7)[0, :2])
print("ok")

"""The paper's own workloads through the library.

S4.2: A d x d iid N(0,1) (not normalised), x0 ~ N(0, I),
b = A x0 + U[0,1]^d, run as 1 chain x T steps and 10 chains x T/10 steps, no
burn-in; "No rejection occurs".  Checked here: every iterate feasible
under fresh FP64 dot products, zero rejections, and per-step parity with the
oracle along the traced trajectory.
"""
import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,chains,steps", [(300, 1, 400), (300, 10, 40), (1000, 10, 20)])
def test_section_4_2_instances(d, chains, steps):
    A, b, x0 = synth.paper_random(d, seed=d)
    s = tm.Sampler(A, b)
    trace, out = s.test_trace(np.tile(x0, (chains, 1)), steps, seed=42, chains=np.arange(chains))
    assert s.stats()["rejections"] == 0
    for it in range(steps + 1):
        slack = trace[it] @ A.T - b
        assert np.max(slack) <= 0.0
    rng = np.random.default_rng(0)
    for it in rng.choice(steps, size=min(steps, 12), replace=False):
        c = int(rng.integers(chains))
        xn, _ = oracle.step(A, b, trace[it, c], 42, int(it), c)
        assert np.max(np.abs(trace[it + 1, c] - xn)) <= 1e-10 * max(1.0, np.max(np.abs(xn)))

"""Constraint-parallel iterations (cp.cu + paper_2407_10449_b200.cp):
rows of A split over ranks, three collectives per iteration.  One rank against the
oracle step by step; two ranks (processes on one GPU, gloo host-driven collectives)
bitwise against one rank -- Prop. 1's associativity plus the fixed
per-element order of the projection make the split invisible."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cp_single_rank_steps_vs_oracle():
    A, b, x0 = synth.paper_random(150, seed=3)
    C = 9
    cp = tm.ConstraintParallel(A, b, record=0)
    X = np.tile(x0, (C, 1))
    for t in range(6):
        Xn = cp.sample(X, 1, seed=21).cpu().numpy()
        for c in range(C):
            xn, _ = oracle.step(A, b, X[c], 21, t, c)
            assert np.max(np.abs(Xn[c] - xn)) <= 1e-10 * max(1.0, np.max(np.abs(xn))), (t, c)
        X = Xn
    assert cp.stats()["steps"] == C * 6


def test_cp_matches_the_throughput_path():
    """Same readings as tmvn_sample: over 30 iterations the chains agree with the
    default path to rounding (both FP64-accurate; different interval code)."""
    A, b, x0 = synth.make_instance(3, m=300, d=60)
    X0 = np.tile(x0, (20, 1))
    ref = tm.Sampler(A, b, latency=0).sample(X0, 30, seed=5)
    out = tm.ConstraintParallel(A, b).sample(X0, 30, seed=5).cpu().numpy()
    assert np.max(np.abs(out - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_cp_two_ranks_bitwise_equal_one_rank():
    with tempfile.TemporaryDirectory() as td:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "tools", "cp_check.py"), td]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        out2 = np.load(os.path.join(td, "out.npy"))
        mom2 = np.load(os.path.join(td, "mom.npy"))
    A, b, x0 = synth.paper_random(200, seed=7)
    cp = tm.ConstraintParallel(A, b, burn_in=3)
    out1 = cp.sample(np.tile(x0, (12, 1)), 40, seed=11).cpu().numpy()
    assert np.array_equal(out1, out2)
    sm, sq, n = cp.moments()
    assert np.array_equal(np.concatenate([sm, sq, [n, cp.stats()["rejections"]]]), mom2)


def test_cp_resume_and_trim():
    """A call split at a multiple of recompute_every resumes bitwise (iter_offset
    auto-advances); the trim epsilon (C7) follows the oracle step."""
    A, b, x0 = synth.make_instance(3, m=200, d=40)
    X0 = np.tile(x0, (7, 1))
    full = tm.ConstraintParallel(A, b).sample(X0, 64, seed=9).cpu().numpy()
    cp = tm.ConstraintParallel(A, b)
    a = cp.sample(X0, 32, seed=9)
    a = cp.sample(a, 32, seed=9).cpu().numpy()
    assert np.array_equal(a, full)
    eps = 1e-3
    ct = tm.ConstraintParallel(A, b, trim_eps=eps, record=0)
    X = X0.copy()
    for t in range(4):
        Xn = ct.sample(X, 1, seed=9).cpu().numpy()
        for c in range(7):
            xn, _ = oracle.step(A, b, X[c], 9, t, c, eps=eps)
            assert np.max(np.abs(Xn[c] - xn)) <= 1e-10 * max(1.0, np.max(np.abs(xn)))
        X = Xn

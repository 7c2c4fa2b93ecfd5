"""Pins for the oracle's counter-based RNG (reading C12): Philox4x32-10 and Box-Muller.

Philox is pinned to (a) the Random123 known-answer vectors published with the
generator (Salmon et al., SC'11) and (b) cuRAND's own ``curand_Philox4x32_10``
compiled for the host from the CUDA toolkit header -- an implementation that is
independent of both the oracle and the CUDA path.  The normals and uniforms are
pinned by their distributions (textbook moments and a KS test).
"""
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

# Random123 kat_vectors, philox4x32 with 10 rounds: (ctr, key) -> out.
KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    assert list(oracle.philox4x32_10(ctr, key)) == want


def test_philox_matches_curand_host():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    here = os.path.dirname(os.path.abspath(__file__))
    src = os.path.join(here, "pins", "curand_host_philox.cu")
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "cph")
        subprocess.check_call([nvcc, "-x", "cu", "-O2", "-Wno-deprecated-gpu-targets", "-o", exe, src])
        rng = np.random.default_rng(7)
        inp = rng.integers(0, 2**32, size=(4000, 6), dtype=np.uint64).astype(np.uint32)
        inp[:50, 1:4] = 0  # small counters, as the sampler uses them
        inp.tofile(os.path.join(td, "in.bin"))
        subprocess.check_call([exe, os.path.join(td, "in.bin"), os.path.join(td, "out.bin")])
        ref = np.fromfile(os.path.join(td, "out.bin"), dtype=np.uint32).reshape(-1, 4)
    mine = np.stack([oracle.philox4x32_10(r[:4], r[4:]) for r in inp])
    assert np.array_equal(ref, mine)


def test_counter_layout():
    """C12: block (j, t, c, s) is Philox(ctr = (j, t, c, s), key = (seed_lo, seed_hi))."""
    seed = 0x0123456789ABCDEF
    w = oracle.philox_block(seed, 5, 17, 99, 1)
    want = oracle.philox4x32_10([5, 17, 99, 1], [seed & 0xFFFFFFFF, seed >> 32])
    assert np.array_equal(w, want)
    # u is U_a of block (0, t, c, 1)
    w = oracle.philox_block(seed, 0, 17, 99, 1)
    bits = (int(w[1]) << 32) | int(w[0])
    assert oracle.uniform(seed, 17, 99) == (bits >> 11) * 2.0**-53


def test_normals_box_muller_closed_form():
    """nu_{2j} = R cos(phi), nu_{2j+1} = R sin(phi), R = sqrt(-2 log(1-U_a)), phi = 2 pi U_b."""
    seed, t, c, d = 42, 3, 11, 7
    nu = oracle.normals(seed, t, c, d)
    for j in range(4):
        w = oracle.philox_block(seed, j, t, c, 0)
        ua = ((int(w[1]) << 32 | int(w[0])) >> 11) * 2.0**-53
        ub = ((int(w[3]) << 32 | int(w[2])) >> 11) * 2.0**-53
        R = math.sqrt(-2.0 * math.log(1.0 - ua))
        phi = 6.283185307179586 * ub
        assert abs(nu[2 * j] - R * math.cos(phi)) <= 4 * np.spacing(abs(R))
        if 2 * j + 1 < d:
            assert abs(nu[2 * j + 1] - R * math.sin(phi)) <= 4 * np.spacing(abs(R))


def _norm_cdf(x):
    return 0.5 * (1.0 + np.vectorize(math.erf)(x / math.sqrt(2.0)))


def test_normals_distribution():
    d = 2000
    xs = np.concatenate([oracle.normals(9, t, c, d) for t in range(10) for c in range(10)])
    n = xs.size  # 2e5
    assert abs(xs.mean()) < 5 / math.sqrt(n)
    assert abs(xs.var() - 1.0) < 5 * math.sqrt(2.0 / n)
    s = np.sort(xs)
    ecdf = np.arange(1, n + 1) / n
    ks = np.max(np.abs(ecdf - _norm_cdf(s)))
    assert ks < 1.95 / math.sqrt(n)  # KS at ~0.1 %
    # different chains / iterations / seeds give different streams
    assert not np.array_equal(oracle.normals(9, 0, 0, 8), oracle.normals(9, 0, 1, 8))
    assert not np.array_equal(oracle.normals(9, 0, 0, 8), oracle.normals(9, 1, 0, 8))
    assert not np.array_equal(oracle.normals(9, 0, 0, 8), oracle.normals(10, 0, 0, 8))


def test_uniform_distribution():
    us = np.array([oracle.uniform(5, t, c) for t in range(100) for c in range(200)])
    assert us.min() >= 0.0 and us.max() < 1.0
    n = us.size
    s = np.sort(us)
    ks = np.max(np.abs(np.arange(1, n + 1) / n - s))
    assert ks < 1.95 / math.sqrt(n)

"""CPU tests of the C ABI: libgt.so loads and exports every function include/gt.h declares; the
host-only planning entry points agree with the oracle (bit-exact) and with the paper's algebra
(Eq. 7/8, Eq. 13/14, Alg. 3; SPEC examples S:464-506)."""
import os
import re
import subprocess

import numpy as np
import pytest

import gtgen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gt():
    from paper_2604_16715_b200 import _build
    _build.build()
    import paper_2604_16715_b200 as g
    g.lib()
    return g


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gt_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(gt):
    names = declared_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", gt.gt.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gt_[a-z0-9_]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(gt.lib(), n)  # resolvable through ctypes


def test_library_is_sm100a(gt):
    out = subprocess.run(["cuobjdump", "--list-elf", gt.gt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_partition_halo_send_lists_match_oracle(gt, seed, p):
    rp, ci = gtgen.random_graph(400 + 37 * seed, 3000 + 500 * seed, seed=300 + seed, directed=bool(seed % 2),
                                power=2.2)
    for mode in (0, 1):
        b = gt.partition(rp, p, mode)
        np.testing.assert_array_equal(b, oracle.partition(rp, p, mode))
    b = oracle.partition(rp, p)
    for r in range(p):
        lo, hi = int(b[r]), int(b[r + 1])
        ho = oracle.halo(rp, ci, lo, hi)
        hi_ = oracle.halo(rp, ci, lo, hi, inward=True)
        np.testing.assert_array_equal(gt.halo(rp, ci, lo, hi), ho)
        np.testing.assert_array_equal(gt.halo(rp, ci, lo, hi, inward=True), hi_)
        for s in range(p):
            if s == r:
                continue
            # what s sends to r == r's halo restricted to s's rows
            np.testing.assert_array_equal(gt.send_list(rp, ci, b[s], b[s + 1], lo, hi), oracle.send_list(ho, b, s))
            np.testing.assert_array_equal(gt.send_list(rp, ci, b[s], b[s + 1], lo, hi, inward=True),
                                          oracle.send_list(hi_, b, s))


def test_estimate_iter_time_spec_example(gt):
    # alpha(1)=2e-9 s/edge, E=1e6, N=1e5; p=1 -> alpha E; p=2 with beta_c(2)=1e-9 -> 1e-3 + 1e-4
    beta = np.zeros((2, 3))
    beta[0, 2] = 1e-9
    assert gt.estimate_iter_time(2e-9, beta, 0, 1, 1e5, 1e6) == pytest.approx(2e-3, rel=1e-15)
    assert gt.estimate_iter_time(2e-9, beta, 0, 2, 1e5, 1e6) == pytest.approx(1.1e-3, rel=1e-12)
    # doubling E doubles only the compute term
    t1 = gt.estimate_iter_time(2e-9, beta, 0, 2, 1e5, 2e6)
    assert t1 - 1e-4 == pytest.approx(2 * (1.1e-3 - 1e-4), rel=1e-12)


def test_agp_select_examples_and_bruteforce(gt):
    # P = 1 -> single GPU
    assert gt.agp_select(1e5, 1.0, np.zeros((2, 2)))[0] == -1
    # GP-A2A-like strategy 1 with much smaller beta at 8 -> (1, 8)
    beta = np.zeros((2, 9))
    beta[0, 2:] = 5e-7
    beta[1, 2:] = 5e-7
    beta[1, 8] = 1e-8
    c, s, sc = gt.agp_select(1e5, 1.0, beta)
    assert (c, s) == (1, 8) and sc == pytest.approx(8 * 1e-8 / 7)
    # k below every score -> single GPU
    assert gt.agp_select(1e5, 1e-9, beta)[:2] == (-1, 1)
    # exhaustive enumeration of Alg. 3 on random profiles; scale invariance
    rng = np.random.default_rng(0)
    for _ in range(300):
        P = int(rng.integers(1, 9))
        B = rng.uniform(1e-9, 1e-6, size=(3, P + 1))
        N, t1 = float(rng.uniform(1e3, 1e7)), float(rng.uniform(1e-3, 10))
        k = t1 / N
        best = None
        for i in range(2, P + 1):
            for cc in range(3):
                score = i * B[cc, i] / (i - 1)
                if score <= k and (best is None or score < best[0]):
                    best = (score, cc, i)
        got = gt.agp_select(N, t1, B)
        if best is None:
            assert got[:2] == (-1, 1)
        else:
            assert got[:2] == (best[1], best[2])
        assert gt.agp_select(N, t1 * 7.0, B * 7.0)[:2] == got[:2]
        # Eq. 13 at p = 1 is exactly the comparison of Eq. 7 times:
        # s beta_c(s) / (s - 1) <= k  <=>  t_iter(s) <= t_iter(1)  with alpha(1) E = t_iter(1)
        for i in range(2, P + 1):
            E = 1e6
            alpha1 = t1 / E
            lhs = i * B[0, i] / (i - 1) <= k
            rhs = gt.estimate_iter_time(alpha1, B, 0, i, N, E) <= gt.estimate_iter_time(alpha1, B, 0, 1, N, E)
            if abs(i * B[0, i] / (i - 1) - k) > 1e-12 * k:
                assert lhs == rhs


def test_fit_beta(gt):
    x = np.array([1e3, 1e4, 1e5, 1e6])
    assert gt.fit_beta(x, 3e-9 * x) == pytest.approx(3e-9, rel=1e-12)
    t = 2e-5 + 3e-9 * np.array([1e7, 1e8, 1e9, 1e10])  # latency offset, sizes >> L/b
    assert gt.fit_beta(np.array([1e7, 1e8, 1e9, 1e10]), t) == pytest.approx(3e-9, rel=0.05)
    with pytest.raises(gt.GTError):
        gt.fit_beta(np.array([1.0]), np.array([1.0]))

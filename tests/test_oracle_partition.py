"""Pins for the oracle's partition and halo sets (integer, bit-exact).

Hand cases: SURVEY.md section 8(c) P6 (computed there by an independent script) using reading Z9
(W(i) = row_ptr[i] + i); SPEC.md S:261-262 for the node-balanced rule.  Brute force: every
bound is the minimum i satisfying the definition, found by exhaustive search; halos by Python sets.
"""
import math

import numpy as np
import pytest

import gtgen
import oracle


def path_graph(n):
    pairs = [(i, i + 1) for i in range(n - 1)] + [(i + 1, i) for i in range(n - 1)]
    return gtgen.csr_from_pairs(n, pairs)


def star_graph(n):
    pairs = [(0, j) for j in range(1, n)] + [(j, 0) for j in range(1, n)]
    return gtgen.csr_from_pairs(n, pairs)


def halos(rp, ci, bounds):
    p = len(bounds) - 1
    return [oracle.halo(rp, ci, bounds[r], bounds[r + 1]).tolist() for r in range(p)]


def test_path_graph_hand_case():
    rp, ci = path_graph(8)
    assert rp.tolist() == [0, 1, 3, 5, 7, 9, 11, 13, 14]
    b2 = oracle.partition(rp, 2)
    assert b2.tolist() == [0, 4, 8]
    assert halos(rp, ci, b2) == [[4], [3]]
    h = halos(rp, ci, b2)
    assert oracle.send_list(np.array(h[0]), b2, 1).tolist() == [4]  # send 1 -> 0
    assert oracle.send_list(np.array(h[1]), b2, 0).tolist() == [3]  # send 0 -> 1
    b3 = oracle.partition(rp, 3)
    assert b3.tolist() == [0, 3, 6, 8]
    assert halos(rp, ci, b3) == [[3], [2, 6], [5]]


def test_star_graph_hand_case():
    rp, ci = star_graph(8)
    b2 = oracle.partition(rp, 2)
    assert b2.tolist() == [0, 3, 8]
    assert halos(rp, ci, b2) == [[3, 4, 5, 6, 7], [0]]
    b3 = oracle.partition(rp, 3)
    assert b3.tolist() == [0, 1, 5, 8]
    h = halos(rp, ci, b3)
    assert h == [[1, 2, 3, 4, 5, 6, 7], [0], [0]]
    assert oracle.send_list(np.array(h[0]), b3, 1).tolist() == [1, 2, 3, 4]
    assert oracle.send_list(np.array(h[0]), b3, 2).tolist() == [5, 6, 7]


def test_empty_graph_more_ranks_than_rows():
    rp = np.zeros(4, np.int64)
    assert oracle.partition(rp, 5).tolist() == [0, 1, 2, 2, 3, 3]


def test_spec_node_balanced():
    assert oracle.partition(np.zeros(9, np.int64), 2, mode=1).tolist() == [0, 4, 8]
    assert oracle.partition(np.zeros(8, np.int64), 3, mode=1).tolist() == [0, 3, 5, 7]
    assert oracle.partition(np.zeros(6, np.int64), 1, mode=1).tolist() == [0, 5]


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_bruteforce_partition_and_halo(seed, p):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    m = int(rng.integers(0, n * 4))
    m = min(m, n * (n - 1))
    rp, ci = gtgen.random_graph(n, m, 100 + seed, directed=bool(seed % 2)) if m else (
        np.zeros(n + 1, np.int64), np.zeros(0, np.int32))
    E = int(rp[-1])
    b = oracle.partition(rp, p).tolist()
    W = [int(rp[i]) + i for i in range(n + 1)]
    exp = [0]
    for r in range(1, p):
        target = math.ceil(r * (E + n) / p)
        exp.append(min(i for i in range(n + 1) if W[i] >= target))
    exp.append(n)
    assert b == exp
    edges = [(i, int(ci[e])) for i in range(n) for e in range(rp[i], rp[i + 1])]
    for r in range(p):
        lo, hi = b[r], b[r + 1]
        out_h = sorted({j for (i, j) in edges if lo <= i < hi and not lo <= j < hi})
        in_h = sorted({i for (i, j) in edges if lo <= j < hi and not lo <= i < hi})
        assert oracle.halo(rp, ci, lo, hi).tolist() == out_h
        assert oracle.halo(rp, ci, lo, hi, inward=True).tolist() == in_h


def test_symmetric_graph_in_halo_equals_out_halo():
    rp, ci = gtgen.random_graph(300, 1200, 7, directed=False, power=2.2)
    b = oracle.partition(rp, 4)
    for r in range(4):
        np.testing.assert_array_equal(oracle.halo(rp, ci, b[r], b[r + 1]),
                                      oracle.halo(rp, ci, b[r], b[r + 1], inward=True))

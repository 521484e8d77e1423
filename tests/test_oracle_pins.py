"""Pins of the oracle (oracle/oracle.c) to things other than itself.

SURVEY.md 8(c) "Pins": hand-worked examples (tests/golden/worked_examples.json),
closed forms, the PageRank mass invariant, union-find / Dijkstra / BFS / hop-
bounded brute force and scipy library routines.  CPU only.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import checkers

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")
with open(GOLDEN) as f:
    WORKED = json.load(f)


def _frac(s):
    return Fraction(s)


def _u32(s):
    return oracle.INF if s == "INF" else int(s)


def _edges(case):
    e = np.array(case["edges"], dtype=np.int64).reshape(-1, 3 if "source" in case else 2)
    return e


# ---------------------------------------------------------------- PageRank

@pytest.mark.parametrize("case", WORKED["pagerank"], ids=lambda c: c["name"])
def test_pagerank_worked_examples(case):
    e = _edges(case)
    r = oracle.pagerank(case["n"], e[:, 0], e[:, 1], k=case["k"])
    want = np.array([float(_frac(v)) for v in case["values"]])
    assert r["status"] == oracle.OK
    assert r["supersteps"] == case["supersteps"]
    np.testing.assert_allclose(r["values"], want, rtol=1e-15, atol=0)


@pytest.mark.parametrize("case", WORKED["pagerank"], ids=lambda c: c["name"])
def test_pagerank_golden_matches_exact_recursion(case):
    # the golden fixtures themselves agree with the exact-rational definition
    e = [tuple(x) for x in case["edges"]]
    exact = checkers.pagerank_exact(case["n"], e, case["k"])
    assert [str(x) for x in exact] == [str(_frac(v)) for v in case["values"]]


@pytest.mark.parametrize("n", [3, 7, 64])
def test_pagerank_cycle_closed_form(n):
    src = np.arange(n)
    dst = (src + 1) % n
    for k in (1, 2, 10):
        r = oracle.pagerank(n, src, dst, k=k)
        np.testing.assert_allclose(r["values"], 1.0 / n, rtol=1e-14)


@pytest.mark.parametrize("n", [2, 5, 17])
def test_pagerank_complete_digraph_closed_form(n):
    s, d = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    keep = s != d
    r = oracle.pagerank(n, s[keep], d[keep], k=10)
    np.testing.assert_allclose(r["values"], 1.0 / n, rtol=1e-13)


@pytest.mark.parametrize("n", [5, 1000, 1 << 16])
def test_pagerank_in_star_closed_form(n):
    leaves = np.arange(1, n)
    for k in (1, 2, 5):
        r = oracle.pagerank(n, leaves, np.zeros(n - 1, dtype=np.int64), k=k)
        c = 0.15 / n + 0.85 * (n - 1) / n if k == 1 else (0.15 / n) * (1 + 0.85 * (n - 1))
        assert r["values"][0] == pytest.approx(c, rel=1e-12)
        np.testing.assert_allclose(r["values"][1:], 0.15 / n, rtol=1e-15)


@pytest.mark.parametrize("n", [5, 1000])
def test_pagerank_out_star_closed_form(n):
    leaves = np.arange(1, n)
    for k in (1, 2, 4):
        r = oracle.pagerank(n, np.zeros(n - 1, dtype=np.int64), leaves, k=k)
        prev0 = 1.0 / n if k == 1 else 0.15 / n
        assert r["values"][0] == pytest.approx(0.15 / n, rel=1e-15)
        np.testing.assert_allclose(r["values"][1:], 0.15 / n + 0.85 * prev0 / (n - 1), rtol=1e-13)


def test_pagerank_mass_invariant_per_superstep():
    # sum_v r_t(v) = 0.15 + 0.85 * sum_{u: outdeg(u)>0} r_{t-1}(u)   (exact identity)
    rng = np.random.default_rng(7)
    n = 300
    src, dst, _ = checkers.random_graph(rng, n, 2000)
    outdeg = np.bincount(src, minlength=n)
    prev = oracle.pagerank(n, src, dst, k=0)["values"]
    for k in range(1, 8):
        cur = oracle.pagerank(n, src, dst, k=k)["values"]
        lhs = math.fsum(cur)
        rhs = 0.15 + 0.85 * math.fsum(prev[outdeg > 0])
        assert lhs == pytest.approx(rhs, rel=1e-13)
        prev = cur


def test_pagerank_counters_and_superstep_count():
    rng = np.random.default_rng(3)
    n = 200
    src, dst, _ = checkers.random_graph(rng, n, 900)
    r = oracle.pagerank(n, src, dst, k=10)
    assert r["supersteps"] == 11  # Fig. 8: halts at superstep 10
    nondangling = int((np.bincount(src, minlength=n) > 0).sum())
    assert list(r["changed"]) == [nondangling] * 10 + [0]
    assert list(r["messages"]) == [len(src)] * 10 + [0]
    assert list(r["ran"]) == [n] * 11


@pytest.mark.parametrize("seed", range(6))
def test_pagerank_random_vs_exact_and_scipy(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 60))
    m = int(rng.integers(0, 4 * n))
    src, dst, _ = checkers.random_graph(rng, n, m)
    k = [0, 1, 3, 10][seed % 4]
    r = oracle.pagerank(n, src, dst, k=k)["values"]
    exact = checkers.pagerank_exact(n, list(zip(src.tolist(), dst.tolist())), k)
    np.testing.assert_allclose(r, [float(x) for x in exact], rtol=1e-14, atol=0)
    np.testing.assert_allclose(r, checkers.pagerank_scipy(n, src, dst, k), rtol=1e-13)


def test_pagerank_rmat_vs_scipy():
    import inputs
    src, dst, _ = inputs.rmat_coo(14, 16, 1)
    r = oracle.pagerank(1 << 14, src, dst, k=10)["values"]
    ref = checkers.pagerank_scipy(1 << 14, src, dst, 10)
    assert np.max(np.abs(r - ref)) < 1e-15
    assert np.max(np.abs(r - ref) / ref) < 1e-12


# ------------------------------------------------- PageRank to convergence (reading R27)
# "a PageRank application would typically run until convergence"; the master
# halts after the first superstep s >= 1 with max_v |r_s(v) - r_{s-1}(v)| <= tol.

@pytest.mark.parametrize("n", [3, 64])
def test_pagerank_tol_cycle_stops_at_once(n):
    src = np.arange(n)
    dst = (src + 1) % n
    r = oracle.pagerank(n, src, dst, k=50, tol=1e-12)
    assert r["supersteps"] == 2                       # r_1 = r_0 = 1/n (up to one rounding)
    assert r["delta"][1] <= 2.0 ** -52 / n
    np.testing.assert_allclose(r["values"], 1.0 / n, rtol=1e-15)
    assert list(r["messages"]) == [n, n]              # the last broadcast is never delivered


@pytest.mark.parametrize("n", [5, 1000])
def test_pagerank_tol_in_star_closed_form(n):
    # in-star (leaves -> 0): r_1 = (0.15/n + 0.85 (n-1)/n, 0.15/n ...),
    # r_2 = ((0.15/n)(1 + 0.85 (n-1)), 0.15/n ...), r_3 = r_2 exactly: delta_3 = 0
    leaves = np.arange(1, n)
    r = oracle.pagerank(n, leaves, np.zeros(n - 1, dtype=np.int64), k=10, tol=0.0)
    assert r["supersteps"] == 4
    c1 = 0.15 / n + 0.85 * (n - 1) / n
    c2 = (0.15 / n) * (1 + 0.85 * (n - 1))
    d1 = max(abs(c1 - 1.0 / n), abs(0.15 / n - 1.0 / n))
    assert r["delta"][1] == pytest.approx(d1, rel=1e-13)
    assert r["delta"][2] == pytest.approx(abs(c2 - c1), rel=1e-13)
    assert r["delta"][3] == 0.0
    assert r["values"][0] == pytest.approx(c2, rel=1e-13)


@pytest.mark.parametrize("seed", range(4))
def test_pagerank_tol_random_vs_exact(seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(5, 40))
    src, dst, _ = checkers.random_graph(rng, n, int(rng.integers(n, 5 * n)))
    kmax = 25
    traj = checkers.pagerank_exact_trajectory(n, list(zip(src.tolist(), dst.tolist())), kmax)
    dex = [0.0] + [float(max(abs(a - b) for a, b in zip(traj[t], traj[t - 1])))
                   for t in range(1, kmax + 1)]
    full = oracle.pagerank(n, src, dst, k=kmax, tol=-1.0)
    # delta is the difference of two f64 iterates: error <= a few ulps of the ranks
    np.testing.assert_allclose(full["delta"][1:kmax + 1], dex[1:], rtol=0, atol=1e-15)
    # a tolerance halfway (geometrically) between two well-separated deltas
    cand = [t for t in range(2, kmax) if dex[t] > 0 and dex[t] < 0.5 * dex[t - 1] and dex[t] > 1e-12]
    if not cand:
        return
    t = cand[len(cand) // 2]
    tol = math.sqrt(dex[t] * dex[t - 1])
    first = next(s for s in range(1, kmax + 1) if dex[s] <= tol)
    r = oracle.pagerank(n, src, dst, k=kmax, tol=tol)
    assert r["supersteps"] == first + 1
    np.testing.assert_allclose(r["values"], [float(x) for x in traj[first]], rtol=1e-14, atol=0)


def test_pagerank_tol_capped_by_k_and_off_is_fig8():
    rng = np.random.default_rng(5)
    n = 100
    src, dst, _ = checkers.random_graph(rng, n, 600)
    a = oracle.pagerank(n, src, dst, k=10)
    b = oracle.pagerank(n, src, dst, k=10, tol=-1.0)
    c = oracle.pagerank(n, src, dst, k=10, tol=1e-300)   # never reached: Fig. 8's k wins
    for r in (b, c):
        np.testing.assert_array_equal(r["values"], a["values"])
        assert r["supersteps"] == 11 and r["messages"][-1] == 0


# ---------------------------------------------------------------- Hash-Min CC

@pytest.mark.parametrize("case", WORKED["cc"], ids=lambda c: c["name"])
def test_cc_worked_examples(case):
    e = _edges(case)
    n = case["n"]
    r = oracle.hashmin_cc(n, e[:, 0], e[:, 1])
    if "trajectory" in case:
        for s, want in enumerate(case["trajectory"]):
            g = oracle.hashmin_cc(n, e[:, 0], e[:, 1], max_supersteps=s + 1)
            assert list(g["values"]) == want, s
        assert list(r["values"]) == case["trajectory"][-1]
    else:
        assert list(r["values"]) == case["values"]
    if "supersteps" in case:
        assert r["supersteps"] == case["supersteps"]
    if "changed" in case:
        assert list(r["changed"]) == case["changed"]
        assert list(r["messages"]) == case["messages"]


@pytest.mark.parametrize("seed", range(8))
def test_cc_random_vs_union_find_and_balls(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(1, 120))
    m = int(rng.integers(0, 2 * n))
    src, dst, _ = checkers.random_graph(rng, n, m, self_loops=bool(seed % 2))
    edges = list(zip(src.tolist(), dst.tolist()))
    r = oracle.hashmin_cc(n, src, dst)
    assert list(r["values"]) == checkers.cc_union_find(n, edges)
    np.testing.assert_array_equal(r["values"], checkers.cc_scipy(n, src, dst))
    deg_sym = np.bincount(src, minlength=n) + np.bincount(dst, minlength=n)
    prev = list(range(n))
    for s in range(r["supersteps"]):
        g = oracle.hashmin_cc(n, src, dst, max_supersteps=s + 1)
        ball = checkers.cc_ball_labels(n, edges, s)
        assert list(g["values"]) == ball
        if s > 0:
            ch = [v for v in range(n) if ball[v] < prev[v]]
            assert r["changed"][s] == len(ch)
            assert r["messages"][s] == int(deg_sym[ch].sum())
        prev = ball
    # termination: one more superstep than the last one with a change
    assert r["messages"][-1] == 0


def test_cc_rmat_vs_scipy():
    import inputs
    src, dst, _ = inputs.rmat_coo(16, 16, 2)
    r = oracle.hashmin_cc(1 << 16, src, dst)
    np.testing.assert_array_equal(r["values"], checkers.cc_scipy(1 << 16, src, dst))


# ---------------------------------------------------------------- SSSP

@pytest.mark.parametrize("case", WORKED["sssp"], ids=lambda c: c["name"])
def test_sssp_worked_examples(case):
    e = _edges(case)
    n = case["n"]
    r = oracle.sssp(n, e[:, 0], e[:, 1], e[:, 2], source=case["source"])
    if "trajectory" in case:
        for s, want in enumerate(case["trajectory"]):
            g = oracle.sssp(n, e[:, 0], e[:, 1], e[:, 2], source=case["source"], max_supersteps=s + 1)
            assert list(g["values"]) == [_u32(x) for x in want], s
        final = case["trajectory"][-1]
    else:
        final = case["values"]
    assert list(r["values"]) == [_u32(x) for x in final]
    assert r["supersteps"] == case["supersteps"]
    if "changed" in case:
        assert list(r["changed"]) == case["changed"]
        assert list(r["messages"]) == case["messages"]


def test_sssp_unit_weights_is_fig10_bfs():
    rng = np.random.default_rng(11)
    n = 150
    src, dst, _ = checkers.random_graph(rng, n, 400)
    want = checkers.bfs_levels(n, list(zip(src.tolist(), dst.tolist())), 0)
    r1 = oracle.sssp(n, src, dst, None, source=0)
    r2 = oracle.sssp(n, src, dst, np.ones(len(src), np.uint32), source=0)
    assert list(r1["values"]) == want
    assert list(r2["values"]) == want
    assert r1["supersteps"] == r2["supersteps"]


@pytest.mark.parametrize("seed", range(8))
def test_sssp_random_vs_dijkstra_and_hops(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 100))
    m = int(rng.integers(0, 4 * n))
    src, dst, w = checkers.random_graph(rng, n, m, weighted=True)
    source = int(rng.integers(0, n))
    edges = list(zip(src.tolist(), dst.tolist(), w.tolist()))
    r = oracle.sssp(n, src, dst, w, source=source)
    assert list(r["values"]) == checkers.dijkstra(n, edges, source)
    outdeg = np.bincount(src, minlength=n)
    prev = None
    for s in range(r["supersteps"]):
        g = oracle.sssp(n, src, dst, w, source=source, max_supersteps=s + 1)
        hop = checkers.hop_bounded(n, edges, source, s)
        assert list(g["values"]) == hop
        if prev is not None:
            ch = [v for v in range(n) if hop[v] < prev[v]]
            assert r["changed"][s] == len(ch)
            assert r["messages"][s] == int(outdeg[ch].sum())
        prev = hop


def test_sssp_rmat_vs_scipy_dijkstra():
    import inputs
    import scipy.sparse as sp
    from scipy.sparse.csgraph import dijkstra
    src, dst, w = inputs.rmat_coo(15, 16, 3, weighted=True)
    n = 1 << 15
    r = oracle.sssp(n, src, dst, w, source=0)
    # scipy's COO->CSR SUMS duplicates: min-deduplicate first
    key = src.astype(np.int64) * n + dst
    order = np.lexsort((w, key))
    key, ws = key[order], w[order]
    first = np.ones(len(key), bool)
    first[1:] = key[1:] != key[:-1]
    A = sp.csr_matrix((ws[first].astype(np.float64), (key[first] // n, key[first] % n)), shape=(n, n))
    d = dijkstra(A, indices=0)
    want = np.where(np.isinf(d), oracle.INF, d).astype(np.uint32)
    np.testing.assert_array_equal(r["values"], want)


def test_sssp_saturation_and_inf():
    # distances that would overflow saturate at INF and never improve anything
    n = 3
    src = np.array([0, 1])
    dst = np.array([1, 2])
    w = np.array([0xFFFFFFF0, 0x20], np.uint32)
    r = oracle.sssp(n, src, dst, w, source=0)
    assert list(r["values"]) == [0, 0xFFFFFFF0, oracle.INF]


# ---------------------------------------------------------------- engine rules

def test_guard_returns_partial_state():
    src = np.arange(9)
    dst = np.arange(1, 10)
    r = oracle.sssp(10, src, dst, None, source=0, max_supersteps=4)
    assert r["status"] == oracle.GUARD
    assert r["supersteps"] == 4
    assert list(r["values"][:5]) == [0, 1, 2, 3, oracle.INF]
    # exactly enough supersteps: no guard
    r = oracle.sssp(10, src, dst, None, source=0, max_supersteps=10)
    assert r["status"] == oracle.OK and r["supersteps"] == 10
    r = oracle.pagerank(10, src, dst, k=3, max_supersteps=3)
    assert r["status"] == oracle.GUARD
    r = oracle.pagerank(10, src, dst, k=3, max_supersteps=4)
    assert r["status"] == oracle.OK


def test_invalid_arguments():
    with pytest.raises(ValueError):
        oracle.sssp(3, np.array([0]), np.array([1]), None, source=3)
    with pytest.raises(ValueError):
        oracle.pagerank(3, np.array([0]), np.array([5]))
    with pytest.raises(ValueError):
        oracle.pagerank(3, np.array([0]), np.array([1]), max_supersteps=0)


def test_chain_superstep_count():
    # reading R16: an n-vertex unit chain runs n supersteps
    for n in (1, 2, 5, 50):
        src = np.arange(n - 1)
        r = oracle.sssp(n, src, src + 1, None, source=0)
        assert r["supersteps"] == n
        assert list(r["values"]) == list(range(n))

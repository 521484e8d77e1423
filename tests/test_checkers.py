"""CPU: the GPU-side PageRank mass check (tests/checkers.assert_pagerank_mass) accepts the exact
trajectory of Fig. 8's recursion and rejects one computed with an edge dropped or doubled."""
import numpy as np
import pytest

from tests import checkers


def sums(n, edges, k):
    outdeg = np.bincount(np.asarray([u for u, _ in edges], np.int64), minlength=n)
    traj = checkers.pagerank_exact_trajectory(n, edges, k)
    m = [float(sum(r)) for r in traj]
    nd = [float(sum(x for x, d in zip(r, outdeg) if d > 0)) for r in traj]
    return {"supersteps": k + 1, "pagerank_mass": m, "pagerank_mass_nd": nd}, \
        int(np.count_nonzero(outdeg))


def random_edges(seed, n=40, m=160):
    rng = np.random.default_rng(seed)
    e = [(int(u), int(v)) for u, v in zip(rng.integers(0, n, m), rng.integers(0, n, m)) if u != v]
    return n, e


@pytest.mark.parametrize("seed", range(5))
def test_mass_check_accepts_exact_trajectory(seed):
    n, e = random_edges(seed)
    st, nd = sums(n, e, 6)
    checkers.assert_pagerank_mass(st, n, nd)


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("fault", ["drop", "double"])
def test_mass_check_rejects_lost_or_extra_message(seed, fault):
    n, e = random_edges(seed)
    st, nd = sums(n, e, 6)
    # the faulty run: superstep 3 delivers with one edge dropped (or doubled) while the
    # out-degrees (the broadcast side) are those of the true graph
    outdeg = np.bincount(np.asarray([u for u, _ in e], np.int64), minlength=n)
    u0, v0 = e[seed % len(e)]
    traj = checkers.pagerank_exact_trajectory(n, e, 2)
    r2 = traj[2]
    acc = [0.0] * n
    for u, v in e:
        acc[v] += float(r2[u]) / outdeg[u]
    acc[v0] += (-1 if fault == "drop" else 1) * float(r2[u0]) / outdeg[u0]
    r3 = [0.15 / n + 0.85 * a for a in acc]
    bad = dict(st)
    bad["supersteps"] = 4
    bad["pagerank_mass"] = st["pagerank_mass"][:3] + [sum(r3)]
    bad["pagerank_mass_nd"] = st["pagerank_mass_nd"][:3] + [0.0]
    with pytest.raises(AssertionError):
        checkers.assert_pagerank_mass(bad, n, nd)

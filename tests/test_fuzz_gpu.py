"""Randomised parity sweep (GPU): skewed graphs (R-MAT plus planted hubs that span many
merge-path ranges), random weights including 0 and near-INF ones, random loopback partitioning,
exchange and direction mode; built-in apps and the paper's programs against the oracle
(bit-exact values and per-superstep counters for the min programs, the PR bar for PageRank)."""
import numpy as np
import pytest

import oracle
from tests.graphs import csr_csc, make_graph

pytestmark = pytest.mark.gpu

PR_ABS, PR_REL = 1e-9, 1e-11
_progs = {}


def prog(name):
    from paper_2010_08781_b200 import programs
    if name not in _progs:
        _progs[name] = programs.compile(name)
    return _progs[name]


def fuzz_graph(seed):
    import inputs
    rng = np.random.default_rng(9000 + seed)
    scale = int(rng.integers(4, 15))
    src, dst, _ = inputs.rmat_coo(scale, int(rng.integers(2, 17)), seed + 1, weighted=False)
    n = 1 << scale
    src, dst = [np.asarray(x, np.int64) for x in (src, dst)]
    if seed % 3 == 0:   # planted hub: one row spanning many ranges (fixup thread and warp paths)
        h = int(rng.integers(0, n))
        k = int(rng.choice([5000, 40000, 150000]))
        src = np.concatenate([src, rng.integers(0, n, k)])
        dst = np.concatenate([dst, np.full(k, h)])
    keep = src != dst
    src, dst = src[keep], dst[keep]
    m = len(src)
    w = rng.integers(0, 64, m).astype(np.uint32)
    if seed % 4 == 1:
        w[rng.random(m) < 0.01] = 0xFFFFFFF0   # saturating sums
    return rng, n, src, dst, w


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_apps_and_programs(seed):
    rng, n, src, dst, w = fuzz_graph(seed)
    parts = int(rng.choice([1, 1, 2, 3, 5]))
    exchange = "auto" if parts == 1 else str(rng.choice(["fused", "collective"]))
    mode = str(rng.choice(["pull", "push", "auto"]))
    source = int(rng.integers(0, n))
    g = csr_csc(n, src, dst, w)
    G = make_graph(g, partitions=parts)
    # Hash-Min and SSSP: values and counters exactly
    for app, o in (("cc", oracle.hashmin_cc(n, src, dst)),
                   ("sssp", oracle.sssp(n, src, dst, w, source=source))):
        G.run(app, mode=mode, source=source, exchange=exchange)
        s = G.stats()
        np.testing.assert_array_equal(G.values(host=True), o["values"], err_msg=app)
        assert s["supersteps"] == o["supersteps"], app
        np.testing.assert_array_equal(s["changed"], o["changed"], err_msg=app)
        np.testing.assert_array_equal(s["messages"], o["messages"], err_msg=app)
    # PageRank (pull: push is order-nondeterministic but within the same bar)
    k = int(rng.choice([1, 3, 10]))
    o = oracle.pagerank(n, src, dst, k=k)
    pr_mode = "pull" if mode == "auto" else mode
    G.run("pagerank", mode=pr_mode, iterations=k, exchange=exchange)
    err = np.abs(G.values(host=True) - o["values"])
    assert err.max() <= PR_ABS
    assert (err / np.maximum(np.abs(o["values"]), 1e-300)).max() <= PR_REL
    # the paper's programs: Fig. 9 and Fig. 10 (with the ipr_settled hint)
    oc = oracle.hashmin_cc(n, src, dst)
    G.run_program(prog("hashmin_cc"), mode=mode, exchange=exchange)
    np.testing.assert_array_equal(G.values(host=True), oc["values"])
    np.testing.assert_array_equal(G.stats()["messages"], oc["messages"])
    os_ = oracle.sssp(n, src, dst, w, source=source)
    G.run_program(prog("sssp"), params=[source], mode=mode, exchange=exchange)
    np.testing.assert_array_equal(G.values(host=True), os_["values"])
    np.testing.assert_array_equal(G.stats()["changed"], os_["changed"])
    G.close()

"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bars (BASELINE.json north_star):
  - CC labels and SSSP distances: bit-exact; superstep count and per-superstep changed /
    messages counters equal to the oracle's.
  - PageRank: max |gpu - oracle| <= 1e-9 (the gate), plus the internal diagnostic
    max relative error <= 1e-11.
"""
import json
import os

import numpy as np
import pytest

import oracle
from tests import checkers
from tests.graphs import csr_csc, make_graph

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")
with open(GOLDEN) as f:
    WORKED = json.load(f)

MODES = ["pull", "push", "auto"]
PR_ABS = 1e-9
PR_REL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_08781_b200 as ipr
    ipr.device_check(0)


def run_gpu(app, n, src, dst, w=None, mode="auto", k=10, source=0, partitions=1,
            max_supersteps=1 << 30, host=False, allow_guard=False):
    g = csr_csc(n, src, dst, w)
    G = make_graph(g, partitions=partitions, host=host, weighted=w is not None)
    pr = app == "pagerank"
    st = G.run(app, max_supersteps=max_supersteps, mode=mode, iterations=k, source=source,
               allow_guard=allow_guard, mass=pr)
    vals = G.values(host=True)
    stats = G.stats()
    G.close()
    if pr and n > 0:   # the mass invariant on the GPU's own per-superstep sums
        nd = int(np.count_nonzero(np.bincount(np.asarray(src, np.int64), minlength=n)))
        checkers.assert_pagerank_mass(stats, n, nd)
    return st, vals, stats


def check_min(app, n, src, dst, w=None, source=0, mode="auto", partitions=1):
    o = oracle.run(oracle.APP_HASHMIN_CC if app == "cc" else oracle.APP_SSSP, n, src, dst, w,
                   source=source)
    st, v, s = run_gpu(app, n, src, dst, w, mode=mode, source=source, partitions=partitions)
    np.testing.assert_array_equal(v, o["values"])
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["changed"], o["changed"])
    np.testing.assert_array_equal(s["messages"], o["messages"])
    return s


def check_pr(n, src, dst, k=10, mode="pull", partitions=1):
    o = oracle.pagerank(n, src, dst, k=k)
    st, v, s = run_gpu("pagerank", n, src, dst, mode=mode, k=k, partitions=partitions)
    err = np.abs(v - o["values"])
    assert err.max() <= PR_ABS
    rel = err / np.maximum(np.abs(o["values"]), 1e-300)
    assert rel.max() <= PR_REL, rel.max()
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["changed"], o["changed"])
    np.testing.assert_array_equal(s["messages"], o["messages"])
    return v


# ------------------------------------------------------------------ worked examples

@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", WORKED["pagerank"], ids=lambda c: c["name"])
def test_pagerank_worked(case, mode):
    from fractions import Fraction
    e = np.array(case["edges"], np.int64).reshape(-1, 2)
    _, v, s = run_gpu("pagerank", case["n"], e[:, 0], e[:, 1], k=case["k"],
                      mode="push" if mode == "push" else "pull")
    want = np.array([float(Fraction(x)) for x in case["values"]])
    np.testing.assert_allclose(v, want, rtol=1e-14, atol=0)
    assert s["supersteps"] == case["supersteps"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", WORKED["cc"], ids=lambda c: c["name"])
def test_cc_worked(case, mode):
    e = np.array(case["edges"], np.int64).reshape(-1, 2)
    _, v, s = run_gpu("cc", case["n"], e[:, 0], e[:, 1], mode=mode)
    want = case["trajectory"][-1] if "trajectory" in case else case["values"]
    assert list(v) == want
    if "supersteps" in case:
        assert s["supersteps"] == case["supersteps"]
    if "changed" in case:
        assert list(s["changed"]) == case["changed"]
        assert list(s["messages"]) == case["messages"]
    if "trajectory" in case:
        for step, traj in enumerate(case["trajectory"][:-1]):
            st, vv, _ = run_gpu("cc", case["n"], e[:, 0], e[:, 1], mode=mode,
                                max_supersteps=step + 1, allow_guard=True)
            assert list(vv) == traj, step


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", WORKED["sssp"], ids=lambda c: c["name"])
def test_sssp_worked(case, mode):
    e = np.array(case["edges"], np.int64).reshape(-1, 3)
    _, v, s = run_gpu("sssp", case["n"], e[:, 0], e[:, 1], e[:, 2], mode=mode,
                      source=case["source"])
    final = case["trajectory"][-1] if "trajectory" in case else case["values"]
    assert list(v) == [oracle.INF if x == "INF" else int(x) for x in final]
    assert s["supersteps"] == case["supersteps"]
    if "changed" in case:
        assert list(s["changed"]) == case["changed"]
        assert list(s["messages"]) == case["messages"]


# ------------------------------------------------------------------ random graphs

@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("mode", MODES)
def test_random_cc(seed, mode):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 6 * n))
    src, dst, _ = checkers.random_graph(rng, n, m)
    check_min("cc", n, src, dst, mode=mode)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("mode", MODES)
def test_random_sssp(seed, mode):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 6 * n))
    src, dst, w = checkers.random_graph(rng, n, m, weighted=True)
    check_min("sssp", n, src, dst, w if seed % 3 else None, source=int(rng.integers(0, n)),
              mode=mode)


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("mode", ["pull", "push"])
def test_random_pagerank(seed, mode):
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(1, 5000))
    m = int(rng.integers(0, 8 * n))
    src, dst, _ = checkers.random_graph(rng, n, m)
    check_pr(n, src, dst, k=[0, 1, 3, 10][seed % 4], mode=mode)


# ------------------------------------------------------------------ edge cases

def test_hub_spanning_many_tiles():
    # in-star with 300k leaves: one row spans ~150 tiles (pull_fixup path); closed form too
    n = 300_001
    leaves = np.arange(1, n)
    hub = np.zeros(n - 1, np.int64)
    v = check_pr(n, leaves, hub, k=3)
    want = (0.15 / n) * (1 + 0.85 * (n - 1))
    assert v[0] == pytest.approx(want, rel=1e-12)
    check_min("cc", n, leaves, hub)
    check_min("sssp", n, hub, leaves, np.full(n - 1, 7, np.uint32))


def test_long_chain_many_supersteps():
    n = 3000
    src = np.arange(n - 1)
    for mode in MODES:
        s = check_min("sssp", n, src, src + 1, mode=mode)
        assert s["supersteps"] == n
    check_min("cc", n, src, src + 1)


def test_single_vertex_and_empty_graph():
    for app in ("cc", "sssp"):
        check_min(app, 1, np.zeros(0, np.int64), np.zeros(0, np.int64))
        check_min(app, 17, np.zeros(0, np.int64), np.zeros(0, np.int64))
    check_pr(1, np.zeros(0, np.int64), np.zeros(0, np.int64))
    check_pr(9, np.zeros(0, np.int64), np.zeros(0, np.int64))


def test_duplicates_and_saturation():
    src = np.array([0, 0, 0, 1, 1, 2])
    dst = np.array([1, 1, 1, 2, 2, 3])
    w = np.array([9, 3, 5, 0xFFFFFFF0, 2, 60], np.uint32)
    check_min("sssp", 4, src, dst, w)
    check_pr(4, src, dst, k=4)


def test_guard_partial_state():
    n = 50
    src = np.arange(n - 1)
    o = oracle.sssp(n, src, src + 1, None, source=0, max_supersteps=7)
    st, v, s = run_gpu("sssp", n, src, src + 1, max_supersteps=7, allow_guard=True)
    import paper_2010_08781_b200 as ipr
    assert st == ipr.ERR_MAX_SUPERSTEPS and o["status"] == oracle.GUARD
    np.testing.assert_array_equal(v, o["values"])
    assert s["supersteps"] == 7
    o = oracle.pagerank(n, src, src + 1, k=10, max_supersteps=4)
    st, v, s = run_gpu("pagerank", n, src, src + 1, k=10, max_supersteps=4, allow_guard=True)
    assert st == ipr.ERR_MAX_SUPERSTEPS
    assert np.abs(v - o["values"]).max() <= 1e-15


def test_combiner_mismatch_and_bad_args():
    import paper_2010_08781_b200 as ipr
    g = make_graph(csr_csc(3, [0, 1], [1, 2]), weighted=False)
    with pytest.raises(ipr.IpregelError) as e:
        g.run("pagerank", combiner=ipr.COMBINE_MIN)
    assert e.value.status == ipr.ERR_INVALID_ARGUMENT
    with pytest.raises(ipr.IpregelError):
        g.run("sssp", source=3)
    with pytest.raises(ipr.IpregelError):
        g.run("cc", max_supersteps=0)
    with pytest.raises(ipr.IpregelError) as e:
        g.values()
    assert e.value.status == ipr.ERR_STATE


def test_validate_rejects_bad_graph():
    import paper_2010_08781_b200 as ipr
    g = csr_csc(4, [0, 1, 2], [1, 2, 3])
    g["csc_idx"] = g["csc_idx"].copy()
    g["csc_idx"][1] = 9
    with pytest.raises(ipr.IpregelError) as e:
        make_graph(g, validate=True, weighted=False)
    assert e.value.status == ipr.ERR_INVALID_GRAPH
    g = csr_csc(4, [0, 1, 2], [1, 2, 3])
    g["csr_off"] = g["csr_off"].copy()
    g["csr_off"][2] = 0
    with pytest.raises(ipr.IpregelError) as e:
        make_graph(g, validate=True, weighted=False)
    assert e.value.status == ipr.ERR_INVALID_GRAPH


def test_host_memory_descriptor_matches_device():
    rng = np.random.default_rng(5)
    n = 2000
    src, dst, w = checkers.random_graph(rng, n, 9000, weighted=True)
    g = csr_csc(n, src, dst, w)
    a = make_graph(g)
    b = make_graph(g, host=True)
    for app in ("pagerank", "cc", "sssp"):
        a.run(app)
        b.run(app)
        np.testing.assert_array_equal(a.values(host=True), b.values(host=True))


def test_message_storage_is_theta_n():
    # single-slot mailboxes -- state bytes do not grow with E
    import paper_2010_08781_b200 as ipr  # noqa: F401
    n = 4096
    small = csr_csc(n, np.arange(n - 1), np.arange(1, n))
    rng = np.random.default_rng(9)
    s2, d2, _ = checkers.random_graph(rng, n, 400_000)
    big = csr_csc(n, s2, d2)
    out = []
    for g in (small, big):
        G = make_graph(g, weighted=False)
        for app in ("pagerank", "cc", "sssp"):
            for mode in ("pull", "push"):
                G.run(app, mode=mode)
        out.append(G.memory_footprint()[1])
    assert out[0] == out[1]
    assert out[0] < 200 * n + (1 << 20)


# ------------------------------------------------------------------ partitions (loopback)

@pytest.mark.parametrize("exchange", ["fused", "collective"])
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_loopback_partitions_bit_identical(parts, exchange):
    """G partitions on one GPU: the fused exchange (epilogue stores into every partition's
    replica) and the collective one (copies after the kernel) give results
    bit-identical to one partition."""
    rng = np.random.default_rng(77)
    import inputs
    src, dst, w = inputs.rmat_coo(13, 16, 11, weighted=True)
    n = 1 << 13
    g = csr_csc(n, src, dst, w)
    ref = {}
    G1 = make_graph(g)
    for app in ("pagerank", "cc", "sssp"):
        for mode in ("pull", "push", "auto"):
            if app == "pagerank" and mode == "auto":
                continue
            G1.run(app, mode=mode)
            ref[(app, mode)] = (G1.values(host=True), G1.stats())
    Gp = make_graph(g, partitions=parts)
    for (app, mode), (v1, s1) in ref.items():
        Gp.run(app, mode=mode, exchange=exchange)
        vp = Gp.values(host=True)
        sp = Gp.stats()
        assert sp["exchange"] == ("collective" if mode == "push" else exchange)
        if app == "pagerank" and mode == "push":
            assert np.abs(vp - v1).max() <= 1e-15  # atomicAdd order
        else:
            np.testing.assert_array_equal(vp, v1)  # bit-identical, PageRank pull included
        assert sp["supersteps"] == s1["supersteps"]
        np.testing.assert_array_equal(sp["changed"], s1["changed"])
        np.testing.assert_array_equal(sp["messages"], s1["messages"])
    o = oracle.sssp(n, src, dst, w, source=0)
    Gp.run("sssp", exchange=exchange)
    np.testing.assert_array_equal(Gp.values(host=True), o["values"])
    del rng


def test_fused_exchange_flags():
    import paper_2010_08781_b200 as ipr
    n = 50
    src = np.arange(n - 1)
    g = csr_csc(n, src, src + 1)
    G = make_graph(g, partitions=2, weighted=False)
    import ctypes
    p = ipr.run_params_default()
    p.flags = ipr.RUN_EXCHANGE_FUSED | ipr.RUN_EXCHANGE_COLLECTIVE
    st = ipr.load().ipregel_run(G.handle, ipr.APP_SSSP, ipr.COMBINE_MIN, 100, ctypes.byref(p))
    assert st == ipr.ERR_INVALID_ARGUMENT
    p.flags = 0x80
    st = ipr.load().ipregel_run(G.handle, ipr.APP_SSSP, ipr.COMBINE_MIN, 100, ctypes.byref(p))
    assert st == ipr.ERR_INVALID_ARGUMENT
    G.run("sssp")
    assert G.stats()["exchange"] == "fused"          # default with reachable replicas
    G1 = make_graph(g, partitions=1, weighted=False)
    G1.run("sssp")
    assert G1.stats()["exchange"] == "none"
    G9 = make_graph(g, partitions=9, weighted=False)  # more partitions than peer slots
    G9.run("sssp")
    assert G9.stats()["exchange"] == "collective"
    with pytest.raises(ipr.IpregelError) as e:
        G9.run("sssp", exchange="fused")
    assert e.value.status == ipr.ERR_UNSUPPORTED
    o = oracle.sssp(n, src, src + 1, None)
    G9.run("pagerank")
    G9.run("sssp", exchange="collective")
    np.testing.assert_array_equal(G9.values(host=True), o["values"])


def test_loopback_with_empty_partition():
    n = 100
    src = np.arange(n - 1)
    g = csr_csc(n, src, src + 1)
    G = make_graph(g, partitions=3, weighted=False, bounds=np.array([0, 0, 60, 100]))
    for app in ("pagerank", "cc", "sssp"):
        G.run(app)
    o = oracle.sssp(n, src, src + 1, None)
    np.testing.assert_array_equal(G.values(host=True), o["values"])


# ------------------------------------------------------------------ internal vertex layouts

def _permuted(n, src, dst, w, perm):
    """Graph arrays with internal id perm[v] for original vertex v; vertex_ids = inverse."""
    g = csr_csc(n, perm[src], perm[dst], w)
    inv = np.empty(n, np.int32)
    inv[perm] = np.arange(n, dtype=np.int32)
    g["vertex_ids"] = inv
    return g


@pytest.mark.parametrize("seed", range(4))
def test_relabelled_layout_matches_oracle(seed):
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(2, 4000))
    src, dst, w = checkers.random_graph(rng, n, 6 * n, weighted=True)
    perm = rng.permutation(n).astype(np.int64)
    g = _permuted(n, src, dst, w, perm)
    d = to_device(g)
    ids = torch.from_numpy(g["vertex_ids"]).cuda()
    source = int(rng.integers(0, n))
    for parts in (1, 3):
        if parts == 1:
            P = ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], d["csr_off"], d["csr_idx"],
                                   d["csc_w"], d["csr_w"], vertex_ids=ids,
                                   degree_ordered=bool(seed % 2))
            G = ipr.Graph(P, validate=True)
        else:
            b = ipr.edge_balanced_bounds(g["csc_off"], parts, g["csr_off"])
            G = ipr.Graph(ipr.split_partitions(n, d["e"], b, d["csc_off"], d["csc_idx"],
                                               d["csr_off"], d["csr_idx"], d["csc_w"], d["csr_w"],
                                               vertex_ids=ids, degree_ordered=bool(seed % 2)))
        for mode in ("pull", "push", "auto"):
            o = oracle.hashmin_cc(n, src, dst)
            G.run("cc", mode=mode)
            np.testing.assert_array_equal(G.values(host=True), o["values"])
            np.testing.assert_array_equal(G.stats()["messages"], o["messages"])
            o = oracle.sssp(n, src, dst, w, source=source)
            G.run("sssp", mode=mode, source=source)
            np.testing.assert_array_equal(G.values(host=True), o["values"])
            np.testing.assert_array_equal(G.stats()["changed"], o["changed"])
        o = oracle.pagerank(n, src, dst)
        G.run("pagerank", mode="pull")
        assert np.abs(G.values(host=True) - o["values"]).max() <= PR_ABS
        G.close()


def test_vertex_ids_must_be_a_permutation():
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    g = csr_csc(5, [0, 1, 2], [1, 2, 3])
    d = to_device(g)
    bad = torch.tensor([0, 1, 1, 3, 4], dtype=torch.int32, device="cuda")
    P = ipr.full_partition(5, 3, d["csc_off"], d["csc_idx"], d["csr_off"], d["csr_idx"],
                           vertex_ids=bad)
    with pytest.raises(ipr.IpregelError) as e:
        ipr.Graph(P, validate=True)
    assert e.value.status == ipr.ERR_INVALID_GRAPH


def test_gpu_fixture_degree_order_matches_cpu_coo():
    # the degree-ordered device layout is the same graph: results equal the oracle's on the COO
    import inputs
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    cfg = inputs.Config("t", "all", 13, 16, 21, True)
    src, dst, w = inputs.rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed, weighted=True)
    for order in (False, True):
        g = config_graph_device(cfg, degree_order=order)
        assert g["e"] == len(src)
        G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                         g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                         degree_ordered=order))
        G.run("cc")
        np.testing.assert_array_equal(G.values(host=True),
                                      oracle.hashmin_cc(cfg.n, src, dst)["values"])
        G.run("sssp")
        np.testing.assert_array_equal(G.values(host=True),
                                      oracle.sssp(cfg.n, src, dst, w)["values"])
        G.run("pagerank", mode="pull")
        assert np.abs(G.values(host=True) - oracle.pagerank(cfg.n, src, dst)["values"]).max() < 1e-12
        if order:
            deg = g["csr_off"].diff().cpu().numpy()
            assert np.all(np.diff(deg) <= 0)  # internal ids ascend by decreasing out-degree


# ------------------------------------------------------------------ NCCL path (world of 1)

@pytest.mark.parametrize("exchange", ["fused", "collective"])
def test_nccl_path_single_rank_matches_oracle(exchange):
    """A graph created with a communicator runs every exchange through NCCL (grouped in-place
    broadcasts, all-reduced counters, all-gathered frontier sizes); with a world of one rank this
    exercises the multi-GPU code path on the one GPU available."""
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    comm = ipr.Comm(0, 1, ipr.nccl_unique_id(), torch.cuda.current_device())
    rng = np.random.default_rng(8)
    n = 3000
    src, dst, w = checkers.random_graph(rng, n, 20000, weighted=True)
    d = to_device(csr_csc(n, src, dst, w))
    G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], d["csr_off"],
                                     d["csr_idx"], d["csc_w"], d["csr_w"]), comm=comm)
    for mode in ("pull", "push", "auto"):
        o = oracle.hashmin_cc(n, src, dst)
        G.run("cc", mode=mode, exchange=exchange)
        np.testing.assert_array_equal(G.values(host=True), o["values"])
        np.testing.assert_array_equal(G.stats()["messages"], o["messages"])
        assert G.stats()["exchange"] == ("collective" if mode == "push" else exchange)
        o = oracle.sssp(n, src, dst, w, source=5)
        G.run("sssp", mode=mode, source=5, exchange=exchange)
        np.testing.assert_array_equal(G.values(host=True), o["values"])
        np.testing.assert_array_equal(G.stats()["changed"], o["changed"])
    for mode in ("pull", "push"):
        o = oracle.pagerank(n, src, dst)
        G.run("pagerank", mode=mode, exchange=exchange)
        assert np.abs(G.values(host=True) - o["values"]).max() <= PR_ABS
        np.testing.assert_array_equal(G.stats()["changed"], o["changed"])
    # a user program on the rank path (the ipr_settled minimum is all-reduced with NCCL)
    from paper_2010_08781_b200 import programs
    p = programs.compile("sssp")
    o = oracle.sssp(n, src, dst, w, source=5)
    for mode in ("pull", "auto"):
        G.run_program(p, params=[5], mode=mode, exchange=exchange)
        np.testing.assert_array_equal(G.values(host=True), o["values"])
        np.testing.assert_array_equal(G.stats()["changed"], o["changed"])
    G.close()
    comm.close()


# ------------------------------------------------------------------ PageRank to convergence

def _pr_tol_case(seed):
    rng = np.random.default_rng(6100 + seed)
    n = int(rng.integers(50, 3000))
    src, dst, _ = checkers.random_graph(rng, n, int(rng.integers(2 * n, 8 * n)))
    full = oracle.pagerank(n, src, dst, k=60)
    dl = full["delta"]
    # a tolerance geometrically between two well-separated deltas, so rounding order cannot
    # move the stopping superstep
    cand = [t for t in range(2, 60) if 0 < dl[t] < 0.5 * dl[t - 1] and dl[t] > 1e-13]
    t = cand[len(cand) // 2] if cand else 3
    return n, src, dst, float(np.sqrt(dl[t] * dl[t - 1]))


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("mode,parts", [("pull", 1), ("push", 1), ("pull", 3)])
def test_pagerank_to_convergence_matches_oracle(seed, mode, parts):
    n, src, dst, tol = _pr_tol_case(seed)
    o = oracle.pagerank(n, src, dst, k=60, tol=tol)
    assert o["supersteps"] < 61
    g = csr_csc(n, src, dst)
    G = make_graph(g, partitions=parts, weighted=False)
    G.run("pagerank", mode=mode, iterations=60, tolerance=tol)
    v = G.values(host=True)
    s = G.stats()
    assert s["supersteps"] == o["supersteps"]
    assert np.abs(v - o["values"]).max() <= PR_ABS
    rel = np.abs(v - o["values"]) / np.maximum(np.abs(o["values"]), 1e-300)
    assert rel.max() <= PR_REL
    np.testing.assert_allclose(s["pagerank_delta"], o["delta"], rtol=1e-9, atol=1e-16)
    np.testing.assert_array_equal(s["messages"], o["messages"])
    G.close()


def test_pagerank_to_convergence_closed_forms_and_k_cap():
    # in-star: delta_3 == 0 exactly -> 4 supersteps with tol = 0 (tests/test_oracle_pins.py)
    n = 1000
    leaves = np.arange(1, n)
    G = make_graph(csr_csc(n, leaves, np.zeros(n - 1, np.int64)), weighted=False)
    G.run("pagerank", mode="pull", iterations=10, tolerance=0.0)
    s = G.stats()
    assert s["supersteps"] == 4 and s["pagerank_delta"][3] == 0.0
    G.close()
    # an unreachable tolerance: Fig. 8's k wins and values equal the plain run
    rng = np.random.default_rng(12)
    src, dst, _ = checkers.random_graph(rng, 500, 3000)
    G = make_graph(csr_csc(500, src, dst), weighted=False)
    G.run("pagerank", mode="pull", iterations=10, tolerance=1e-300)
    a = G.values(host=True)
    assert G.stats()["supersteps"] == 11
    G.run("pagerank", mode="pull", iterations=10)
    np.testing.assert_array_equal(a, G.values(host=True))
    assert not G.stats()["pagerank_delta"].any()
    import paper_2010_08781_b200 as ipr
    with pytest.raises(ipr.IpregelError) as e:
        G.run("pagerank", tolerance=float("nan"))
    assert e.value.status == ipr.ERR_INVALID_ARGUMENT
    G.close()


def test_pagerank_to_convergence_cfg3_scale():
    """BASELINE configs[3]'s graph (R-MAT scale 22, ef 28, seed 4) to convergence at 1e-10."""
    import inputs
    from inputs.gpu import config_graph_device
    import paper_2010_08781_b200 as ipr
    cfg = inputs.CONFIGS["cfg3"]
    src, dst, _ = inputs.rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed)
    o = oracle.pagerank(cfg.n, src, dst, k=100, tol=1e-10)
    g = config_graph_device(cfg, degree_order=True)
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                     g["csr_idx"], None, None, g["vertex_ids"], degree_ordered=True))
    G.run("pagerank", mode="pull", iterations=100, tolerance=1e-10)
    s = G.stats()
    d = o["delta"]
    # the stopping decision is robust only if no delta sits within rounding of the tolerance
    assert np.all(np.abs(d[1:] - 1e-10) > 1e-14)
    assert s["supersteps"] == o["supersteps"]
    v = G.values(host=True)
    assert np.abs(v - o["values"]).max() <= PR_ABS
    # deltas are differences of f64 sums taken in another order: equal up to ~1e-16 absolute
    np.testing.assert_allclose(s["pagerank_delta"], d, rtol=1e-9, atol=1e-15)
    G.close()


# ------------------------------------------------------------------ Hash-Min row-list pull

@pytest.mark.parametrize("parts,mode", [(1, "pull"), (3, "pull"), (1, "auto"), (2, "auto")])
def test_cc_rowlist_pull_matches_oracle(parts, mode):
    """Once the rows not at label 0 hold < 5 % of the symmetrised edges, pull supersteps gather
    only over those rows (mode 3 in the stats); values and every counter stay the oracle's."""
    import inputs
    src, dst, _ = inputs.rmat_coo(14, 16, 33)
    n = 1 << 14
    o = oracle.hashmin_cc(n, src, dst)
    G = make_graph(csr_csc(n, src, dst), partitions=parts, weighted=False)
    G.run("cc", mode=mode, push_fraction=0.0 if mode == "pull" else 0.001)
    s = G.stats()
    np.testing.assert_array_equal(G.values(host=True), o["values"])
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["changed"], o["changed"])
    np.testing.assert_array_equal(s["messages"], o["messages"])
    assert 3 in list(s["mode"]), list(s["mode"])
    G.close()


# ------------------------------------------------------------------ CSR derived from the CSC

@pytest.mark.parametrize("host,windows", [(False, None), (True, None), (True, "7")])
def test_csr_derived_on_device_matches_given_csr(host, windows, monkeypatch):
    """windows: the host upload of the CSC weights in 7 windows, each permuted into the derived
    CSR's weights as it lands (create.cuh finish_uploads; cfg4 uses 8)."""
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    if windows:
        monkeypatch.setenv("IPREGEL_WEIGHT_WINDOWS", windows)
    rng = np.random.default_rng(31)
    n = 2500
    src, dst, w = checkers.random_graph(rng, n, 15000, weighted=True)
    g = csr_csc(n, src, dst, w)
    full = make_graph(g)
    if host:
        h = {k: np.ascontiguousarray(g[k]).view(np.int32) for k in ("csc_off", "csc_idx", "csc_w")}
        part = ipr.Partition(n, g["e"], 0, n, h["csc_off"], h["csc_idx"], None, None, h["csc_w"], None)
    else:
        d = to_device(g)
        part = ipr.Partition(n, g["e"], 0, n, d["csc_off"], d["csc_idx"], None, None, d["csc_w"], None)
    derived = ipr.Graph(part, validate=True)
    for app, mode in (("pagerank", "pull"), ("pagerank", "push"), ("cc", "pull"), ("cc", "push"),
                      ("cc", "auto"), ("sssp", "pull"), ("sssp", "push"), ("sssp", "auto")):
        full.run(app, mode=mode, source=3)
        derived.run(app, mode=mode, source=3)
        a, b = full.values(host=True), derived.values(host=True)
        if app == "pagerank" and mode == "push":
            assert np.abs(a - b).max() <= 1e-15
        else:
            np.testing.assert_array_equal(a, b)
        sa, sb = full.stats(), derived.stats()
        np.testing.assert_array_equal(sa["messages"], sb["messages"])
    o = oracle.sssp(n, src, dst, w, source=3)
    np.testing.assert_array_equal(derived.values(host=True), o["values"])
    full.close()
    derived.close()


def test_csr_derivation_needs_one_whole_partition():
    import ctypes
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    n = 100
    src = np.arange(n - 1)
    d = to_device(csr_csc(n, src, src + 1))
    b = np.array([0, 50, 100])
    parts = ipr.split_partitions(n, n - 1, b, d["csc_off"], d["csc_idx"], d["csr_off"], d["csr_idx"])
    for p in parts:
        p.csr_offsets = p.csr_indices = None
    descs = (ipr.ipregel.GraphDesc * 2)(*[p.desc() for p in parts])
    h = ctypes.c_void_p()
    st = ipr.load().ipregel_graph_create_partitioned(descs, 2, None, ctypes.byref(h))
    assert st == ipr.ERR_UNSUPPORTED


def test_pagerank_graph_replay_matches_first_run():
    """Fixed-k pull PageRank is captured as a CUDA graph on its first run and replayed: replays
    give the same values, counters and timing records; other k / max_supersteps re-capture."""
    import paper_2010_08781_b200 as ipr
    rng = np.random.default_rng(21)
    n = 4000
    src, dst, _ = checkers.random_graph(rng, n, 30000)
    G = make_graph(csr_csc(n, src, dst), partitions=2, weighted=False)
    launches = []
    vals = []
    for k in (10, 10, 10, 3, 10):
        before = ipr.kernel_launches()
        G.run("pagerank", mode="pull", iterations=k)
        launches.append(ipr.kernel_launches() - before)
        vals.append(G.values(host=True))
        s = G.stats()
        assert s["supersteps"] == k + 1 and (s["time_ms"] > 0).all()
    np.testing.assert_array_equal(vals[0], vals[1])
    np.testing.assert_array_equal(vals[0], vals[2])
    np.testing.assert_array_equal(vals[0], vals[4])
    # replays count the captured kernels; the first run also builds the hot/cold split
    assert launches[0] >= launches[1] == launches[2]
    o = oracle.pagerank(n, src, dst, k=3)
    assert np.abs(vals[3] - o["values"]).max() <= PR_ABS
    st = G.run("pagerank", mode="pull", iterations=10, max_supersteps=5, allow_guard=True)
    assert st == ipr.ERR_MAX_SUPERSTEPS and G.stats()["supersteps"] == 5
    G.close()


@pytest.mark.parametrize("exchange", ["fused", "collective"])
def test_pagerank_pull_bit_identical_random_bounds(exchange):
    """PageRank pull sums of many terms (rows of 0..400 in-edges, so chunks hold zero, one or
    many row ends) are bit-identical between one partition and four partitions at random
    bounds: every row's combine tree depends on its own edge positions on the global 128-edge
    grid only (E4), whatever rows the partition boundaries cut off a chunk."""
    rng = np.random.default_rng(3)
    n = 3000
    kind = rng.integers(0, 3, n)
    deg = np.where(kind == 0, rng.integers(0, 6, n),
                   np.where(kind == 1, rng.integers(6, 100, n), rng.integers(100, 400, n)))
    dst = np.repeat(np.arange(n), deg)
    src = rng.integers(0, n, len(dst))
    keep = src != dst
    g = csr_csc(n, src[keep], dst[keep])
    G1 = make_graph(g, weighted=False)
    G1.run("pagerank", mode="pull")
    v1 = G1.values(host=True)
    G1.close()
    for _ in range(12):
        b = np.sort(rng.choice(np.arange(1, n), 3, replace=False))
        bounds = np.concatenate([[0], b, [n]])
        Gp = make_graph(g, partitions=4, weighted=False, bounds=bounds)
        Gp.run("pagerank", mode="pull", exchange=exchange)
        np.testing.assert_array_equal(Gp.values(host=True), v1, err_msg=str(bounds.tolist()))
        Gp.close()


@pytest.mark.parametrize("exchange", ["fused", "collective"])
def test_pagerank_flagged_hub_rows_and_phantom_ends(exchange):
    """The flagged PageRank superstep (pr_flag.cuh) where its bookkeeping is stretched: hub rows
    of 300,000 and 140,000 in-edges (cut by more than 16 range boundaries: the warp-tree joins),
    a run of 2,000-edge rows (chunks inside rows, rows cut by one boundary), runs of rows without
    in-edges between rows of 1-3 in-edges (ordinals skip them; chunks with many ends), and
    partitions whose first edge is off the 8192-edge range grid (phantom end at local -1), or
    whose first rows have no in-edges -- equal to the oracle (Fig. 8), the mass invariant on the
    GPU's sums, and bit-identical across partitionings."""
    rng = np.random.default_rng(17)
    n = 6000
    deg = rng.integers(0, 4, n) * (rng.random(n) < 0.5)
    deg[10] = 300000
    deg[2500] = 140000
    deg[4000:4100] = 2000
    deg[5990:] = 0
    dst = np.repeat(np.arange(n), deg)
    src = rng.integers(0, n, len(dst))
    keep = src != dst
    src, dst = src[keep], dst[keep]
    o = oracle.pagerank(n, src, dst, k=10)
    g = csr_csc(n, src, dst)
    nd = int(np.count_nonzero(np.bincount(src, minlength=n)))
    G1 = make_graph(g, weighted=False)
    G1.run("pagerank", mode="pull", mass=True)
    v1 = G1.values(host=True)
    checkers.assert_pagerank_mass(G1.stats(), n, nd)
    G1.close()
    err = np.abs(v1 - o["values"])
    assert err.max() <= PR_ABS
    assert (err / np.abs(o["values"])).max() <= PR_REL
    empty = np.flatnonzero(deg == 0)
    cases = [[0, 11, n], [0, 2500, 2501, n], [0, 4050, n], [0, int(empty[3]), n],
             [0, 10, 11, 3000, n]]
    for _ in range(6):
        cases.append([0] + sorted(rng.choice(np.arange(1, n), 3, replace=False).tolist()) + [n])
    for bounds in cases:
        Gp = make_graph(g, partitions=len(bounds) - 1, weighted=False, bounds=np.array(bounds))
        Gp.run("pagerank", mode="pull", exchange=exchange)
        np.testing.assert_array_equal(Gp.values(host=True), v1, err_msg=str(bounds))
        Gp.close()


@pytest.mark.parametrize("n,m", [(1, 0), (5, 0), (7, 3), (300, 40000)])
def test_host_create_derived_csr_small_and_empty(n, m, monkeypatch):
    """The host-memory create pipeline (structure upload, derived CSR, weight windows permuted on
    a side stream, kernel-copy readbacks) on empty, tiny and duplicate-heavy graphs."""
    import paper_2010_08781_b200 as ipr
    monkeypatch.setenv("IPREGEL_WEIGHT_WINDOWS", "3")
    rng = np.random.default_rng(n + m)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    w = rng.integers(0, 50, len(src)).astype(np.uint32)
    g = csr_csc(n, src, dst, w)
    h = {k: np.ascontiguousarray(g[k]).view(np.int32) for k in ("csc_off", "csc_idx", "csc_w")}
    G = ipr.Graph(ipr.Partition(n, g["e"], 0, n, h["csc_off"], h["csc_idx"], None, None,
                                h["csc_w"], None), validate=True)
    for mode in ("pull", "push", "auto"):
        G.run("cc", mode=mode)
        np.testing.assert_array_equal(G.values(host=True), oracle.hashmin_cc(n, src, dst)["values"])
        G.run("sssp", mode=mode, source=0)
        np.testing.assert_array_equal(G.values(host=True),
                                      oracle.sssp(n, src, dst, w, source=0)["values"])
    G.run("pagerank", mode="pull")
    assert np.abs(G.values(host=True) - oracle.pagerank(n, src, dst)["values"]).max() <= PR_ABS
    G.close()


@pytest.mark.parametrize("ids,parts", [(False, 1), (True, 1), (False, 3)])
def test_get_values_async_matches_sync(ids, parts):
    """ipregel_get_values_async: each app's values staged privately and copied on the copy
    stream while the next app runs; after sync they equal the synchronous readback."""
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    rng = np.random.default_rng(41)
    n = 5000
    src, dst, w = checkers.random_graph(rng, n, 40000, weighted=True)
    perm = rng.permutation(n) if ids else np.arange(n)
    g = csr_csc(n, perm[src], perm[dst], w)
    d = to_device(g)
    vid = None
    if ids:
        inv = np.empty(n, np.int32)
        inv[perm] = np.arange(n, dtype=np.int32)
        vid = torch.from_numpy(inv).cuda()
    if parts == 1:
        G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], d["csr_off"],
                                         d["csr_idx"], d["csc_w"], d["csr_w"], vertex_ids=vid))
    else:
        G = make_graph(g, partitions=parts)
    want, got = {}, {}
    for app in ("pagerank", "cc", "sssp"):
        G.run(app)
        want[app] = G.values(host=True).copy()
        got[app] = torch.empty(n, dtype=torch.float64 if app == "pagerank" else torch.int32,
                               pin_memory=True)
        G.values_async(got[app])
    G.run("pagerank", iterations=3)   # a later run of an app already read must not matter
    G.sync()
    for app in want:
        np.testing.assert_array_equal(got[app].numpy().view(want[app].dtype), want[app])
    G.close()


# ------------------------------------------------------------------ library degree relabel

@pytest.mark.parametrize("memory", ["device", "host"])
@pytest.mark.parametrize("with_csr", [True, False])
@pytest.mark.parametrize("seed", range(3))
def test_layout_degree_matches_oracle(seed, memory, with_csr):
    """IPREGEL_LAYOUT_DEGREE: the library relabels an original-id graph by out-degree during
    create; every app's results (in original ids), counters and the SSSP source (an original id)
    equal the oracle's, and the internal CSC it built is degree-ordered with sorted rows."""
    import paper_2010_08781_b200 as ipr
    rng = np.random.default_rng(5100 + seed)
    n = int(rng.integers(2, 4000))
    src, dst, w = checkers.random_graph(rng, n, int(rng.integers(0, 8 * n)), weighted=True)
    g = csr_csc(n, src, dst, w)
    host = memory == "host"
    if host:
        arr = {k: (None if g[k] is None else np.ascontiguousarray(g[k]).view(np.int32))
               for k in ("csc_off", "csc_idx", "csc_w", "csr_off", "csr_idx", "csr_w")}
    else:
        from tests.graphs import to_device
        arr = to_device(g)
    p = ipr.full_partition(n, len(src), arr["csc_off"], arr["csc_idx"],
                           arr["csr_off"] if with_csr else None,
                           arr["csr_idx"] if with_csr else None, arr["csc_w"],
                           arr["csr_w"] if with_csr else None, layout=ipr.LAYOUT_DEGREE)
    G = ipr.Graph(p, validate=True)
    source = int(rng.integers(0, n))
    # the CSR is still being built on the library's aux stream when create returns: run a CSR
    # reader (Hash-Min, push) first on odd seeds
    apps = ("pagerank", "cc", "sssp") if seed % 2 == 0 else ("cc", "sssp", "pagerank")
    for app in apps:
        mode = "pull" if app == "pagerank" else ("push" if seed == 1 else "auto")
        G.run(app, mode=mode, source=source, mass=app == "pagerank")
        v = G.values(host=True)
        s = G.stats()
        if app == "pagerank":
            o = oracle.pagerank(n, src, dst, k=10)
            assert np.abs(v - o["values"]).max() <= PR_ABS
            assert (np.abs(v - o["values"]) / o["values"]).max() <= PR_REL
            nd = int(np.count_nonzero(np.bincount(np.asarray(src, np.int64), minlength=n)))
            checkers.assert_pagerank_mass(s, n, nd)
        else:
            o = oracle.run(oracle.APP_HASHMIN_CC if app == "cc" else oracle.APP_SSSP, n, src, dst,
                           w if app == "sssp" else None, source=source)
            np.testing.assert_array_equal(v, o["values"])
        assert s["supersteps"] == o["supersteps"]
        np.testing.assert_array_equal(s["changed"], o["changed"])
        np.testing.assert_array_equal(s["messages"], o["messages"])
    G.close()


def test_layout_degree_equals_fixture_layout_bitwise():
    """The library's relabel and the fixture's degree-ordered layout (inputs/gpu.py, the same
    order: decreasing out-degree, ties by id) give bit-identical PageRank values."""
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    g0 = config_graph_device("cfg0", weighted=False, degree_order=False)
    g1 = config_graph_device("cfg0", weighted=False, degree_order=True)
    Ga = ipr.Graph(ipr.full_partition(g0["n"], g0["e"], g0["csc_off"], g0["csc_idx"], None, None,
                                      layout=ipr.LAYOUT_DEGREE))
    Gb = ipr.Graph(ipr.full_partition(g1["n"], g1["e"], g1["csc_off"], g1["csc_idx"],
                                      g1["csr_off"], g1["csr_idx"], None, None, g1["vertex_ids"],
                                      degree_ordered=True))
    Ga.run("pagerank", mode="pull")
    Gb.run("pagerank", mode="pull")
    np.testing.assert_array_equal(Ga.values(host=True), Gb.values(host=True))
    Ga.close()
    Gb.close()


def test_layout_degree_rejects_bad_combinations():
    import ctypes

    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    n = 10
    src = np.array([0, 1, 2], np.int64)
    dst = np.array([1, 2, 3], np.int64)
    d = to_device(csr_csc(n, src, dst, None))
    ids = __import__("torch").arange(n, dtype=__import__("torch").int32, device="cuda")
    for kw in ({"vertex_ids": ids}, {"degree_ordered": True}):
        p = ipr.full_partition(n, 3, d["csc_off"], d["csc_idx"], None, None,
                               layout=ipr.LAYOUT_DEGREE, **kw)
        h = ctypes.c_void_p()
        st = ipr.load().ipregel_graph_create(ctypes.byref(p.desc()), None, None, ctypes.byref(h))
        assert st == ipr.ERR_INVALID_ARGUMENT
    bad = ipr.full_partition(n, 3, d["csc_off"], d["csc_idx"], None, None)
    desc = bad.desc()
    desc.layout = 7
    h = ctypes.c_void_p()
    assert ipr.load().ipregel_graph_create(ctypes.byref(desc), None, None,
                                           ctypes.byref(h)) == ipr.ERR_INVALID_ARGUMENT

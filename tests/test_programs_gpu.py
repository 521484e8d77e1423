"""GPU parity of user vertex programs (NVRTC-compiled, csrc/program.cuh) through the C ABI.

The paper's three programs written against the program API (paper_2010_08781_b200/programs.py,
Figs. 8-10) must equal the oracle exactly as the built-in apps do (CC / SSSP bit-exact with
every per-superstep counter; PageRank <= 1e-9 abs, <= 1e-11 rel), in pull, push and AUTO, on
one partition and on loopback partitions with either exchange.  Programs beyond the paper are
pinned to brute force (tests/checkers.py).
"""
import numpy as np
import pytest

import oracle
from tests import checkers
from tests.graphs import csr_csc, make_graph

pytestmark = pytest.mark.gpu

PR_ABS = 1e-9
PR_REL = 1e-11
_cache = {}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_08781_b200 as ipr
    ipr.device_check(0)


def prog(name):
    from paper_2010_08781_b200 import programs
    if name not in _cache:
        _cache[name] = programs.compile(name)
    return _cache[name]


def graph(seed, n=None, m_per=6, weighted=True):
    rng = np.random.default_rng(seed)
    n = n or int(rng.integers(50, 3000))
    src, dst, w = checkers.random_graph(rng, n, m_per * n, weighted=weighted)
    return n, src, dst, w


CONFIGS = [("pull", 1, "auto"), ("push", 1, "auto"), ("auto", 1, "auto"),
           ("auto", 3, "fused"), ("auto", 3, "collective"), ("push", 2, "fused")]


@pytest.mark.parametrize("mode,parts,exchange", CONFIGS)
@pytest.mark.parametrize("seed", range(2))
def test_paper_programs_equal_the_oracle(seed, mode, parts, exchange):
    n, src, dst, w = graph(700 + seed)
    G = make_graph(csr_csc(n, src, dst, w), partitions=parts)
    # Fig. 9 Hash-Min
    o = oracle.hashmin_cc(n, src, dst)
    G.run_program(prog("hashmin_cc"), mode=mode, exchange=exchange)
    s = G.stats()
    np.testing.assert_array_equal(G.values(host=True), o["values"])
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["changed"], o["changed"])
    np.testing.assert_array_equal(s["messages"], o["messages"])
    # Fig. 10 SSSP (weighted)
    source = int(np.random.default_rng(seed).integers(0, n))
    o = oracle.sssp(n, src, dst, w, source=source)
    G.run_program(prog("sssp"), params=[source], mode=mode, exchange=exchange)
    s = G.stats()
    np.testing.assert_array_equal(G.values(host=True), o["values"])
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["changed"], o["changed"])
    np.testing.assert_array_equal(s["messages"], o["messages"])
    # Fig. 8 PageRank, k = 10 (and k = 3)
    for k in (10, 3):
        o = oracle.pagerank(n, src, dst, k=k)
        G.run_program(prog("pagerank"), params=[k], mode=mode, exchange=exchange)
        v = G.values(host=True)
        s = G.stats()
        err = np.abs(v - o["values"])
        assert err.max() <= PR_ABS
        assert (err / np.maximum(np.abs(o["values"]), 1e-300)).max() <= PR_REL
        assert s["supersteps"] == o["supersteps"]
        np.testing.assert_array_equal(s["changed"], o["changed"])
        np.testing.assert_array_equal(s["messages"], o["messages"])
    G.close()


def test_program_pagerank_pull_equals_builtin():
    # the same IEEE operations per term; the built-in sums each row with the flagged superstep's
    # combine tree (pr_flag.cuh), the program with the range kernels' (pull.cuh): the two differ
    # only by summation order, a few ulps after k = 10 supersteps
    n, src, dst, _ = graph(11, n=5000)
    G = make_graph(csr_csc(n, src, dst), weighted=False)
    G.run("pagerank", mode="pull")
    a = G.values(host=True)
    G.run_program(prog("pagerank"), params=[10], mode="pull")
    np.testing.assert_allclose(G.values(host=True), a, rtol=1e-13, atol=0)
    G.close()


@pytest.mark.parametrize("mode", ["pull", "push", "auto"])
def test_new_programs_against_brute_force(mode):
    n, src, dst, w = graph(42, n=1500)
    G = make_graph(csr_csc(n, src, dst, w))
    e3 = list(zip(src.tolist(), dst.tolist(), w.tolist()))
    e2 = list(zip(src.tolist(), dst.tolist()))
    source = 3
    G.run_program(prog("bfs"), params=[source], mode=mode)
    np.testing.assert_array_equal(G.values(host=True), checkers.bfs_levels(n, e2, source))
    G.run_program(prog("widest_path"), params=[source], mode=mode)
    np.testing.assert_array_equal(G.values(host=True), checkers.widest_path(n, e3, source))
    G.run_program(prog("max_label"), mode=mode)
    np.testing.assert_array_equal(G.values(host=True), checkers.cc_max_label(n, e2))
    G.run_program(prog("in_degree"), mode=mode)
    np.testing.assert_array_equal(G.values(host=True), np.bincount(dst, minlength=n))
    assert G.stats()["supersteps"] == 2
    G.run_program(prog("sssp_f64"), params=[source], mode=mode)
    d = np.array(checkers.dijkstra(n, e3, source), dtype=np.float64)
    d[d == checkers.INF] = np.inf
    np.testing.assert_array_equal(G.values(host=True), d)
    G.close()


def test_program_on_relabelled_layout_sees_original_ids():
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    rng = np.random.default_rng(5)
    n = 2000
    src, dst, w = checkers.random_graph(rng, n, 8000, weighted=True)
    perm = rng.permutation(n).astype(np.int64)
    g = csr_csc(n, perm[src], perm[dst], w)
    inv = np.empty(n, np.int32)
    inv[perm] = np.arange(n, dtype=np.int32)
    d = to_device(g)
    ids = torch.from_numpy(inv).cuda()
    G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], d["csr_off"],
                                     d["csr_idx"], d["csc_w"], d["csr_w"], vertex_ids=ids))
    G.run_program(prog("hashmin_cc"))
    np.testing.assert_array_equal(G.values(host=True), oracle.hashmin_cc(n, src, dst)["values"])
    G.run_program(prog("sssp"), params=[7])
    np.testing.assert_array_equal(G.values(host=True), oracle.sssp(n, src, dst, w, source=7)["values"])
    G.close()


def test_program_guard_and_bad_params():
    import ctypes
    import paper_2010_08781_b200 as ipr
    n = 40
    src = np.arange(n - 1)
    G = make_graph(csr_csc(n, src, src + 1), weighted=False)
    st = G.run_program(prog("bfs"), params=[0], max_supersteps=5, allow_guard=True)
    assert st == ipr.ERR_MAX_SUPERSTEPS
    v = G.values(host=True)
    assert list(v[:5]) == [0, 1, 2, 3, 4] and v[5] == 0xFFFFFFFF   # state after superstep 4
    vals = (ctypes.c_double * 9)()
    st = ipr.load().ipregel_run_program(G.handle, prog("bfs").handle, 100, None, vals, 9)
    assert st == ipr.ERR_INVALID_ARGUMENT
    G.close()


def test_program_cc_at_baseline_config1():
    """BASELINE configs[1] (R-MAT scale 20, ef 16, seed 2, symmetrised) with the Fig. 9 program,
    degree-ordered layout, AUTO: bit-exact with every counter."""
    import inputs
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    cfg = inputs.CONFIGS["cfg1"]
    src, dst, _ = inputs.rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed)
    o = oracle.hashmin_cc(cfg.n, src, dst)
    g = config_graph_device(cfg, degree_order=True)
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                     g["csr_idx"], None, None, g["vertex_ids"], degree_ordered=True))
    G.run_program(prog("hashmin_cc"))
    s = G.stats()
    np.testing.assert_array_equal(G.values(host=True), o["values"])
    assert s["supersteps"] == o["supersteps"]
    np.testing.assert_array_equal(s["messages"], o["messages"])
    G.close()


# ------------------------------------------------------------------ Fig. 2 services

@pytest.mark.parametrize("mode,parts", [("pull", 1), ("push", 1), ("auto", 3), ("push", 4)])
def test_point_to_point_send(mode, parts):
    """IP_send_message: every vertex v > 0 sends v to (v - 1) / 2; values = sum of children."""
    n, src, dst, _ = graph(9, n=3000)
    G = make_graph(csr_csc(n, src, dst), partitions=parts, weighted=False)
    G.run_program(prog("heap_children_sum"), mode=mode)
    v = G.values(host=True).astype(np.int64)
    ids = np.arange(n)
    want = np.where(2 * ids + 1 < n, 2 * ids + 1, 0) + np.where(2 * ids + 2 < n, 2 * ids + 2, 0)
    np.testing.assert_array_equal(v, want)
    s = G.stats()
    assert s["supersteps"] == 2 and s["messages"][0] == n - 1
    G.close()


def test_point_to_point_send_original_ids_under_relabelling():
    import torch
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    rng = np.random.default_rng(3)
    n = 1000
    src, dst, _ = checkers.random_graph(rng, n, 4000)
    perm = rng.permutation(n).astype(np.int64)
    g = csr_csc(n, perm[src], perm[dst])
    inv = np.empty(n, np.int32)
    inv[perm] = np.arange(n, dtype=np.int32)
    d = to_device(g)
    G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], d["csr_off"],
                                     d["csr_idx"], vertex_ids=torch.from_numpy(inv).cuda()))
    G.run_program(prog("heap_children_sum"), mode="push")
    ids = np.arange(n)
    want = np.where(2 * ids + 1 < n, 2 * ids + 1, 0) + np.where(2 * ids + 2 < n, 2 * ids + 2, 0)
    np.testing.assert_array_equal(G.values(host=True).astype(np.int64), want)
    G.close()


@pytest.mark.parametrize("parts", [1, 3])
def test_aggregator_counts_vertices(parts):
    n, src, dst, _ = graph(5, n=2222)
    G = make_graph(csr_csc(n, src, dst), partitions=parts, weighted=False)
    G.run_program(prog("count_vertices"))
    np.testing.assert_array_equal(G.values(host=True), np.full(n, float(n)))
    G.close()


@pytest.mark.parametrize("mode,parts", [("pull", 1), ("push", 1), ("pull", 3)])
def test_pagerank_converge_program_equals_oracle(mode, parts):
    """PageRank to convergence written with a MAX aggregator halts one superstep after the
    oracle's master halt, with the same values (reading R27)."""
    rng = np.random.default_rng(6200)
    n = 2000
    src, dst, _ = checkers.random_graph(rng, n, 12000)
    full = oracle.pagerank(n, src, dst, k=60)
    dl = full["delta"]
    cand = [t for t in range(2, 60) if 0 < dl[t] < 0.5 * dl[t - 1] and dl[t] > 1e-13]
    t = cand[len(cand) // 2]
    tol = float(np.sqrt(dl[t] * dl[t - 1]))
    o = oracle.pagerank(n, src, dst, k=60, tol=tol)
    G = make_graph(csr_csc(n, src, dst), partitions=parts, weighted=False)
    G.run_program(prog("pagerank_converge"), params=[60, tol], mode=mode)
    v = G.values(host=True)
    assert np.abs(v - o["values"]).max() <= PR_ABS
    assert G.stats()["supersteps"] == o["supersteps"] + 1
    G.close()


# ------------------------------------------------------------------ other value types

@pytest.mark.parametrize("mode,parts", [("pull", 1), ("push", 1), ("auto", 3)])
def test_typed_programs(mode, parts):
    """f32 / i32 / u64 / i64 values: the same programs, pinned to brute force."""
    n, src, dst, w = graph(77, n=1800)
    G = make_graph(csr_csc(n, src, dst, w), partitions=parts)
    e3 = list(zip(src.tolist(), dst.tolist(), w.tolist()))
    e2 = list(zip(src.tolist(), dst.tolist()))
    d = np.array(checkers.dijkstra(n, e3, 4), dtype=np.int64)
    G.run_program(prog("sssp_i32"), params=[4], mode=mode)
    want = np.where(d == checkers.INF, 0x7FFFFFFF, d).astype(np.int32)
    np.testing.assert_array_equal(G.values(host=True), want)
    G.run_program(prog("sssp_f32"), params=[4], mode=mode)
    want = np.where(d == checkers.INF, np.inf, d).astype(np.float32)   # integer sums < 2^24
    np.testing.assert_array_equal(G.values(host=True), want)
    lab = np.array(checkers.cc_union_find(n, e2), dtype=np.uint64)
    G.run_program(prog("hashmin_u64"), mode=mode)
    np.testing.assert_array_equal(G.values(host=True), lab)
    G.run_program(prog("min_neg_label_i64"), mode=mode)
    np.testing.assert_array_equal(G.values(host=True), -np.array(checkers.cc_max_label(n, e2), np.int64))
    G.close()


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("n", [1, 17])
@pytest.mark.parametrize("parts", [1, 3])
def test_programs_on_edgeless_graphs(n, parts):
    if parts > n:
        pytest.skip("more partitions than vertices")
    e = np.zeros(0, np.int64)
    G = make_graph(csr_csc(n, e, e), partitions=parts, weighted=False)
    for mode in ("pull", "push", "auto"):
        G.run_program(prog("hashmin_cc"), mode=mode)
        np.testing.assert_array_equal(G.values(host=True), oracle.hashmin_cc(n, e, e)["values"])
        G.run_program(prog("pagerank"), params=[10], mode=mode)
        o = oracle.pagerank(n, e, e, k=10)
        assert np.abs(G.values(host=True) - o["values"]).max() <= PR_ABS
        assert G.stats()["supersteps"] == o["supersteps"]
        G.run_program(prog("heap_children_sum"), mode=mode)
        ids = np.arange(n)
        want = np.where(2 * ids + 1 < n, 2 * ids + 1, 0) + np.where(2 * ids + 2 < n, 2 * ids + 2, 0)
        np.testing.assert_array_equal(G.values(host=True).astype(np.int64), want)
    G.close()


def test_program_guard_with_sends_and_aggregate_counts():
    # sends count as messages for termination: a chain of point-to-point hand-offs
    import paper_2010_08781_b200 as ipr
    src = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned*) {
    *value = 0;
    if (c.id == 0) ipr_send(c, 1, 1u);
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx& c, unsigned* value, unsigned mailbox, unsigned*) {
    if (mailbox) {                       // got the token: keep it, pass it on
        *value = mailbox;
        ipr_send(c, c.id + 1, mailbox + 1);
        ipr_aggregate(c, 1.0);
    }
    return 0;
}
__device__ unsigned ipr_edge(unsigned m, unsigned) { return m; }
"""
    p = ipr.Program(src, "u32", "sum", aggregator="sum")
    n = 50
    e = np.zeros(0, np.int64)
    for parts in (1, 4):
        G = make_graph(csr_csc(n, e, e), partitions=parts, weighted=False)
        G.run_program(p, mode="push")
        v = G.values(host=True)
        np.testing.assert_array_equal(v, np.concatenate([[0], np.arange(1, n)]))
        s = G.stats()
        assert s["supersteps"] == n            # the token visits every vertex, then stops
        assert list(s["messages"][:-1]) == [1] * (n - 1)
        st = G.run_program(p, mode="pull", max_supersteps=10, allow_guard=True)
        assert st == ipr.ERR_MAX_SUPERSTEPS
        G.close()


PULSE = r"""
// s=0,1: everyone broadcasts 1 (pull supersteps).  s=2: vertex 0 broadcasts, even ids stay
// active, odd ids halt -> few messages, so AUTO pushes at s=3, where the even ids broadcast id+1
// and the odd ids (halted, mostly without messages) must leave NO stale value in the outbox
// buffer they last wrote at s=1: s=4 pulls it, summing only the even senders.
__device__ unsigned ipr_init(const ipr_ctx&, unsigned* value, unsigned* message) {
    *value = 0;
    *message = 1;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx& c, unsigned* value, unsigned mailbox, unsigned* message) {
    if (c.superstep == 1) { *message = 1; return IPR_BROADCAST; }
    if (c.superstep == 2) {
        if (c.id == 0) { *message = 7; return IPR_BROADCAST | IPR_STAY_ACTIVE; }
        return (c.id % 2 == 0) ? IPR_STAY_ACTIVE : 0;
    }
    if (c.superstep == 3) {
        if (c.id % 2 == 0) { *message = (unsigned)c.id + 1; return IPR_BROADCAST; }
        return 0;
    }
    *value = mailbox;
    return 0;
}
__device__ unsigned ipr_edge(unsigned m, unsigned) { return m; }
"""


@pytest.mark.parametrize("parts,exchange", [(1, "auto"), (3, "fused"), (3, "collective")])
def test_push_superstep_clears_stale_outbox(parts, exchange):
    """Push supersteps skip idle rows (program.cuh k_prog_apply, flag bit 2 = broadcast two
    supersteps ago): a halted row without messages must still clear the outbox slot it wrote two
    supersteps earlier, or the next pull superstep would gather its stale message."""
    import paper_2010_08781_b200 as ipr
    p = ipr.Program(PULSE, "u32", "sum")
    rng = np.random.default_rng(17)
    n = 3000
    src, dst, _ = checkers.random_graph(rng, n, 30000, weighted=False)
    src = np.concatenate([src, np.zeros(3, np.int64)])
    dst = np.concatenate([dst, np.array([5, 6, 9])])
    G = make_graph(csr_csc(n, src, dst), partitions=parts, weighted=False)
    G.run_program(p, mode="auto", push_fraction=0.05, exchange=exchange)
    s = G.stats()
    modes = "".join("ilpr"[m] for m in s["mode"])
    assert modes[3] == "p" and modes[4] == "l", modes   # push at s=3, pull at s=4
    even = (src % 2) == 0
    want = np.bincount(dst[even], weights=(src[even] + 1), minlength=n).astype(np.uint32)
    np.testing.assert_array_equal(G.values(host=True), want)
    G.close()


@pytest.mark.parametrize("mode", ["pull", "push", "auto"])
def test_programs_on_library_relabel(mode):
    """User programs on a graph the library relabelled itself (IPREGEL_LAYOUT_DEGREE): the CSR is
    still being built on the library's aux stream when the first program runs; ids seen by the
    programs (ipr_ctx.id, ipr_send targets, the SSSP source parameter) are original ids."""
    import paper_2010_08781_b200 as ipr
    from tests.graphs import to_device
    n, src, dst, w = graph(913)
    d = to_device(csr_csc(n, src, dst, w))
    G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], None, None,
                                     d["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
    G.run_program(prog("hashmin_cc"), mode=mode)
    np.testing.assert_array_equal(G.values(host=True), oracle.hashmin_cc(n, src, dst)["values"])
    G.run_program(prog("sssp"), params=[11], mode=mode)
    np.testing.assert_array_equal(G.values(host=True),
                                  oracle.sssp(n, src, dst, w, source=11)["values"])
    G.run_program(prog("pagerank"), params=[10], mode="pull" if mode == "auto" else mode)
    o = oracle.pagerank(n, src, dst, k=10)
    assert np.abs(G.values(host=True) - o["values"]).max() <= PR_ABS
    G.close()
    G = ipr.Graph(ipr.full_partition(n, d["e"], d["csc_off"], d["csc_idx"], None, None,
                                     layout=ipr.LAYOUT_DEGREE))
    G.run_program(prog("heap_children_sum"), mode="push")
    ids = np.arange(n)
    want = np.where(2 * ids + 1 < n, 2 * ids + 1, 0) + np.where(2 * ids + 2 < n, 2 * ids + 2, 0)
    np.testing.assert_array_equal(G.values(host=True).astype(np.int64), want)
    G.close()

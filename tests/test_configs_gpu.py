"""Parity at BASELINE.json's sizes (configs[0..4]) through the C ABI, in the launch
configuration bench.py times (the library's degree relabel of the original-id CSC, PageRank pull,
CC/SSSP AUTO), in the fixture's degree-ordered layout and in the original layout.

configs[0..3]: against the oracle run live on the box's CPU (seconds to ~20 s each).
configs[4] (1.88e9 edges): against tests/golden/cfg4_oracle.json, written by
tests/golden/make_cfg4_golden.py from the oracle alone -- CC labels and SSSP distances by a
sha256 of the whole array (bit-exact), PageRank at 65,565 sampled vertices (the 1e-9 gate and the
1e-11 relative diagnostic) plus the whole-vector sum, and every per-superstep counter.
"""
import json
import os

import numpy as np
import pytest

import inputs
import oracle
from tests import checkers

pytestmark = pytest.mark.gpu
GOLDEN4 = os.path.join(os.path.dirname(__file__), "golden", "cfg4_oracle.json")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def device_graph(cfg, order):
    """order: True -- the fixture's degree-ordered layout with vertex_ids; False -- original ids;
    "library" -- original-id CSC only, relabelled by the library (IPREGEL_LAYOUT_DEGREE, the CSR
    derived on the device): bench.py's graph."""
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    if order == "library":
        g = config_graph_device(cfg, weighted=True, degree_order=False)
        G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                         g["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
        return g, G
    g = config_graph_device(cfg, weighted=True, degree_order=order)
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                     g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                     degree_ordered=order))
    return g, G


def check_counters(stats, want):
    assert stats["supersteps"] == want["supersteps"]
    np.testing.assert_array_equal(stats["changed"], np.asarray(want["changed"], np.uint64))
    np.testing.assert_array_equal(stats["messages"], np.asarray(want["messages"], np.uint64))


@pytest.mark.parametrize("order", [True, False, "library"])
@pytest.mark.parametrize("name", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_config_vs_live_oracle(name, order):
    cfg = inputs.CONFIGS[name]
    src, dst, w = inputs.rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed, weighted=True)
    g, G = device_graph(cfg, order)
    assert g["e"] == len(src)
    if cfg.app == "pagerank":
        o = oracle.pagerank(cfg.n, src, dst, k=cfg.iterations)
        nd = int(((g["csr_off"][1:] - g["csr_off"][:-1]) > 0).sum().item())
        for mode in ("pull", "push"):
            G.run("pagerank", mode=mode, iterations=cfg.iterations, mass=True)
            v = G.values(host=True)
            err = np.abs(v - o["values"])
            assert err.max() <= 1e-9
            assert (err / o["values"]).max() <= 1e-11
            check_counters(G.stats(), o)
            checkers.assert_pagerank_mass(G.stats(), cfg.n, nd)
    elif cfg.app == "cc":
        o = oracle.hashmin_cc(cfg.n, src, dst)
        for mode in ("auto", "pull", "push"):
            G.run("cc", mode=mode)
            np.testing.assert_array_equal(G.values(host=True), o["values"])
            check_counters(G.stats(), o)
    else:
        o = oracle.sssp(cfg.n, src, dst, w, source=0)
        for mode in ("auto", "pull", "push"):
            G.run("sssp", mode=mode)
            np.testing.assert_array_equal(G.values(host=True), o["values"])
            check_counters(G.stats(), o)
    G.close()


@pytest.mark.parametrize("order", [True, False, "library"])
def test_cfg4_vs_golden(order):
    if not os.path.exists(GOLDEN4):
        pytest.skip("golden file missing")
    with open(GOLDEN4) as f:
        gold = json.load(f)
    cfg = inputs.CONFIGS["cfg4"]
    g, G = device_graph(cfg, order)
    assert g["e"] == gold["edges"]
    ids = np.asarray(gold["sample_ids"], np.int64)
    # PageRank, pull (the bench's mode)
    G.run("pagerank", mode="pull", iterations=cfg.iterations)
    v = G.values(host=True)
    want = np.asarray(gold["apps"]["pagerank"]["sample_values"])
    err = np.abs(v[ids] - want)
    assert err.max() <= 1e-9
    assert (err / want).max() <= 1e-11
    assert abs(float(v.sum()) - gold["apps"]["pagerank"]["sum"]) <= 1e-9
    check_counters(G.stats(), gold["apps"]["pagerank"])
    # CC and SSSP, AUTO (pull for dense supersteps, push for the sparse tail)
    for app in ("cc", "sssp"):
        G.run(app)
        vals = G.values(host=True)
        assert inputs.array_digest(vals) == gold["apps"][app]["values_sha256"], app
        np.testing.assert_array_equal(vals[ids], np.asarray(gold["apps"][app]["sample_values"],
                                                            np.uint32))
        check_counters(G.stats(), gold["apps"][app])
    G.close()


def test_library_relabel_from_host_matches_device():
    """bench.py's e2e create: the library relabel from pinned HOST memory without validation,
    where the out-degree histogram runs window by window during the index upload (E >= 2^24),
    builds the same graph as the relabel from device memory -- every app's values and counters
    bit-identical (configs[2], 6.7e7 edges)."""
    import torch

    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    cfg = inputs.CONFIGS["cfg2"]
    g = config_graph_device(cfg, weighted=True, degree_order=False)
    assert g["e"] >= 1 << 24
    host = {}
    for k in ("csc_off", "csc_idx", "csc_w"):
        h = torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True)
        h.copy_(g[k])
        host[k] = h.numpy()
    Gd = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                      g["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
    Gh = ipr.Graph(ipr.full_partition(g["n"], g["e"], host["csc_off"], host["csc_idx"], None, None,
                                      host["csc_w"], None, layout=ipr.LAYOUT_DEGREE),
                   validate=False)
    for app in ("pagerank", "cc", "sssp"):
        mode = "pull" if app == "pagerank" else "auto"
        Gd.run(app, mode=mode)
        Gh.run(app, mode=mode)
        np.testing.assert_array_equal(Gh.values(host=True), Gd.values(host=True))
        sd, sh = Gd.stats(), Gh.stats()
        np.testing.assert_array_equal(sh["changed"], sd["changed"])
        np.testing.assert_array_equal(sh["messages"], sd["messages"])
    Gd.close()
    Gh.close()


@pytest.mark.parametrize("parts", [2, 5])
def test_cfg3_pagerank_partitions_bit_identical(parts):
    """configs[3] (1.17e8 edges, degree-ordered layout) split into 2 / 5 edge-balanced destination
    partitions (loopback; both exchanges): every PageRank value bit-identical to the one-partition
    run -- the flagged superstep's ranges sit on the global 8192-edge grid and every partition
    whose first edge is off that grid starts with a phantom end (pr_flag.cuh)."""
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    cfg = inputs.CONFIGS["cfg3"]
    g = config_graph_device(cfg, weighted=False, degree_order=True)
    G1 = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                      g["csr_idx"], vertex_ids=g["vertex_ids"],
                                      degree_ordered=True))
    G1.run("pagerank", mode="pull", iterations=cfg.iterations)
    v1 = G1.values(host=True)
    G1.close()
    bounds = ipr.edge_balanced_bounds(g["csc_off"].cpu().numpy(), parts,
                                      g["csr_off"].cpu().numpy())
    for exchange in ("fused", "collective"):
        ps = ipr.split_partitions(g["n"], g["e"], bounds, g["csc_off"], g["csc_idx"], g["csr_off"],
                                  g["csr_idx"], vertex_ids=g["vertex_ids"], degree_ordered=True)
        Gp = ipr.Graph(ps)
        Gp.run("pagerank", mode="pull", iterations=cfg.iterations, exchange=exchange)
        np.testing.assert_array_equal(Gp.values(host=True), v1, err_msg=exchange)
        Gp.close()

"""The PageRank pull variants behind build-free knobs, each in a fresh process (the library reads
its knobs once, when it loads):

  IPREGEL_PR_FLAG=0  the round-1 range kernel (k_pull_ranges<PageRankSum>): equal to the oracle
                     (Fig. 8) within the parity bar;
  IPREGEL_PR_FUSE=1  the flagged superstep with Fig. 8's update in its epilogue: the same IEEE
                     operations as the separate update pass, so bit-identical to the default.

Graphs: rows of 0-400 in-edges (chunks with zero, one or many row ends), one and three
partitions.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, ROOT)
from tests.graphs import csr_csc, make_graph
rng = np.random.default_rng(5)
n = 4000
deg = np.where(rng.random(n) < 0.5, rng.integers(0, 6, n), rng.integers(6, 400, n))
dst = np.repeat(np.arange(n), deg)
src = rng.integers(0, n, len(dst))
keep = src != dst
g = csr_csc(n, src[keep], dst[keep])
out = {}
for parts in (1, 3):
    G = make_graph(g, partitions=parts, weighted=False)
    G.run("pagerank", mode="pull")
    out[parts] = G.values(host=True).tolist()
    G.close()
np.save(OUT, np.array([out[1], out[3]]))
"""


def run_child(tmp_path, tag, env_extra):
    out = str(tmp_path / f"{tag}.npy")
    code = CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def graph_edges():
    rng = np.random.default_rng(5)
    n = 4000
    deg = np.where(rng.random(n) < 0.5, rng.integers(0, 6, n), rng.integers(6, 400, n))
    dst = np.repeat(np.arange(n), deg)
    src = rng.integers(0, n, len(dst))
    keep = src != dst
    return n, src[keep], dst[keep]


@pytest.fixture(scope="module")
def default_values(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return run_child(tmp_path_factory.mktemp("knobs"), "default", {})


def test_round1_range_kernel_matches_oracle(default_values, tmp_path):
    v = run_child(tmp_path, "flag0", {"IPREGEL_PR_FLAG": "0"})
    n, src, dst = graph_edges()
    o = oracle.pagerank(n, src, dst, k=10)["values"]
    for row in (v[0], v[1], default_values[0]):
        err = np.abs(row - o)
        assert err.max() <= 1e-9
        assert (err / np.abs(o)).max() <= 1e-11
    # each kernel is bit-identical across partitionings
    np.testing.assert_array_equal(v[0], v[1])
    np.testing.assert_array_equal(default_values[0], default_values[1])


def test_fused_update_is_bit_identical(default_values, tmp_path):
    v = run_child(tmp_path, "fuse1", {"IPREGEL_PR_FUSE": "1"})
    np.testing.assert_array_equal(v, default_values)

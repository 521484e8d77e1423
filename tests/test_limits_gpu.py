"""The int32 limit of a partition (create.cuh: rows + edges <= INT32_MAX - 4 x 128, the range
kernels' merge coordinates plus the 3 chunks they look ahead), exercised at that limit.

A ragged circulant graph with N = 2^20 vertices and E = INT32_MAX - 512 - N edges (2.146e9):
row v lists the sources v+1, ..., v+d_v (mod N), d_v = 2047 or 2048.  One PageRank superstep
(Fig. 8 with k = 1) then has a closed form per vertex that the host evaluates
exactly from the structure -- r_1(v) = 0.15/N + 0.85 * sum_{k=1..d_v} (1/N) / outdeg(v+k) --
checked at every vertex to 1e-12 relative (2047 equal-sized terms summed in any order stay within
~2.5e-13), the rows whose merge coordinates sit just below INT32_MAX included.
One edge more is refused.  Needs ~60 GB of device memory (the graph, the derived CSR and the
transpose's temporaries).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 1 << 20
KCHUNK = 128
E_MAX = 2147483647 - 4 * KCHUNK - N   # rows + edges at the documented limit


@pytest.fixture(scope="module")
def circulant():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base, rem = divmod(E_MAX, N)
    deg = np.full(N, base, np.int64)
    deg[:rem] += 1                       # ragged: the first `rem` rows have one edge more
    off = np.zeros(N + 1, np.int64)
    off[1:] = np.cumsum(deg)
    assert off[-1] == E_MAX and off[-1] + N == 2147483647 - 4 * KCHUNK
    d_off = torch.from_numpy(off.astype(np.int32)).cuda()
    # sources of edge e in row v: v + 1 + (e - off[v])  (mod N), built in slabs of rows
    idx = torch.empty(E_MAX, dtype=torch.int32, device="cuda")
    slab = 1 << 16
    for r0 in range(0, N, slab):
        r1 = min(N, r0 + slab)
        rows = torch.arange(r0, r1, device="cuda", dtype=torch.int64)
        d = torch.from_numpy(deg[r0:r1]).cuda()
        row_of = torch.repeat_interleave(rows, d)
        first = torch.from_numpy(off[r0:r1]).cuda()
        k = torch.arange(int(off[r0]), int(off[r1]), device="cuda", dtype=torch.int64) - \
            torch.repeat_interleave(first, d)
        idx[int(off[r0]):int(off[r1])] = ((row_of + 1 + k) % N).to(torch.int32)
        del rows, d, row_of, first, k
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # out-degree of u: base, plus one for the row v = u - base - 1 (mod N) when v < rem
    outdeg = np.full(N, base, np.int64)
    v = (np.arange(N) - base - 1) % N
    outdeg[v < rem] += 1
    return d_off, idx, deg, off, outdeg


def test_pagerank_at_the_int32_partition_limit(circulant):
    import torch

    import paper_2010_08781_b200 as ipr
    d_off, idx, deg, off, outdeg = circulant
    G = ipr.Graph(ipr.full_partition(N, E_MAX, d_off, idx, None, None))
    G.run("pagerank", mode="pull", iterations=1)
    got = G.values(host=True)
    s = G.stats()
    G.close()
    torch.cuda.empty_cache()
    assert s["supersteps"] == 2 and int(s["messages"][0]) == E_MAX
    # closed form per vertex: outdeg takes two values, base and base + 1, so the sum is
    # (d - m) / (N base) + m / (N (base + 1)) with m (the row's sources of out-degree base + 1)
    # counted exactly by integer prefix sums over the doubled ring
    base = int(outdeg.min())
    ind = (outdeg == base + 1).astype(np.int64)
    cnt = np.concatenate([[0], np.cumsum(np.concatenate([ind, ind]))])
    vv = np.arange(N)
    m = cnt[vv + 1 + deg] - cnt[vv + 1]
    want = 0.15 / N + 0.85 * ((deg - m) * ((1.0 / N) / base) + m * ((1.0 / N) / (base + 1)))
    rel = np.abs(got - want) / want
    assert rel.max() <= 1e-12, (int(np.argmax(rel)), float(rel.max()))


def test_one_edge_past_the_limit_is_refused(circulant):
    import ctypes

    import paper_2010_08781_b200 as ipr
    d_off, idx, deg, off, outdeg = circulant
    desc = ipr.full_partition(N, E_MAX + 1, d_off, idx, None, None).desc()
    desc.csc_edges = E_MAX + 1   # refused from the sizes alone, before any array is read
    h = ctypes.c_void_p()
    st = ipr.load().ipregel_graph_create(ctypes.byref(desc), None, None, ctypes.byref(h))
    assert st == ipr.ERR_UNSUPPORTED
    assert "int32" in ipr.last_error()

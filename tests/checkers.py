"""Brute-force checkers that pin the oracle to things other than itself.

Each is a different algorithm for the same mathematical result (SURVEY.md
8(c) "Pins"): exact-rational k-step PageRank recursion, union-find and
BFS balls for Hash-Min CC, Dijkstra and hop-bounded Bellman-Ford for SSSP.
None of them imports oracle/ or the CUDA package.
"""
from __future__ import annotations

import heapq
from collections import defaultdict
from fractions import Fraction

import numpy as np

INF = 0xFFFFFFFF


def pagerank_exact(n, edges, k):
    """r_0 = 1/N; r_t(v) = 3/20/N + 17/20 * sum_{(u->v)} r_{t-1}(u)/outdeg(u) in
    exact rationals; dangling u contribute nothing."""
    outdeg = [0] * n
    for u, _ in edges:
        outdeg[u] += 1
    r = [Fraction(1, n)] * n
    for _ in range(k):
        acc = [Fraction(0)] * n
        for u, v in edges:
            acc[v] += r[u] / outdeg[u]
        r = [Fraction(3, 20) / n + Fraction(17, 20) * a for a in acc]
    return r


def pagerank_exact_trajectory(n, edges, kmax):
    """[r_0, r_1, ..., r_kmax] of the same exact-rational recursion."""
    outdeg = [0] * n
    for u, _ in edges:
        outdeg[u] += 1
    r = [Fraction(1, n)] * n
    out = [r]
    for _ in range(kmax):
        acc = [Fraction(0)] * n
        for u, v in edges:
            acc[v] += r[u] / outdeg[u]
        r = [Fraction(3, 20) / n + Fraction(17, 20) * a for a in acc]
        out.append(r)
    return out


def pagerank_scipy(n, src, dst, k):
    """k steps of r <- 0.15/N + 0.85 * A^T D^+ r with scipy sparse (f64);
    duplicate edges are summed into A, i.e. counted with multiplicity."""
    import scipy.sparse as sp
    m = len(src)
    A = sp.csr_matrix((np.ones(m), (np.asarray(dst), np.asarray(src))), shape=(n, n))
    outdeg = np.bincount(np.asarray(src), minlength=n).astype(np.float64)
    inv = np.zeros(n)
    nz = outdeg > 0
    inv[nz] = 1.0 / outdeg[nz]
    r = np.full(n, 1.0 / n)
    for _ in range(k):
        r = 0.15 / n + 0.85 * (A @ (r * inv))
    return r


def cc_union_find(n, edges):
    """label(v) = min vertex id of v's component in the undirected graph."""
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for u, v in edges:
        a, b = find(u), find(v)
        if a != b:
            if a < b:
                parent[b] = a
            else:
                parent[a] = b
    return [find(v) for v in range(n)]


def cc_scipy(n, src, dst):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    m = len(src)
    A = sp.csr_matrix((np.ones(m), (np.asarray(src), np.asarray(dst))), shape=(n, n))
    _, comp = connected_components(A, directed=False)
    minid = np.full(comp.max() + 1, n, dtype=np.int64)
    np.minimum.at(minid, comp, np.arange(n))
    return minid[comp].astype(np.uint32)


def cc_ball_labels(n, edges, s):
    """min id within s hops in the undirected graph (Hash-Min after s supersteps)."""
    nbr = defaultdict(list)
    for u, v in edges:
        nbr[u].append(v)
        nbr[v].append(u)
    lab = list(range(n))
    for _ in range(s):
        new = lab[:]
        for v in range(n):
            for u in nbr[v]:
                if lab[u] < new[v]:
                    new[v] = lab[u]
        lab = new
    return lab


def dijkstra(n, edges, source):
    """edges: (u, v, w); INF for unreachable.  Duplicates: min weight wins."""
    adj = defaultdict(list)
    for u, v, w in edges:
        adj[u].append((v, w))
    dist = [INF] * n
    dist[source] = 0
    pq = [(0, source)]
    while pq:
        d, u = heapq.heappop(pq)
        if d != dist[u]:
            continue
        for v, w in adj[u]:
            nd = d + w
            if nd < dist[v]:
                dist[v] = nd
                heapq.heappush(pq, (nd, v))
    return dist


def hop_bounded(n, edges, source, s):
    """min total weight over walks of <= s edges (Bellman-Ford after s rounds)."""
    dist = [INF] * n
    dist[source] = 0
    for _ in range(s):
        new = dist[:]
        for u, v, w in edges:
            if dist[u] != INF and dist[u] + w < new[v]:
                new[v] = dist[u] + w
        dist = new
    return dist


def bfs_levels(n, edges, source):
    adj = defaultdict(list)
    for u, v in edges:
        adj[u].append(v)
    dist = [INF] * n
    dist[source] = 0
    frontier = [source]
    while frontier:
        nxt = []
        for u in frontier:
            for v in adj[u]:
                if dist[v] == INF:
                    dist[v] = dist[u] + 1
                    nxt.append(v)
        frontier = nxt
    return dist


def random_graph(rng, n, m, weighted=False, self_loops=False):
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    if not self_loops:
        keep = src != dst
        src, dst = src[keep], dst[keep]
    w = rng.integers(1, 65, len(src)).astype(np.uint32) if weighted else None
    return src, dst, w


def widest_path(n, edges, source):
    """max over paths source ~> v of the min edge weight (bottleneck Dijkstra); the source gets
    INF (empty path), unreachable vertices 0."""
    adj = defaultdict(list)
    for u, v, w in edges:
        adj[u].append((v, w))
    best = [0] * n
    best[source] = INF
    pq = [(-INF, source)]
    while pq:
        b, u = heapq.heappop(pq)
        b = -b
        if b != best[u]:
            continue
        for v, w in adj[u]:
            nb = min(b, w)
            if nb > best[v]:
                best[v] = nb
                heapq.heappush(pq, (-nb, v))
    return best


def cc_max_label(n, edges):
    """label(v) = max vertex id of v's component in the undirected graph (union-find)."""
    mn = cc_union_find(n, edges)
    top = {}
    for v in range(n):
        top[mn[v]] = max(top.get(mn[v], v), v)
    return [top[mn[v]] for v in range(n)]


def assert_pagerank_mass(stats, n, outdeg_positive=None, rel=1e-12):
    """The rank mass invariant on the GPU's own per-superstep sums (IPREGEL_RUN_PAGERANK_MASS):
    sum_v r_s(v) = 0.15 + 0.85 * sum_{outdeg(u)>0} r_{s-1}(u) for s >= 1 (dangling mass dropped,
    DESIGN.md R4; Pregel's PageRank PAPER.md:515-533), and at superstep 0
    sum r_0 = 1 (r_0 = 1/N) and sum_nd r_0 = (#vertices with outdeg > 0) / N.  A dropped or
    doubled edge moves the left side by its message but not the right side."""
    m, nd = np.asarray(stats["pagerank_mass"]), np.asarray(stats["pagerank_mass_nd"])
    s = int(stats["supersteps"])
    assert s >= 1 and len(m) >= s
    assert abs(m[0] - 1.0) <= rel, m[0]
    if outdeg_positive is not None:
        assert abs(nd[0] - outdeg_positive / n) <= rel * max(outdeg_positive / n, 1e-300), nd[0]
    for t in range(1, s):
        want = 0.15 + 0.85 * nd[t - 1]
        assert abs(m[t] - want) <= rel * want, (t, m[t], want)
        assert 0.0 <= nd[t] <= m[t] * (1 + rel)

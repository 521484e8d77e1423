"""Test helpers: COO -> CSR/CSC arrays (numpy) and library handles for the GPU tests.

Marshalling only; no method arithmetic.  Rows list neighbours in ascending (id, weight) order,
the same canonical order the GPU fixture (inputs/rmat_gpu.cu) produces.
"""
from __future__ import annotations

import numpy as np


def adjacency(n, src, dst, w=None, by_dst=True):
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    row, nbr = (dst, src) if by_dst else (src, dst)
    wk = np.zeros(len(src), np.int64) if w is None else np.asarray(w, np.int64)
    order = np.lexsort((wk, nbr, row))
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, row + 1, 1)
    off = np.cumsum(off).astype(np.int32)
    idx = nbr[order].astype(np.int32)
    ws = None if w is None else np.asarray(w, np.uint32)[order]
    return off, idx, ws


def csr_csc(n, src, dst, w=None):
    csc = adjacency(n, src, dst, w, by_dst=True)
    csr = adjacency(n, src, dst, w, by_dst=False)
    return {"n": int(n), "e": int(len(src)), "csc_off": csc[0], "csc_idx": csc[1], "csc_w": csc[2],
            "csr_off": csr[0], "csr_idx": csr[1], "csr_w": csr[2]}


def to_device(g):
    import torch
    out = dict(g)
    for k in ("csc_off", "csc_idx", "csc_w", "csr_off", "csr_idx", "csr_w"):
        a = g[k]
        if a is None:
            out[k] = None
        else:
            out[k] = torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
    return out


def make_graph(g, partitions=1, host=False, validate=False, weighted=True, bounds=None):
    """Library handle for a graph dict (numpy or torch arrays)."""
    import paper_2010_08781_b200 as ipr
    wkeys = ("csc_w", "csr_w") if weighted else (None, None)
    if host:
        h = {k: (None if g[k] is None else np.ascontiguousarray(
            g[k].cpu().numpy() if hasattr(g[k], "cpu") else g[k]).view(np.int32))
            for k in ("csc_off", "csc_idx", "csc_w", "csr_off", "csr_idx", "csr_w")}
        p = ipr.full_partition(g["n"], g["e"], h["csc_off"], h["csc_idx"], h["csr_off"],
                               h["csr_idx"], h["csc_w"] if weighted else None,
                               h["csr_w"] if weighted else None)
        return ipr.Graph(p, validate=validate)
    d = g if not isinstance(g["csc_off"], np.ndarray) else to_device(g)
    cw = d["csc_w"] if weighted else None
    rw = d["csr_w"] if weighted else None
    if partitions == 1:
        p = ipr.full_partition(d["n"], d["e"], d["csc_off"], d["csc_idx"], d["csr_off"],
                               d["csr_idx"], cw, rw)
        return ipr.Graph(p, validate=validate)
    if bounds is None:
        bounds = ipr.edge_balanced_bounds(d["csc_off"].cpu().numpy(), partitions,
                                          d["csr_off"].cpu().numpy())
    parts = ipr.split_partitions(d["n"], d["e"], bounds, d["csc_off"], d["csc_idx"],
                                 d["csr_off"], d["csr_idx"], cw, rw)
    return ipr.Graph(parts, validate=validate)


def values_np(graph):
    v = graph.values(host=True)
    return v

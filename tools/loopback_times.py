"""PageRank on G loopback partitions of one GPU (the multi-GPU code path minus NVLink): the cost of
the exchange -- fused epilogue stores into the other replicas vs the collective copies after the
kernel -- next to one partition.  Not product code; one GPU cannot show NVLink scaling.

    python tools/loopback_times.py [--config cfg4] [--parts 1,2,4,8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--parts", default="1,2,4,8")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=False, degree_order=True)
n, e = g["n"], g["e"]
ref = None
for parts in [int(x) for x in a.parts.split(",")]:
    if parts == 1:
        ps = [ipr.full_partition(n, e, g["csc_off"], g["csc_idx"], g["csr_off"], g["csr_idx"],
                                 vertex_ids=g["vertex_ids"], degree_ordered=True)]
        modes = ("auto",)
    else:
        bounds = ipr.edge_balanced_bounds(g["csc_off"].cpu().numpy(), parts,
                                          g["csr_off"].cpu().numpy())
        ps = ipr.split_partitions(n, e, bounds, g["csc_off"], g["csc_idx"], g["csr_off"],
                                  g["csr_idx"], vertex_ids=g["vertex_ids"], degree_ordered=True)
        modes = ("fused", "collective")
    G = ipr.Graph(ps)
    for ex in modes:
        for _ in range(2):
            G.run("pagerank", mode="pull", exchange=ex)
        s = G.stats()
        v = G.values(host=True)
        if ref is None:
            ref = v
        same = bool(np.array_equal(v, ref))
        t = s["time_ms"][1:]
        print(f"{parts} partition(s), exchange {ex:10s}: run {float(s['time_ms'].sum()):7.2f} ms, "
              f"gather superstep median {float(np.median(t)):.3f} ms, bit-identical {same}",
              flush=True)
    G.close()

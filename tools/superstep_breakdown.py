"""Per-superstep wall (time_ms) vs delivery-kernel (kernel_ms) time of the three apps at cfg4
(library events).  Not product code."""
import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2010_08781_b200 as ipr
from inputs.gpu import config_graph_device
g = config_graph_device("cfg4", weighted=True, degree_order=True)
G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                 g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"], degree_ordered=True))
for app in ("cc", "sssp", "pagerank"):
    for _ in range(2):
        G.run(app, mode="pull" if app == "pagerank" else "auto")
    s = G.stats()
    print(app, "modes", "".join("ilpr"[m] for m in s["mode"]))
    print("  time  ", [round(float(x), 3) for x in s["time_ms"]])
    print("  kernel", [round(float(x), 3) for x in s["kernel_ms"]])
